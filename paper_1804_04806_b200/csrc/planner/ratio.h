// Exact 64-bit rational used for every time value the planner touches.
//
// Semantics follow the reference's Rat64 (/root/reference/proj/include/
// ubatch/rational.hpp:33-230): values are kept gcd-normalised with a positive
// denominator, arithmetic goes through 128-bit intermediates and a normalised
// result that does not fit 64 bits raises std::overflow_error. Because the
// normalised form of a rational is unique, any correct implementation of
// these operations yields the same (num, den) pairs as the reference, which
// is what makes plans and machine reports byte-comparable.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>

namespace ucudnn {

using i128 = __int128;

class Ratio {
 public:
  constexpr Ratio() = default;
  constexpr Ratio(std::int64_t v) : n_(v), d_(1) {}  // NOLINT implicit int
  Ratio(std::int64_t n, std::int64_t d) { *this = reduce(n, d); }

  // "17", "-4.25", ".5", "3/4" (reference parse: rational.hpp:161-202).
  static Ratio parse(std::string_view s);

  std::int64_t num() const { return n_; }
  std::int64_t den() const { return d_; }
  bool zero() const { return n_ == 0; }
  bool negative() const { return n_ < 0; }
  double as_double() const { return double(n_) / double(d_); }

  // Exact decimal when den = 2^a 5^b with max(a,b) <= 18, else "n/d"
  // (reference to_string: rational.hpp:204-230).
  std::string str() const;

  friend Ratio operator+(const Ratio& a, const Ratio& b) { return add(a, b, false); }
  friend Ratio operator-(const Ratio& a, const Ratio& b) { return add(a, b, true); }
  friend Ratio operator*(const Ratio& a, const Ratio& b) {
    // cross-cancel before multiplying so the 128-bit products cannot overflow
    std::int64_t g1 = gcd64(a.n_, b.d_), g2 = gcd64(b.n_, a.d_);
    return reduce(i128(a.n_ / g1) * (b.n_ / g2), i128(a.d_ / g2) * (b.d_ / g1));
  }
  friend Ratio operator/(const Ratio& a, const Ratio& b) {
    if (b.n_ == 0) throw std::domain_error("Ratio: division by zero");
    std::int64_t g1 = gcd64(a.n_, b.n_), g2 = gcd64(a.d_, b.d_);
    return reduce(i128(a.n_ / g1) * (b.d_ / g2), i128(a.d_ / g2) * (b.n_ / g1));
  }
  Ratio& operator+=(const Ratio& o) { return *this = *this + o; }
  Ratio& operator-=(const Ratio& o) { return *this = *this - o; }

  friend bool operator==(const Ratio& a, const Ratio& b) { return a.n_ == b.n_ && a.d_ == b.d_; }
  friend bool operator!=(const Ratio& a, const Ratio& b) { return !(a == b); }
  friend bool operator<(const Ratio& a, const Ratio& b) { return cmp(a, b) < 0; }
  friend bool operator>(const Ratio& a, const Ratio& b) { return cmp(a, b) > 0; }
  friend bool operator<=(const Ratio& a, const Ratio& b) { return cmp(a, b) <= 0; }
  friend bool operator>=(const Ratio& a, const Ratio& b) { return cmp(a, b) >= 0; }
  static int cmp(const Ratio& a, const Ratio& b) {
    i128 l = i128(a.n_) * b.d_, r = i128(b.n_) * a.d_;
    return l < r ? -1 : (l > r ? 1 : 0);
  }

  static std::int64_t gcd64(std::int64_t a, std::int64_t b) {
    std::uint64_t x = a < 0 ? 0 - std::uint64_t(a) : std::uint64_t(a);
    std::uint64_t y = b < 0 ? 0 - std::uint64_t(b) : std::uint64_t(b);
    while (y) { std::uint64_t t = x % y; x = y; y = t; }
    return x == 0 ? 1 : std::int64_t(x);
  }

  static Ratio reduce(i128 n, i128 d);

 private:
  static Ratio add(const Ratio& a, const Ratio& b, bool sub) {
    std::int64_t g = gcd64(a.d_, b.d_);
    i128 rhs = i128(b.n_) * (a.d_ / g);
    i128 n = i128(a.n_) * (b.d_ / g) + (sub ? -rhs : rhs);
    return reduce(n, i128(a.d_ / g) * b.d_);
  }
  std::int64_t n_ = 0;
  std::int64_t d_ = 1;
};

std::string i128_to_string(i128 v);

}  // namespace ucudnn
