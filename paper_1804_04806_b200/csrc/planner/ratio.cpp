#include "ratio.h"

#include <limits>

namespace ucudnn {

std::string i128_to_string(i128 v) {
  if (v == 0) return "0";
  bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
  char buf[64];
  int p = 63;
  buf[p] = 0;
  while (u) { buf[--p] = char('0' + int(u % 10)); u /= 10; }
  if (neg) buf[--p] = '-';
  return std::string(buf + p);
}

Ratio Ratio::reduce(i128 n, i128 d) {
  if (d == 0) throw std::domain_error("Ratio: zero denominator");
  if (d < 0) { n = -n; d = -d; }
  i128 a = n < 0 ? -n : n, b = d;
  while (b != 0) { i128 t = a % b; a = b; b = t; }
  if (a > 1) { n /= a; d /= a; }
  const i128 hi = std::numeric_limits<std::int64_t>::max();
  const i128 lo = std::numeric_limits<std::int64_t>::min();
  if (n > hi || n < lo || d > hi) throw std::overflow_error("Ratio: value does not fit 64 bits");
  Ratio r;
  r.n_ = std::int64_t(n);
  r.d_ = std::int64_t(d);
  return r;
}

Ratio Ratio::parse(std::string_view s) {
  if (s.empty()) throw std::invalid_argument("Ratio: empty value");
  if (auto slash = s.find('/'); slash != std::string_view::npos) {
    Ratio a = parse(s.substr(0, slash)), b = parse(s.substr(slash + 1));
    if (a.d_ != 1 || b.d_ != 1) throw std::invalid_argument("Ratio: fraction parts must be integers");
    return reduce(a.n_, b.n_);
  }
  std::size_t i = 0;
  bool neg = false;
  if (s[0] == '+' || s[0] == '-') { neg = s[0] == '-'; i = 1; }
  const i128 cap = std::numeric_limits<std::int64_t>::max();
  i128 n = 0, d = 1;
  bool digits = false, point = false;
  for (; i < s.size(); ++i) {
    char c = s[i];
    if (c == '.') {
      if (point) throw std::invalid_argument("Ratio: repeated decimal point");
      point = true;
      continue;
    }
    if (c < '0' || c > '9') throw std::invalid_argument("Ratio: invalid character in number");
    n = n * 10 + (c - '0');
    if (point) d *= 10;
    if (n > cap || d > cap) throw std::overflow_error("Ratio: literal too large");
    digits = true;
  }
  if (!digits) throw std::invalid_argument("Ratio: no digits in number");
  return reduce(neg ? -n : n, d);
}

std::string Ratio::str() const {
  if (d_ == 1) return std::to_string(n_);
  std::int64_t rest = d_;
  int p2 = 0, p5 = 0;
  while (rest % 2 == 0) { rest /= 2; ++p2; }
  while (rest % 5 == 0) { rest /= 5; ++p5; }
  int k = p2 > p5 ? p2 : p5;
  if (rest != 1 || k > 18) return std::to_string(n_) + "/" + std::to_string(d_);
  i128 scale = 1;
  for (int i = 0; i < k; ++i) scale *= 10;
  i128 mag = i128(n_ < 0 ? -i128(n_) : i128(n_)) * (scale / d_);
  std::string frac = i128_to_string(mag % scale);
  if (int(frac.size()) < k) frac.insert(0, std::size_t(k) - frac.size(), '0');
  return std::string(n_ < 0 ? "-" : "") + i128_to_string(mag / scale) + "." + frac;
}

}  // namespace ucudnn
