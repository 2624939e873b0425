// Kernel shapes, canonical hashing, plans and micro-batch policies.
#include <functional>

#include "planner.h"

namespace ucudnn {

const char* op_name(Op op) {
  switch (op) {
    case Op::Forward: return "Forward";
    case Op::BackwardData: return "BackwardData";
    case Op::BackwardFilter: return "BackwardFilter";
  }
  return "?";
}

bool parse_op(std::string_view s, Op* out) {
  static const Op all[] = {Op::Forward, Op::BackwardData, Op::BackwardFilter};
  for (Op o : all)
    if (s == op_name(o)) { *out = o; return true; }
  return false;
}

// Field validation, reference domain.hpp:133-157.
void Kernel::check() const {
  const std::pair<const char*, std::int64_t> must_be_positive[] = {
      {"batch", batch}, {"in_channels", c}, {"height", h}, {"width", w},
      {"out_channels", k}, {"kernel_h", r}, {"kernel_w", s},
      {"stride_h", stride_h}, {"stride_w", stride_w}};
  for (auto& [label, v] : must_be_positive)
    if (v < 1) throw std::invalid_argument(std::string("kernel field ") + label + " must be >= 1");
  if (pad_h < 0 || pad_w < 0) throw std::invalid_argument("kernel padding must be >= 0");
  if (out_h() < 1 || out_w() < 1)
    throw std::invalid_argument("kernel '" + name + "' has empty output for the given shape/pad/stride");
}

// 64-bit FNV-1a over twelve little-endian 8-byte fields; the layer name is not
// hashed so replicated layers share cost rows (reference domain.hpp:159-180).
std::uint64_t Kernel::hash() const {
  const std::uint64_t fields[12] = {
      std::uint64_t(op), std::uint64_t(batch), std::uint64_t(c), std::uint64_t(h),
      std::uint64_t(w), std::uint64_t(k), std::uint64_t(r), std::uint64_t(s),
      std::uint64_t(pad_h), std::uint64_t(pad_w), std::uint64_t(stride_h), std::uint64_t(stride_w)};
  std::uint64_t x = 0xcbf29ce484222325ULL;  // offset basis 14695981039346656037
  for (std::uint64_t f : fields)
    for (int byte = 0; byte < 8; ++byte) {
      x ^= (f >> (8 * byte)) & 0xff;
      x *= 0x100000001b3ULL;  // prime 1099511628211
    }
  return x;
}

bool Kernel::same_shape(const Kernel& o) const {
  return op == o.op && batch == o.batch && c == o.c && h == o.h && w == o.w && k == o.k &&
         r == o.r && s == o.s && pad_h == o.pad_h && pad_w == o.pad_w &&
         stride_h == o.stride_h && stride_w == o.stride_w;
}

Plan::Plan(std::vector<Micro> micros) : m_(std::move(micros)) {
  if (m_.empty()) throw std::invalid_argument("configuration must not be empty");
  for (const Micro& x : m_) {
    if (x.batch < 1) throw std::invalid_argument("micro_batch must be >= 1");
    if (x.time.negative() || x.ws < 0) throw std::invalid_argument("micro-configuration cost must be >= 0");
  }
  std::sort(m_.begin(), m_.end(), micro_before);
  finish();
}

void Plan::finish() {
  covered_ = 0;
  time_ = Ratio(0);
  ws_ = 0;
  for (const Micro& x : m_) {
    covered_ += x.batch;
    time_ += x.time;
    ws_ = std::max(ws_, x.ws);
  }
}

Plan Plan::one(const Micro& m) { return Plan(std::vector<Micro>{m}); }

// Both inputs are already canonical, so a merge yields the canonical order of
// the union (elements that tie under micro_before are identical).
Plan Plan::join(const Plan& a, const Plan& b) {
  Plan out;
  out.m_.resize(a.m_.size() + b.m_.size());
  std::merge(a.m_.begin(), a.m_.end(), b.m_.begin(), b.m_.end(), out.m_.begin(), micro_before);
  out.covered_ = a.covered_ + b.covered_;
  out.time_ = a.time_ + b.time_;
  out.ws_ = std::max(a.ws_, b.ws_);
  return out;
}

bool plan_before(const Plan& a, const Plan& b) {
  if (a.size() != b.size()) return a.size() < b.size();
  const auto& x = a.micros();
  const auto& y = b.micros();
  for (std::size_t i = 0; i < x.size(); ++i)
    if (x[i] != y[i]) return micro_before(x[i], y[i]);
  return false;
}

const char* policy_name(Policy p) {
  switch (p) {
    case Policy::All: return "all";
    case Policy::PowerOfTwo: return "powerOfTwo";
    case Policy::Undivided: return "undivided";
  }
  return "?";
}

bool parse_policy(std::string_view s, Policy* out) {
  for (Policy p : {Policy::All, Policy::PowerOfTwo, Policy::Undivided})
    if (s == policy_name(p)) { *out = p; return true; }
  return false;
}

// all: 1..B; powerOfTwo: 1,2,4,... <= B plus B itself; undivided: B
// (reference cost_provider.hpp:60-82).
std::vector<std::int64_t> micro_sizes(Policy p, std::int64_t B) {
  if (B < 1) throw std::invalid_argument("mini_batch must be >= 1");
  std::vector<std::int64_t> out;
  if (p == Policy::All) {
    for (std::int64_t b = 1; b <= B; ++b) out.push_back(b);
  } else if (p == Policy::PowerOfTwo) {
    for (std::int64_t b = 1; b > 0 && b <= B; b <<= 1) out.push_back(b);
    if (out.back() != B) out.push_back(B);
  } else {
    out.push_back(B);
  }
  return out;
}

void run_parallel(std::size_t n, unsigned jobs, const std::function<void(std::size_t)>& fn);

}  // namespace ucudnn
