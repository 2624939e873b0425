// Host-side micro-batch planner: cost table -> WR dynamic program / WD
// multiple-choice-knapsack -> per-kernel plans, plus the machine report that
// is the parity document against the reference.
//
// This is a from-scratch restatement of the reference planner `ubatch`
// (/root/reference/proj/include/ubatch/*.hpp). Every decision that can change
// a plan -- canonical orders, tie rules, the DP recurrence, front pruning,
// the branch-and-bound search order -- follows the reference exactly so that
// plans are bit-identical given the same timing table; file:line citations
// sit next to each such rule.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <shared_mutex>
#include <string>
#include <utility>
#include <vector>

#include "ratio.h"

namespace ucudnn {

// ---------------------------------------------------------------- errors --
struct ParseError : std::runtime_error {
  ParseError(const std::string& m, std::size_t line, std::size_t col = 0)
      : std::runtime_error(m), line(line), col(col) {}
  std::size_t line, col;
};
// No plan fits the workspace; min_total_ws >= 0 when the WD solver knows the
// smallest achievable total (reference domain.hpp:48-58).
struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& m, std::int64_t min_total_ws = -1)
      : std::runtime_error(m), min_total_ws(min_total_ws) {}
  std::int64_t min_total_ws;
};

// ------------------------------------------------------------ kernel shape --
enum class Op : std::uint8_t { Forward = 0, BackwardData = 1, BackwardFilter = 2 };
const char* op_name(Op op);
bool parse_op(std::string_view s, Op* out);

// One convolution kernel instance (reference KernelDescriptor,
// domain.hpp:89-121). `batch` is the mini-batch the plan must cover.
struct Kernel {
  Op op = Op::Forward;
  std::int64_t batch = 1, c = 1, h = 1, w = 1, k = 1, r = 1, s = 1;
  std::int64_t pad_h = 0, pad_w = 0, stride_h = 1, stride_w = 1;
  std::string name;

  std::int64_t out_h() const { return (h + 2 * pad_h - r) / stride_h + 1; }
  std::int64_t out_w() const { return (w + 2 * pad_w - s) / stride_w + 1; }
  void check() const;            // domain.hpp:133-157
  std::uint64_t hash() const;    // FNV-1a, domain.hpp:159-180
  bool same_shape(const Kernel& o) const;
};

// -------------------------------------------------------------- plans ------
// One (algorithm, micro-batch) invocation and its cost (domain.hpp:191-207).
struct Micro {
  std::int32_t alg = 0;
  std::int64_t batch = 1;
  Ratio time;            // microseconds
  std::int64_t ws = 0;   // bytes
  bool operator==(const Micro& o) const {
    return alg == o.alg && batch == o.batch && time == o.time && ws == o.ws;
  }
  bool operator!=(const Micro& o) const { return !(*this == o); }
};

// micro-batch descending, algorithm ascending, then time, then workspace
// (domain.hpp:211-217).
inline bool micro_before(const Micro& a, const Micro& b) {
  if (a.batch != b.batch) return a.batch > b.batch;
  if (a.alg != b.alg) return a.alg < b.alg;
  if (a.time != b.time) return a.time < b.time;
  return a.ws < b.ws;
}

// A configuration: micro-batches run back to back sharing one workspace slot,
// so time = sum and workspace = max (domain.hpp:227-267). Members are kept in
// canonical order; equal multisets compare equal.
class Plan {
 public:
  Plan() = default;
  explicit Plan(std::vector<Micro> micros);
  static Plan one(const Micro& m);
  static Plan join(const Plan& a, const Plan& b);  // concat, domain.hpp:269-273

  const std::vector<Micro>& micros() const { return m_; }
  std::size_t size() const { return m_.size(); }
  std::int64_t covered() const { return covered_; }
  const Ratio& time() const { return time_; }
  std::int64_t ws() const { return ws_; }
  bool operator==(const Plan& o) const { return covered_ == o.covered_ && m_ == o.m_; }
  bool operator!=(const Plan& o) const { return !(*this == o); }

 private:
  void finish();
  std::vector<Micro> m_;
  std::int64_t covered_ = 0;
  Ratio time_;
  std::int64_t ws_ = 0;
};

// fewer micro-batches first, then element-wise canonical order
// (domain.hpp:277-285).
bool plan_before(const Plan& a, const Plan& b);

// ------------------------------------------------------------ cost table ---
struct CostKey {
  std::uint64_t hash = 0;
  Op op = Op::Forward;
  std::int32_t alg = 0;
  std::int64_t batch = 1;
  bool operator<(const CostKey& o) const {
    if (hash != o.hash) return hash < o.hash;
    if (op != o.op) return op < o.op;
    if (alg != o.alg) return alg < o.alg;
    return batch < o.batch;
  }
};
struct CostRecord {
  CostKey key;
  Ratio time;
  std::int64_t ws = 0;
  bool feasible = false;
};

// Analytic archetype (cost_model.hpp:33-64): time = setup + tps *
// ceil(b/q)*q * C*K*R*S*OH*OW, ws = ws_fixed + wsps * b * C*H*W.
struct AlgCost {
  Ratio tps, setup;
  std::int64_t wsps = 0, ws_fixed = 0, min_batch = 1, quantum = 1;
};
struct AlgSpec {
  std::int32_t id = 0;
  std::string name;
  AlgCost cost;
};
struct CostModel {
  std::vector<AlgSpec> algs;  // sorted by id, unique
  static CostModel builtin();                                    // cost_model.hpp:165-177
  static CostModel parse(const std::string& text, const std::string& src);  // 182-275
  static CostModel load(const std::string& path);
  void finalize();
  CostRecord evaluate(const Kernel& k, std::int32_t alg, std::int64_t b) const;  // 134-157
};

// Thread-safe keyed store with the reference CSV wire format
// (cost_database.hpp:32-222).
extern const char* const kCsvHeader;
class CostTable {
 public:
  static std::unique_ptr<CostTable> from_csv_text(const std::string& text, const std::string& src);
  static std::unique_ptr<CostTable> load(const std::string& path);
  static std::unique_ptr<CostTable> open(const std::string& path);  // load if exists
  std::optional<CostRecord> get(const CostKey& k) const;
  void put(const CostRecord& r);
  std::vector<CostRecord> records() const;
  std::size_t size() const;
  std::string to_csv() const;
  void flush_to(const std::string& path) const;  // tmp + rename
  const std::string& path() const { return path_; }
  void set_path(const std::string& p) { path_ = p; }
  static std::string format(const CostRecord& r);

 private:
  mutable std::shared_mutex mu_;
  std::map<CostKey, CostRecord> rows_;
  std::string path_;
};

// ------------------------------------------------------------ policies -----
enum class Policy { All = 0, PowerOfTwo = 1, Undivided = 2 };
const char* policy_name(Policy p);
bool parse_policy(std::string_view s, Policy* out);
std::vector<std::int64_t> micro_sizes(Policy p, std::int64_t B);  // cost_provider.hpp:60-82

// Costs for (kernel, algorithm, micro-batch): model-backed with an optional
// write-through table, or table-only where absent rows are infeasible
// (cost_provider.hpp:84-191).
class CostSource {
 public:
  CostSource(CostModel model, CostTable* cache);
  static CostSource table_only(CostTable* table);

  const std::vector<std::int32_t>& algs() const { return ids_; }
  std::string alg_name(std::int32_t id) const;
  CostRecord query(const Kernel& k, std::int32_t alg, std::int64_t b) const;
  std::optional<Micro> fastest(const Kernel& k, std::int64_t b, std::int64_t limit) const;
  std::vector<Micro> front(const Kernel& k, std::int64_t b, std::int64_t limit) const;

 private:
  CostSource() = default;
  std::optional<CostModel> model_;
  CostTable* table_ = nullptr;
  std::vector<std::int32_t> ids_;
  std::vector<std::string> names_;
};

// (time, workspace) Pareto front, pareto.hpp:28-43: sort by (time, ws, tie),
// keep strictly decreasing workspace.
template <class T, class TimeOf, class WsOf, class Tie>
std::vector<T> pareto(std::vector<T> v, TimeOf t, WsOf w, Tie tie) {
  std::sort(v.begin(), v.end(), [&](const T& a, const T& b) {
    int c = Ratio::cmp(t(a), t(b));
    if (c) return c < 0;
    if (w(a) != w(b)) return w(a) < w(b);
    return tie(a, b);
  });
  std::vector<T> out;
  for (auto& x : v)
    if (out.empty() || w(x) < w(out.back())) out.push_back(std::move(x));
  return out;
}

// ------------------------------------------------------------ planners -----
struct WrRow {
  bool ok = false;
  Ratio time;
  std::int64_t split = 0;
  std::optional<Plan> plan;
};
std::vector<WrRow> wr_table(const CostSource& src, const Kernel& k, std::int64_t B,
                            std::int64_t limit, Policy p);
struct WrPlan {
  Plan plan;
  Ratio time;
};
WrPlan wr_plan(const CostSource& src, const Kernel& k, std::int64_t B, std::int64_t limit, Policy p);

constexpr std::size_t kFrontCap = 4096;
std::vector<Plan> desirable(std::vector<Plan> plans);  // wd_optimizer.hpp:41-64
struct PlanSet {
  Kernel kernel;
  std::vector<Plan> members;  // time ascending, workspace descending
};
PlanSet plan_front(const CostSource& src, const Kernel& k, std::int64_t B, std::int64_t budget,
                   Policy p, std::size_t cap = kFrontCap);
struct Selection {
  std::vector<Plan> chosen;
  Ratio time;
  std::int64_t ws = 0;
};
struct SelectionProblem {
  std::vector<PlanSet> sets;
  std::int64_t budget = 0;
};
Selection select_plans(const SelectionProblem& prob);  // ilp_solve, 569-572
void check_selection(const SelectionProblem& prob, const Selection& s);
struct WdPlan {
  std::vector<Kernel> kernels;
  std::vector<Plan> chosen;
  Ratio time;
  std::int64_t ws = 0;
  std::size_t variables = 0, max_front = 0, unique_kernels = 0;
};
WdPlan wd_plan(const CostSource& src, const std::vector<Kernel>& kernels, std::int64_t budget,
               Policy p, unsigned jobs = 1, std::size_t cap = kFrontCap);

void run_parallel(std::size_t n, unsigned jobs, const std::function<void(std::size_t)>& fn);

// ------------------------------------------------------------ reports ------
enum class Mode { WR = 0, WD = 1 };
struct KernelResult {
  Kernel kernel;
  Plan plan;
  Ratio time;
  std::int64_t ws = 0;
  std::optional<Ratio> baseline;
};
struct Report {
  Mode mode = Mode::WR;
  Policy policy = Policy::All;
  std::string network;
  std::int64_t batch = 0;
  std::int64_t limit = 0;
  std::vector<std::pair<std::int32_t, std::string>> algs;
  std::vector<KernelResult> rows;
  Ratio total;
  std::int64_t total_ws = 0;
  std::optional<Ratio> baseline;
  std::size_t variables = 0, max_front = 0, unique_kernels = 0;
  double planner_ms = 0;
  std::optional<double> speedup() const;
  void check() const;
};
struct RunConfig {
  Mode mode = Mode::WR;
  Policy policy = Policy::All;
  std::int64_t limit = 0;
  unsigned jobs = 1;
  std::size_t cap = kFrontCap;
};
Report plan_network(const CostSource& src, const std::string& name, const std::vector<Kernel>& kernels,
                    const RunConfig& cfg);  // harness.hpp:43-106
std::string machine_report(const Report& r);  // report.hpp:148-197
std::string text_report(const Report& r);     // report.hpp:199-254
std::string plan_summary(const Plan& p, const Report& r);

// ------------------------------------------------------------ networks -----
struct Layer {
  std::string name;
  std::int64_t c = 1, h = 1, w = 1, k = 1, r = 1, s = 1, pad = 0, stride = 1;
};
struct Network {
  std::string name;
  std::int64_t batch = 1;
  std::vector<Layer> layers;
};
Network parse_network(const std::string& text, const std::string& src);  // network.hpp:56-169
Network load_network(const std::string& path);
std::vector<Kernel> expand(const Network& net, std::int64_t batch_override = 0);  // 183-212

}  // namespace ucudnn
