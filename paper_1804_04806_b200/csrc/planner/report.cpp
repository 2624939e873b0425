// Network description files, the whole-network planning harness and the
// reports (the machine report is the byte-level parity document).
#include <cctype>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iomanip>
#include <set>
#include <sstream>

#include "planner.h"

namespace ucudnn {

// ------------------------------------------------------------ harness ------
// WR: each kernel planned independently under the per-kernel limit. WD: one
// selection under the total budget. The undivided baseline is recomputed in
// the same run -- per kernel at the same limit (WR) or at limit / #kernels
// (WD) -- and only totals when every kernel has one (harness.hpp:43-106).
Report plan_network(const CostSource& src, const std::string& name, const std::vector<Kernel>& kernels,
                    const RunConfig& cfg) {
  if (kernels.empty()) throw std::invalid_argument("no kernels to optimize");
  auto t0 = std::chrono::steady_clock::now();
  Report rep;
  rep.mode = cfg.mode;
  rep.policy = cfg.policy;
  rep.network = name;
  rep.batch = kernels.front().batch;
  rep.limit = cfg.limit;
  for (std::int32_t id : src.algs()) rep.algs.emplace_back(id, src.alg_name(id));

  std::vector<Plan> chosen;
  std::int64_t base_limit = cfg.limit;
  if (cfg.mode == Mode::WR) {
    std::vector<std::optional<Plan>> out(kernels.size());
    run_parallel(kernels.size(), cfg.jobs, [&](std::size_t i) {
      out[i] = wr_plan(src, kernels[i], kernels[i].batch, cfg.limit, cfg.policy).plan;
    });
    for (auto& p : out) chosen.push_back(std::move(*p));
  } else {
    WdPlan wd = wd_plan(src, kernels, cfg.limit, cfg.policy, cfg.jobs, cfg.cap);
    chosen = std::move(wd.chosen);
    rep.variables = wd.variables;
    rep.max_front = wd.max_front;
    rep.unique_kernels = wd.unique_kernels;
    base_limit = cfg.limit / std::int64_t(kernels.size());
  }

  bool every = true;
  Ratio base_sum;
  for (std::size_t i = 0; i < kernels.size(); ++i) {
    KernelResult row{kernels[i], chosen[i], chosen[i].time(), chosen[i].ws(), std::nullopt};
    if (auto u = src.fastest(kernels[i], kernels[i].batch, base_limit)) {
      row.baseline = u->time;
      base_sum += u->time;
    } else {
      every = false;
    }
    rep.total += row.time;
    rep.total_ws += row.ws;
    rep.rows.push_back(std::move(row));
  }
  if (every) rep.baseline = base_sum;
  rep.planner_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  rep.check();
  return rep;
}

std::optional<double> Report::speedup() const {
  if (!baseline || total.zero()) return std::nullopt;
  return (*baseline / total).as_double();
}

// Internal consistency (report.hpp:70-99).
void Report::check() const {
  Ratio t, b;
  std::int64_t ws = 0;
  bool every = true;
  for (const KernelResult& r : rows) {
    if (r.time != r.plan.time() || r.ws != r.plan.ws())
      throw std::logic_error("report row disagrees with its configuration");
    t += r.time;
    ws += r.ws;
    if (r.baseline) b += *r.baseline;
    else every = false;
  }
  if (t != total || ws != total_ws) throw std::logic_error("report totals do not match the rows");
  std::optional<Ratio> want = (every && !rows.empty()) ? std::optional<Ratio>(b) : std::nullopt;
  if (baseline != want) throw std::logic_error("baseline total does not match the rows");
  if (mode == Mode::WD && total_ws > limit) throw std::logic_error("wd workspace division exceeds the budget");
}

namespace {
std::string fixed(double v, int digits) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.*f", digits, v);
  return buf;
}
std::string hex16(std::uint64_t h) {
  char buf[24];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return buf;
}
}  // namespace

// Fixed-order "key value" lines (report.hpp:148-197). The first line and the
// note keep the reference's wording so reports diff byte-for-byte.
std::string machine_report(const Report& r) {
  r.check();
  std::ostringstream o;
  o << "ubatch-report 1\n"
    << "mode " << (r.mode == Mode::WR ? "wr" : "wd") << '\n'
    << "policy " << policy_name(r.policy) << '\n'
    << "network " << r.network << '\n'
    << "batch-size " << r.batch << '\n'
    << "workspace-limit " << r.limit << '\n'
    << "workspace-limit-scope " << (r.mode == Mode::WR ? "per-kernel" : "total") << '\n'
    << "algorithm-count " << r.algs.size() << '\n';
  for (auto& [id, nm] : r.algs) o << "algorithm " << id << ' ' << nm << '\n';
  o << "kernel-count " << r.rows.size() << '\n';
  for (std::size_t i = 0; i < r.rows.size(); ++i) {
    const KernelResult& row = r.rows[i];
    const std::string tag = "kernel " + std::to_string(i) + " ";
    o << tag << "layer " << row.kernel.name << '\n'
      << tag << "op " << op_name(row.kernel.op) << '\n'
      << tag << "hash " << hex16(row.kernel.hash()) << '\n'
      << tag << "micro-count " << row.plan.size() << '\n';
    const auto& ms = row.plan.micros();
    for (std::size_t j = 0; j < ms.size(); ++j)
      o << tag << "micro " << j << " algorithm " << ms[j].alg << " batch " << ms[j].batch << " time-us "
        << ms[j].time.str() << " workspace-bytes " << ms[j].ws << '\n';
    o << tag << "time-us " << row.time.str() << '\n'
      << tag << "workspace-bytes " << row.ws << '\n'
      << tag << "baseline-time-us " << (row.baseline ? row.baseline->str() : "n/a") << '\n';
  }
  auto sp = r.speedup();
  o << "total-time-us " << r.total.str() << '\n'
    << "total-workspace-bytes " << r.total_ws << '\n'
    << "baseline-time-us " << (r.baseline ? r.baseline->str() : "n/a") << '\n'
    << "speedup " << (sp ? fixed(*sp, 6) : "n/a") << '\n'
    << "variable-count " << r.variables << '\n'
    << "max-front-size " << r.max_front << '\n'
    << "unique-kernel-count " << r.unique_kernels << '\n'
    << "note times are cost-model sums, not measured wall clock\n"
    << "end\n";
  return o.str();
}

// "FFT@32x8+WINOGRAD@16" (report.hpp:118-141).
std::string plan_summary(const Plan& p, const Report& r) {
  auto name = [&](std::int32_t id) {
    for (auto& [a, nm] : r.algs)
      if (a == id) return nm;
    return "alg" + std::to_string(id);
  };
  std::string out;
  const auto& ms = p.micros();
  for (std::size_t i = 0; i < ms.size();) {
    std::size_t j = i;
    while (j < ms.size() && ms[j].alg == ms[i].alg && ms[j].batch == ms[i].batch) ++j;
    if (!out.empty()) out += '+';
    out += name(ms[i].alg) + "@" + std::to_string(ms[i].batch);
    if (j - i > 1) out += "x" + std::to_string(j - i);
    i = j;
  }
  return out;
}

std::string text_report(const Report& r) {
  r.check();
  std::ostringstream o;
  o << "network " << r.network << ", batch " << r.batch << ", " << r.rows.size() << " kernels\n"
    << "mode " << (r.mode == Mode::WR ? "wr" : "wd") << ", policy " << policy_name(r.policy)
    << ", workspace limit " << r.limit << " B (" << (r.mode == Mode::WR ? "per kernel" : "total") << ")\n\n";
  o << std::left << std::setw(14) << "layer" << std::setw(16) << "op" << std::right << std::setw(14)
    << "time(us)" << std::setw(14) << "ws(bytes)" << std::setw(14) << "baseline(us)" << std::setw(9)
    << "speedup" << "  plan\n";
  for (const KernelResult& row : r.rows) {
    o << std::left << std::setw(14) << row.kernel.name << std::setw(16) << op_name(row.kernel.op) << std::right
      << std::setw(14) << fixed(row.time.as_double(), 2) << std::setw(14) << row.ws;
    if (row.baseline)
      o << std::setw(14) << fixed(row.baseline->as_double(), 2) << std::setw(9)
        << fixed(row.time.zero() ? 0.0 : (*row.baseline / row.time).as_double(), 2);
    else
      o << std::setw(14) << "n/a" << std::setw(9) << "n/a";
    o << "  " << plan_summary(row.plan, r) << '\n';
  }
  o << "\ntotal time " << fixed(r.total.as_double(), 2) << " us";
  if (r.baseline) o << ", undivided baseline " << fixed(r.baseline->as_double(), 2) << " us";
  if (auto sp = r.speedup()) o << ", speedup " << fixed(*sp, 3) << "x";
  o << "\n";
  if (r.mode == Mode::WD)
    o << "workspace division: " << r.total_ws << " of " << r.limit << " B assigned across " << r.rows.size()
      << " kernels (" << r.unique_kernels << " unique), " << r.variables << " choice variables, largest front "
      << r.max_front << "\n";
  else
    o << "total workspace " << r.total_ws << " B across per-kernel slots\n";
  o << "optimizer time " << fixed(r.planner_ms, 2) << " ms\n";
  o << "note: times are cost-table sums, not measured wall clock.\n";
  return o.str();
}

// ------------------------------------------------------------ networks -----
// network NAME / minibatch N / layer NAME channels=C size=HxW filters=K
// kernel=RxS [pad=P] [stride=S]; '#' comments (network.hpp:52-169).
Network parse_network(const std::string& text, const std::string& src) {
  Network net;
  bool have_batch = false;
  std::set<std::string> seen;
  std::size_t ln = 0;
  auto fail = [&](const std::string& msg, std::size_t col = 0) -> void {
    std::string where = src + ":" + std::to_string(ln) + (col ? ":" + std::to_string(col) : "");
    throw ParseError(where + ": " + msg, ln, col);
  };
  auto as_int = [&](const std::string& t, std::size_t col) -> std::int64_t {
    try {
      std::size_t used = 0;
      std::int64_t v = std::stoll(t, &used);
      if (used == t.size()) return v;
    } catch (const std::exception&) {
    }
    fail("expected an integer, got '" + t + "'", col);
    return 0;
  };
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    ++ln;
    if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
    std::vector<std::pair<std::string, std::size_t>> tok;  // token, 1-based column
    for (std::size_t i = 0; i < line.size();) {
      while (i < line.size() && std::isspace((unsigned char)line[i])) ++i;
      std::size_t j = i;
      while (j < line.size() && !std::isspace((unsigned char)line[j])) ++j;
      if (j > i) tok.emplace_back(line.substr(i, j - i), i + 1);
      i = j;
    }
    if (tok.empty()) continue;
    const std::string& d = tok[0].first;
    if (d == "network") {
      if (tok.size() != 2) fail("expected 'network NAME'");
      net.name = tok[1].first;
    } else if (d == "minibatch") {
      if (tok.size() != 2) fail("expected 'minibatch N'");
      net.batch = as_int(tok[1].first, tok[1].second);
      if (net.batch < 1) fail("minibatch must be >= 1", tok[1].second);
      have_batch = true;
    } else if (d == "layer") {
      if (tok.size() < 2) fail("expected 'layer NAME key=value...'");
      Layer L;
      L.name = tok[1].first;
      if (!seen.insert(L.name).second) fail("duplicate layer name '" + L.name + "'", tok[1].second);
      unsigned have = 0;
      for (std::size_t t = 2; t < tok.size(); ++t) {
        const auto& [kv, col] = tok[t];
        auto eq = kv.find('=');
        if (eq == std::string::npos) fail("expected 'key=value'", col);
        std::string key = kv.substr(0, eq), val = kv.substr(eq + 1);
        std::size_t vcol = col + eq + 1;
        auto pair = [&](std::int64_t& a, std::int64_t& b) {
          auto x = val.find('x');
          if (x == std::string::npos) fail("expected 'HxW'", vcol);
          a = as_int(val.substr(0, x), vcol);
          b = as_int(val.substr(x + 1), vcol + x + 1);
        };
        if (key == "channels") { L.c = as_int(val, vcol); have |= 1; }
        else if (key == "size") { pair(L.h, L.w); have |= 2; }
        else if (key == "filters") { L.k = as_int(val, vcol); have |= 4; }
        else if (key == "kernel") { pair(L.r, L.s); have |= 8; }
        else if (key == "pad") L.pad = as_int(val, vcol);
        else if (key == "stride") L.stride = as_int(val, vcol);
        else fail("unknown layer key '" + key + "'", col);
      }
      if (have != 15) fail("layer '" + L.name + "' needs channels=, size=, filters= and kernel=");
      if (L.c < 1 || L.h < 1 || L.w < 1 || L.k < 1 || L.r < 1 || L.s < 1 || L.stride < 1 || L.pad < 0)
        fail("layer '" + L.name + "' has a non-positive dimension");
      net.layers.push_back(L);
    } else {
      fail("unknown directive '" + d + "'", tok[0].second);
    }
  }
  ++ln;
  if (net.layers.empty()) fail("network has no layers");
  if (!have_batch) fail("network is missing 'minibatch N'");
  if (net.name.empty()) net.name = "unnamed";
  return net;
}

Network load_network(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open network file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  std::filesystem::path p(path);
  Network net = parse_network(ss.str(), p.filename().string());
  if (net.name == "unnamed") net.name = p.stem().string();
  return net;
}

// F, BD, BF per layer in layer order (network.hpp:183-212).
std::vector<Kernel> expand(const Network& net, std::int64_t batch_override) {
  std::int64_t B = batch_override > 0 ? batch_override : net.batch;
  if (B < 1) throw std::invalid_argument("batch must be >= 1");
  std::vector<Kernel> out;
  for (const Layer& L : net.layers)
    for (Op op : {Op::Forward, Op::BackwardData, Op::BackwardFilter}) {
      Kernel k;
      k.op = op;
      k.batch = B;
      k.c = L.c; k.h = L.h; k.w = L.w; k.k = L.k; k.r = L.r; k.s = L.s;
      k.pad_h = k.pad_w = L.pad;
      k.stride_h = k.stride_w = L.stride;
      k.name = L.name;
      k.check();
      out.push_back(k);
    }
  return out;
}

}  // namespace ucudnn
