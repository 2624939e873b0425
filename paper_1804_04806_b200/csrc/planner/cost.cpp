// Cost sources: the analytic archetype model, the CSV cost table (the wire
// format between the device benchmarker and both planners) and the provider
// that answers T_mu(b) / C_mu(b) queries.
#include <filesystem>
#include <fstream>
#include <limits>
#include <set>
#include <sstream>

#include "planner.h"

namespace ucudnn {

namespace {

std::int64_t mul_checked(std::int64_t a, std::int64_t b) {
  i128 p = i128(a) * b;
  if (p > std::numeric_limits<std::int64_t>::max() || p < std::numeric_limits<std::int64_t>::min())
    throw std::overflow_error("cost computation overflow");
  return std::int64_t(p);
}

std::string trim(const std::string& s, const char* ws = " \t\r") {
  auto b = s.find_first_not_of(ws);
  if (b == std::string::npos) return "";
  auto e = s.find_last_not_of(ws);
  return s.substr(b, e - b + 1);
}

std::string read_file(const std::string& path, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error(std::string("cannot open ") + what + ": " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

std::string base_name(const std::string& path) {
  return std::filesystem::path(path).filename().string();
}

}  // namespace

// ------------------------------------------------------------ model --------
void CostModel::finalize() {
  std::sort(algs.begin(), algs.end(), [](const AlgSpec& a, const AlgSpec& b) { return a.id < b.id; });
  for (std::size_t i = 0; i < algs.size(); ++i) {
    const AlgCost& c = algs[i].cost;
    if (!(c.tps > Ratio(0))) throw std::invalid_argument("time_per_sample must be > 0");
    if (c.setup.negative()) throw std::invalid_argument("time_setup must be >= 0");
    if (c.wsps < 0 || c.ws_fixed < 0) throw std::invalid_argument("workspace parameters must be >= 0");
    if (c.min_batch < 1) throw std::invalid_argument("min_batch must be >= 1");
    if (c.quantum < 1) throw std::invalid_argument("quantum must be >= 1");
    if (i && algs[i].id == algs[i - 1].id)
      throw std::invalid_argument("duplicate algorithm id " + std::to_string(algs[i].id));
  }
}

// The three synthetic archetypes of reference cost_model.hpp:165-177 /
// data/default.model: (tps, setup, wsps, ws_fixed, min_batch, quantum).
CostModel CostModel::builtin() {
  CostModel m;
  m.algs.push_back({0, "IMPLICIT_GEMM", {Ratio::parse("0.00000005"), Ratio(1), 0, 0, 1, 1}});
  m.algs.push_back({1, "WINOGRAD", {Ratio::parse("0.000000032"), Ratio(1), 8, 16384, 16, 4}});
  m.algs.push_back({2, "FFT", {Ratio::parse("0.000000022"), Ratio(2), 18, 65536, 1, 32}});
  m.finalize();
  return m;
}

// "[algorithm NAME]" sections of "key = value" lines; '#' comments
// (reference cost_model.hpp:182-275).
CostModel CostModel::parse(const std::string& text, const std::string& src) {
  CostModel m;
  std::istringstream in(text);
  std::string line;
  std::size_t ln = 0;
  bool open = false, have_id = false, have_tps = false;
  AlgSpec cur;
  auto fail = [&](const std::string& msg) -> void {
    throw ParseError(src + ":" + std::to_string(ln) + ": " + msg, ln);
  };
  auto close = [&] {
    if (!open) return;
    if (!have_id) fail("algorithm section is missing 'id'");
    if (!have_tps) fail("algorithm section is missing 'time_per_sample'");
    m.algs.push_back(cur);
  };
  while (std::getline(in, line)) {
    ++ln;
    if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
    std::string t = trim(line);
    if (t.empty()) continue;
    if (t[0] == '[') {
      if (t.back() != ']') fail("unterminated section header");
      std::istringstream hs(t.substr(1, t.size() - 2));
      std::string kind, name, extra;
      hs >> kind >> name;
      if (kind != "algorithm" || name.empty() || (hs >> extra)) fail("expected '[algorithm NAME]'");
      close();
      cur = AlgSpec{};
      cur.name = name;
      open = true;
      have_id = have_tps = false;
      continue;
    }
    if (!open) fail("expected '[algorithm NAME]' before parameters");
    auto eq = t.find('=');
    if (eq == std::string::npos) fail("expected 'key = value'");
    std::string key = trim(t.substr(0, eq), " \t"), val = trim(t.substr(eq + 1), " \t");
    if (key.empty() || val.empty()) fail("expected 'key = value'");
    try {
      if (key == "id") { cur.id = std::int32_t(std::stol(val)); have_id = true; }
      else if (key == "time_per_sample") { cur.cost.tps = Ratio::parse(val); have_tps = true; }
      else if (key == "time_setup") cur.cost.setup = Ratio::parse(val);
      else if (key == "ws_per_sample") cur.cost.wsps = std::stoll(val);
      else if (key == "ws_fixed") cur.cost.ws_fixed = std::stoll(val);
      else if (key == "min_batch") cur.cost.min_batch = std::stoll(val);
      else if (key == "quantum") cur.cost.quantum = std::stoll(val);
      else fail("unknown model parameter '" + key + "'");
    } catch (const ParseError&) {
      throw;
    } catch (const std::exception& e) {
      fail("invalid value for '" + key + "': " + e.what());
    }
  }
  close();
  if (m.algs.empty()) throw ParseError(src + ": no algorithm sections", ln);
  try {
    m.finalize();
  } catch (const std::exception& e) {
    throw ParseError(src + ": " + e.what(), ln);
  }
  return m;
}

CostModel CostModel::load(const std::string& path) {
  return parse(read_file(path, "cost model file"), base_name(path));
}

// cost_model.hpp:134-157.
CostRecord CostModel::evaluate(const Kernel& k, std::int32_t alg, std::int64_t b) const {
  const AlgSpec* spec = nullptr;
  for (const AlgSpec& a : algs)
    if (a.id == alg) spec = &a;
  if (!spec) throw std::invalid_argument("unknown algorithm id " + std::to_string(alg));
  k.check();
  if (b < 1) throw std::invalid_argument("micro_batch must be >= 1");
  CostRecord r{{k.hash(), k.op, alg, b}, Ratio(0), 0, false};
  const AlgCost& c = spec->cost;
  if (b < c.min_batch) return r;
  std::int64_t macs = mul_checked(mul_checked(mul_checked(mul_checked(mul_checked(k.c, k.k), k.r), k.s),
                                              k.out_h()), k.out_w());
  std::int64_t input = mul_checked(mul_checked(k.c, k.h), k.w);
  std::int64_t charged = (b + c.quantum - 1) / c.quantum * c.quantum;
  r.time = c.setup + c.tps * Ratio(mul_checked(charged, macs));
  r.ws = c.ws_fixed + mul_checked(c.wsps, mul_checked(b, input));
  if (r.time.negative() || r.ws < 0) throw std::invalid_argument("cost record values must be >= 0");
  r.feasible = true;
  return r;
}

// ------------------------------------------------------------ table --------
const char* const kCsvHeader = "kernel_hash,op_type,algorithm,micro_batch,time_us,workspace_bytes,feasible";

std::string CostTable::format(const CostRecord& r) {
  char hex[24];
  std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)r.key.hash);
  std::string out = hex;
  out += ',';
  out += op_name(r.key.op);
  out += ',' + std::to_string(r.key.alg) + ',' + std::to_string(r.key.batch) + ',' + r.time.str() + ',' +
         std::to_string(r.ws) + ',' + (r.feasible ? "1" : "0");
  return out;
}

// cost_database.hpp:158-222.
std::unique_ptr<CostTable> CostTable::from_csv_text(const std::string& text, const std::string& src) {
  auto t = std::make_unique<CostTable>();
  std::istringstream in(text);
  std::string line;
  std::size_t ln = 0;
  auto fail = [&](const std::string& msg) -> void {
    throw ParseError(src + ":" + std::to_string(ln) + ": " + msg, ln);
  };
  if (!std::getline(in, line)) { ln = 1; fail("empty cost database"); }
  ++ln;
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != kCsvHeader) fail("unexpected header");
  while (std::getline(in, line)) {
    ++ln;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    std::vector<std::string> f;
    for (std::size_t at = 0;;) {
      auto comma = line.find(',', at);
      f.push_back(line.substr(at, comma == std::string::npos ? std::string::npos : comma - at));
      if (comma == std::string::npos) break;
      at = comma + 1;
    }
    if (f.size() != 7) fail("expected 7 comma-separated fields");
    CostRecord r;
    try {
      r.key.hash = std::stoull(f[0], nullptr, 16);
      if (!parse_op(f[1], &r.key.op)) fail("unknown op_type '" + f[1] + "'");
      r.key.alg = std::int32_t(std::stol(f[2]));
      r.key.batch = std::stoll(f[3]);
      r.time = Ratio::parse(f[4]);
      r.ws = std::stoll(f[5]);
      if (f[6] == "1") r.feasible = true;
      else if (f[6] == "0") r.feasible = false;
      else fail("feasible must be 0 or 1");
    } catch (const ParseError&) {
      throw;
    } catch (const std::exception& e) {
      fail(std::string("malformed record: ") + e.what());
    }
    if (r.key.batch < 1) fail("micro_batch must be >= 1");
    if (r.time.negative() || r.ws < 0) fail("costs must be >= 0");
    if (!r.feasible) { r.time = Ratio(0); r.ws = 0; }
    t->rows_[r.key] = r;
  }
  return t;
}

std::unique_ptr<CostTable> CostTable::load(const std::string& path) {
  auto t = from_csv_text(read_file(path, "cost database"), base_name(path));
  t->path_ = path;
  return t;
}

std::unique_ptr<CostTable> CostTable::open(const std::string& path) {
  if (std::filesystem::exists(path)) return load(path);
  auto t = std::make_unique<CostTable>();
  t->path_ = path;
  return t;
}

std::optional<CostRecord> CostTable::get(const CostKey& k) const {
  std::shared_lock lock(mu_);
  auto it = rows_.find(k);
  if (it == rows_.end()) return std::nullopt;
  return it->second;
}

void CostTable::put(const CostRecord& r) {
  std::unique_lock lock(mu_);
  rows_[r.key] = r;
}

std::vector<CostRecord> CostTable::records() const {
  std::shared_lock lock(mu_);
  std::vector<CostRecord> out;
  out.reserve(rows_.size());
  for (auto& kv : rows_) out.push_back(kv.second);
  return out;
}

std::size_t CostTable::size() const {
  std::shared_lock lock(mu_);
  return rows_.size();
}

std::string CostTable::to_csv() const {
  std::shared_lock lock(mu_);
  std::string out = std::string(kCsvHeader) + "\n";
  for (auto& kv : rows_) out += format(kv.second) + "\n";
  return out;
}

// Whole-file rewrite through a temp file + rename so readers never see a torn
// table (cost_database.hpp:119-137).
void CostTable::flush_to(const std::string& path) const {
  std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::trunc | std::ios::binary);
    if (!out) throw std::runtime_error("cannot write cost database: " + tmp);
    out << to_csv();
    if (!out.good()) throw std::runtime_error("write failed: " + tmp);
  }
  std::filesystem::rename(tmp, path);
}

// ------------------------------------------------------------ provider -----
CostSource::CostSource(CostModel model, CostTable* cache) : model_(std::move(model)), table_(cache) {
  for (const AlgSpec& a : model_->algs) {
    ids_.push_back(a.id);
    names_.push_back(a.name);
  }
  if (ids_.empty()) throw std::invalid_argument("cost model has no algorithms");
}

// Algorithm ids are exactly those present in the table; names "alg<id>"
// (cost_provider.hpp:173-185).
CostSource CostSource::table_only(CostTable* table) {
  CostSource s;
  s.table_ = table;
  std::set<std::int32_t> ids;
  for (const CostRecord& r : table->records()) ids.insert(r.key.alg);
  if (ids.empty()) throw std::invalid_argument("measurement database has no records");
  for (std::int32_t id : ids) {
    s.ids_.push_back(id);
    s.names_.push_back("alg" + std::to_string(id));
  }
  return s;
}

std::string CostSource::alg_name(std::int32_t id) const {
  for (std::size_t i = 0; i < ids_.size(); ++i)
    if (ids_[i] == id) return names_[i];
  return "alg" + std::to_string(id);
}

CostRecord CostSource::query(const Kernel& k, std::int32_t alg, std::int64_t b) const {
  CostKey key{k.hash(), k.op, alg, b};
  if (table_)
    if (auto hit = table_->get(key)) return *hit;
  if (!model_) return CostRecord{key, Ratio(0), 0, false};
  CostRecord r = model_->evaluate(k, alg, b);
  if (table_) table_->put(r);
  return r;
}

// T_mu(b): fastest fitting algorithm, ties to smaller workspace then smaller
// id (cost_provider.hpp:132-149).
std::optional<Micro> CostSource::fastest(const Kernel& k, std::int64_t b, std::int64_t limit) const {
  std::optional<Micro> best;
  for (std::int32_t id : ids_) {
    CostRecord r = query(k, id, b);
    if (!r.feasible || r.ws > limit) continue;
    Micro m{id, b, r.time, r.ws};
    if (!best || m.time < best->time ||
        (m.time == best->time && (m.ws < best->ws || (m.ws == best->ws && m.alg < best->alg))))
      best = m;
  }
  return best;
}

// C_mu(b): Pareto front of the fitting algorithms, tie by id
// (cost_provider.hpp:154-170).
std::vector<Micro> CostSource::front(const Kernel& k, std::int64_t b, std::int64_t limit) const {
  std::vector<Micro> cand;
  for (std::int32_t id : ids_) {
    CostRecord r = query(k, id, b);
    if (!r.feasible || r.ws > limit) continue;
    cand.push_back(Micro{id, b, r.time, r.ws});
  }
  return pareto(
      std::move(cand), [](const Micro& m) -> const Ratio& { return m.time; },
      [](const Micro& m) { return m.ws; }, [](const Micro& a, const Micro& b) { return a.alg < b.alg; });
}

}  // namespace ucudnn
