// TEST INFRASTRUCTURE ONLY -- the planner oracle.
//
// A thin driver over the *unmodified* reference planner headers, compiled
// straight from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/ref_plan. It does what the reference CLI `ubatch optimize`
// does (tools/main.cpp:116-155; that CLI needs CLI11, which is absent) and
// generates the seeded random instances used for planner parity. Only tests/
// and tests/golden/make_golden.py run it; the product never does.
//
//   ref_plan optimize NET BATCH MODE POLICY LIMIT JOBS COST [FLUSH_CSV]
//       COST = "builtin" | model file | measurement CSV (by header)
//       prints the machine report (report.hpp:148-197)
//   ref_plan random OUTDIR COUNT SEED0
//       writes OUTDIR/<i>.{net,model,csv,args,report} for COUNT seeded
//       instances: a random synthetic model (random_instances.hpp:49-63),
//       1-3 tiny layers, batch 1-12, random mode/policy/budget. The CSV is
//       the model-backed run's write-through cache (cost_provider.hpp:120-126).
#include <cstdio>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "ubatch/cost_database.hpp"
#include "ubatch/cost_model.hpp"
#include "ubatch/cost_provider.hpp"
#include "ubatch/harness.hpp"
#include "ubatch/network.hpp"
#include "ubatch/random_instances.hpp"
#include "ubatch/report.hpp"

using namespace ubatch;

static bool is_csv(const std::string& path) {
  std::ifstream in(path);
  std::string first;
  if (!in || !std::getline(in, first)) return false;
  if (!first.empty() && first.back() == '\r') first.pop_back();
  return first == kCostCsvHeader;
}

static int optimize(int argc, char** argv) {
  if (argc < 9) return 2;
  NetworkDescription net = load_network(argv[2]);
  long long batch = std::stoll(argv[3]);
  std::vector<KernelDescriptor> kernels =
      expand_kernels(net, batch > 0 ? std::optional<std::int64_t>(batch) : std::nullopt);
  RunOptions opt;
  opt.mode = std::string(argv[4]) == "wd" ? OptMode::kWd : OptMode::kWr;
  opt.policy = *parse_policy(argv[5]);
  opt.workspace_limit = std::stoll(argv[6]);
  opt.jobs = unsigned(std::stoul(argv[7]));
  std::string cost = argv[8];
  std::optional<CostDatabase> meas, cache;
  std::optional<CostProvider> provider;
  if (cost != "builtin" && is_csv(cost)) {
    meas = CostDatabase::load(cost);
    provider = CostProvider::from_database(*meas);
  } else {
    CostModel model = cost == "builtin" ? builtin_model() : load_model(cost);
    if (argc > 9) cache = CostDatabase::open(argv[9]);
    provider.emplace(std::move(model), cache ? &*cache : nullptr);
  }
  try {
    OptimizationReport rep = run_optimization(*provider, net.name, kernels, opt);
    write_machine_report(std::cout, rep);
  } catch (const infeasible_error& e) {
    std::cout << "infeasible " << e.min_total_workspace() << "\n" << e.what() << "\n";
    if (cache) cache->flush();
    return 3;
  }
  if (cache) cache->flush();
  return 0;
}

static void write_model(std::ostream& o, const CostModel& m) {
  for (const auto& a : m.algorithms()) {
    o << "[algorithm " << a.name << "]\n"
      << "id = " << a.id.value << "\n"
      << "time_per_sample = " << a.cost.time_per_sample.to_string() << "\n"
      << "time_setup = " << a.cost.time_setup.to_string() << "\n"
      << "ws_per_sample = " << a.cost.ws_per_sample << "\n"
      << "ws_fixed = " << a.cost.ws_fixed << "\n"
      << "min_batch = " << a.cost.min_batch << "\n"
      << "quantum = " << a.cost.quantum << "\n\n";
  }
}

static int random_instances(int argc, char** argv) {
  if (argc < 5) return 2;
  std::string dir = argv[2];
  int count = std::stoi(argv[3]);
  std::uint64_t seed0 = std::stoull(argv[4]);
  const BatchSizePolicy policies[] = {BatchSizePolicy::kAll, BatchSizePolicy::kPowerOfTwo,
                                      BatchSizePolicy::kUndivided};
  for (int i = 0; i < count; ++i) {
    std::mt19937_64 rng(seed0 + std::uint64_t(i));
    CostModel model = random_model(rng, int(pick(rng, 1, 3)));
    bool wd = pick(rng, 0, 1) == 1;
    std::int64_t batch = pick(rng, 1, wd ? 8 : 12);
    int layers = int(pick(rng, 1, 3));
    std::ostringstream net;
    net << "network rnd" << i << "\nminibatch " << batch << "\n";
    for (int l = 0; l < layers; ++l) {
      // channels 1..3 scale every cost; a repeated channel count yields
      // replicated kernel hashes (shared fronts in WD)
      net << "layer L" << l << " channels=" << pick(rng, 1, 3) << " size=1x1 filters=1 kernel=1x1\n";
    }
    BatchSizePolicy policy = policies[pick(rng, 0, 2)];
    std::int64_t limit = random_budget(rng, batch) * (wd ? 3 * layers : 1);
    std::string base = dir + "/" + std::to_string(i);
    { std::ofstream(base + ".net") << net.str(); }
    { std::ofstream o(base + ".model"); write_model(o, model); }
    {
      std::ofstream(base + ".args") << (wd ? "wd" : "wr") << " " << to_string(policy) << " " << limit << "\n";
    }
    NetworkDescription nd = load_network(base + ".net");
    std::vector<KernelDescriptor> kernels = expand_kernels(nd);
    CostDatabase db;
    CostProvider provider(model, &db);
    RunOptions opt;
    opt.mode = wd ? OptMode::kWd : OptMode::kWr;
    opt.policy = policy;
    opt.workspace_limit = limit;
    std::ofstream rep(base + ".report");
    try {
      write_machine_report(rep, run_optimization(provider, nd.name, kernels, opt));
    } catch (const infeasible_error& e) {
      rep << "infeasible " << e.min_total_workspace() << "\n";
    }
    db.flush_to(base + ".csv");
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::string cmd = argv[1];
  try {
    if (cmd == "optimize") return optimize(argc, argv);
    if (cmd == "random") return random_instances(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
  return 2;
}
