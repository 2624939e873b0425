// C ABI (include/ucudnn.h): handle, descriptors, benchmarker, planner glue
// and the micro-batch executor. No exception crosses this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/ucudnn.h"
#include "../kernels/igemm.h"
#include "../planner/planner.h"
#include "algos.h"
#include "../kernels/bfilter.h"
#include "../kernels/precomp.h"

using namespace ucudnn;

// ------------------------------------------------------------ errors -------
namespace {
thread_local std::string g_last_error;
thread_local std::int64_t g_min_ws = -1;

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
ucudnnStatus_t guarded(F&& body) {
  g_last_error.clear();
  try {
    return body();
  } catch (const InfeasibleError& e) {
    g_last_error = e.what();
    g_min_ws = e.min_total_ws;
    return UCUDNN_STATUS_NOT_SUPPORTED;
  } catch (const ParseError& e) {
    g_last_error = e.what();
    return UCUDNN_STATUS_BAD_PARAM;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return UCUDNN_STATUS_BAD_PARAM;
  } catch (const CudaFailure& e) {
    g_last_error = e.what();
    return UCUDNN_STATUS_EXECUTION_FAILED;
  } catch (const std::bad_alloc& e) {
    g_last_error = "allocation failed";
    return UCUDNN_STATUS_ALLOC_FAILED;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return UCUDNN_STATUS_INTERNAL_ERROR;
  } catch (...) {
    g_last_error = "unknown error";
    return UCUDNN_STATUS_INTERNAL_ERROR;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// The handle's deterministic setting on the launching host thread for the
// duration of a call (kernel launchers read it when sizing split-K grids).
// Same for the FP32-faithful math mode (workspace sizes and runs read it).
struct ModeScope {
  bool prev_det, prev_faithful;
  ModeScope(bool det, bool faith) : prev_det(deterministic()), prev_faithful(faithful()) {
    set_deterministic(det);
    set_faithful(faith);
  }
  ~ModeScope() {
    set_deterministic(prev_det);
    set_faithful(prev_faithful);
  }
};
}  // namespace

struct ucudnnTensorStruct {
  int n = 0, c = 0, h = 0, w = 0;
};
struct ucudnnFilterStruct {
  int k = 0, c = 0, r = 0, s = 0;
};
struct ucudnnConvolutionStruct {
  int ph = 0, pw = 0, sh = 1, sw = 1;
};

struct ucudnnContext {
  int device = 0;
  cudaStream_t stream = nullptr;
  Policy policy = Policy::PowerOfTwo;
  Mode mode = Mode::WR;
  std::int64_t total_ws = 0;
  std::int64_t report_limit = 0;
  int warmup = 3, iters = 10;
  bool deterministic = false;  // ucudnnSetDeterministic / UCUDNN_DETERMINISTIC
  bool faithful = false;       // ucudnnSetMathMode(UCUDNN_MATH_FP32_FAITHFUL) / UCUDNN_MATH_MODE=fp32
  std::unique_ptr<CostTable> table = std::make_unique<CostTable>();
  std::string db_path;

  struct Entry {
    Kernel kernel;
    std::int64_t limit = 0;
    bool planned = false;
    Plan plan;
    std::size_t arena_offset = 0;
  };
  std::vector<Entry> entries;
  bool wd_stale = true;
  // WD: after the first optimisation the network is known; a repeated
  // Get*Algorithm for a registered (op, shape) returns its entry instead of
  // registering another kernel ("a library call after network
  // initialization, which ignores subsequent cudnnGetConvolution*Algorithm
  // calls"), so framework re-queries neither grow the ILP nor move the arena
  bool wd_frozen = false;
  void* arena = nullptr;
  std::size_t arena_bytes = 0;

  // Benchmark state of one device: operand scratch, workspace, events and
  // the L2 flush buffer (a plan's micro-batches stream their slices from
  // HBM; timing L2-hot repeats under-costs bandwidth-bound algorithms.
  // UCUDNN_BENCH_FLUSH_MB, default 256 (> the 126 MB L2); 0 = off).
  struct BenchSlot {
    int device = 0;
    cudaStream_t stream = nullptr;  // own stream; the primary slot uses the handle's
    float* scratch = nullptr;
    std::size_t scratch_elems = 0;
    void* ws = nullptr;
    std::size_t ws_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void* flush = nullptr;
    std::size_t flush_bytes = std::size_t(-1);
    void release() {
      if (scratch) cudaFree(scratch);
      if (ws) cudaFree(ws);
      if (flush) cudaFree(flush);
      if (ev0) cudaEventDestroy(ev0);
      if (ev1) cudaEventDestroy(ev1);
      if (stream) cudaStreamDestroy(stream);
      *this = BenchSlot{};
    }
  };
  BenchSlot primary;
  // ucudnnSetBenchmarkDevices: one slot (and host thread) per listed device;
  // empty = the primary slot on the handle's device and stream
  std::vector<std::unique_ptr<BenchSlot>> slots;

  void release_slots() {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& sl : slots) {
      cudaSetDevice(sl->device);
      sl->release();
    }
    slots.clear();
    cudaSetDevice(cur);
  }

  ~ucudnnContext() {
    if (arena) cudaFree(arena);
    primary.stream = nullptr;  // the handle's stream is the caller's
    primary.release();
    release_slots();
  }
};

namespace {

ConvShape shape_from11(const std::int64_t* s) {
  ConvShape c;
  c.N = int(s[0]); c.C = int(s[1]); c.H = int(s[2]); c.W = int(s[3]); c.K = int(s[4]); c.R = int(s[5]);
  c.S = int(s[6]); c.ph = int(s[7]); c.pw = int(s[8]); c.sh = int(s[9]); c.sw = int(s[10]);
  return c;
}

Kernel kernel_from(Op op, const ConvShape& s, const std::string& name) {
  Kernel k;
  k.op = op; k.batch = s.N; k.c = s.C; k.h = s.H; k.w = s.W; k.k = s.K; k.r = s.R; k.s = s.S;
  k.pad_h = s.ph; k.pad_w = s.pw; k.stride_h = s.sh; k.stride_w = s.sw;
  k.name = name;
  k.check();
  return k;
}

ConvShape shape_of(const Kernel& k) {
  ConvShape s;
  s.N = int(k.batch); s.C = int(k.c); s.H = int(k.h); s.W = int(k.w); s.K = int(k.k); s.R = int(k.r);
  s.S = int(k.s); s.ph = int(k.pad_h); s.pw = int(k.pad_w); s.sh = int(k.stride_h); s.sw = int(k.stride_w);
  return s;
}

ConvShape conv_shape(const ucudnnTensorStruct* x, const ucudnnFilterStruct* w, const ucudnnConvolutionStruct* c) {
  require(x && w && c, "null descriptor");
  require(x->c == w->c, "filter in-channels must match input");
  ConvShape s;
  s.N = x->n; s.C = x->c; s.H = x->h; s.W = x->w; s.K = w->k; s.R = w->r; s.S = w->s;
  s.ph = c->ph; s.pw = c->pw; s.sh = c->sh; s.sw = c->sw;
  require(s.N > 0 && s.C > 0 && s.H > 0 && s.W > 0 && s.K > 0 && s.R > 0 && s.S > 0, "dims must be >= 1");
  require(s.OH() >= 1 && s.OW() >= 1, "empty convolution output");
  return s;
}

std::int64_t algo_ws(int op, const ConvShape& s, int algo, bool* ok) {
  const AlgoImpl* a = find_algo(algo);
  // the FP32-faithful mode needs operands the tensor core consumes as given
  *ok = a && a->supports(op, s) && (!faithful() || a->splits_exact);
  return *ok ? algo_workspace(a, op, s) : 0;
}

using BenchSlot = ucudnnContext::BenchSlot;

void ensure_scratch(BenchSlot* h, std::size_t elems) {
  if (elems <= h->scratch_elems) return;
  if (h->scratch) cudaFree(h->scratch);
  h->scratch = nullptr;
  h->scratch_elems = 0;
  cuda_check(cudaMalloc(&h->scratch, elems * sizeof(float)), "cudaMalloc(bench scratch)");
  h->scratch_elems = elems;
  // deterministic pseudo-random contents (values in [-1, 1))
  std::vector<float> host(std::min<std::size_t>(elems, 1 << 22));
  std::mt19937 rng(1804);
  for (auto& v : host) v = float(int(rng() % 2001) - 1000) / 1000.f;
  for (std::size_t off = 0; off < elems; off += host.size()) {
    std::size_t n = std::min(host.size(), elems - off);
    cuda_check(cudaMemcpy(h->scratch + off, host.data(), n * sizeof(float), cudaMemcpyHostToDevice),
               "cudaMemcpy(bench scratch)");
  }
}

// false when the device cannot hold the workspace (the row is then recorded
// infeasible instead of aborting the whole Get*Algorithm)
bool ensure_bench_ws(BenchSlot* h, std::size_t bytes) {
  if (bytes <= h->ws_bytes) return true;
  if (h->ws) cudaFree(h->ws);
  h->ws = nullptr;
  h->ws_bytes = 0;
  cudaError_t e = cudaMalloc(&h->ws, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // clear the sticky-free allocation error
    return false;
  }
  cuda_check(e, "cudaMalloc(bench workspace)");
  h->ws_bytes = bytes;
  return true;
}

// CUDA-event steady-state time of one algorithm at one micro-batch, in
// integer ns (median of `iters` L2-flushed runs with the filter operand
// already prepared, kFilterReady), on `h`'s device and `stream` (the caller
// has made that device current); -1 when its workspace does not fit in
// device memory. With `prep_ms` non-null and negative, also measures the
// batch-independent filter preparation (packing, Winograd / FFT filter
// transforms) as median(whole call) - median(steady) from interleaved runs.
std::int64_t time_once(BenchSlot* h, cudaStream_t stream, int warmup, int iters, int op, const ConvShape& s,
                       int algo, std::int64_t ws, double* prep_ms = nullptr) {
  const AlgoImpl* a = find_algo(algo);
  // sub-buffers 256 B aligned, as a framework's allocations are: TMA maps
  // built on user tensors (dy read in place) need 16 B aligned bases
  auto al = [](std::size_t e) { return (e + 63) / 64 * 64; };
  std::size_t xe = al(std::size_t(s.x_elems())), ye = al(std::size_t(s.y_elems())), we = std::size_t(s.w_elems());
  ensure_scratch(h, xe + ye + we + 64);
  if (!ensure_bench_ws(h, std::size_t(std::max<std::int64_t>(ws, 256)))) return -1;
  float* x = h->scratch;
  float* y = x + xe;
  float* w = y + ye;
  const float *ia, *ib;
  float* out;
  if (op == 0) { ia = x; ib = w; out = y; }
  else if (op == 1) { ia = y; ib = w; out = x; }
  else { ia = x; ib = y; out = w; }
  if (!h->ev0) {
    cuda_check(cudaEventCreate(&h->ev0), "cudaEventCreate");
    cuda_check(cudaEventCreate(&h->ev1), "cudaEventCreate");
  }
  for (int i = 0; i < std::max(1, warmup); ++i)
    cuda_check(algo_run(a, op, s, ia, ib, out, h->ws, 1.f, 0.f, stream, i ? kFilterReady : 0), "benchmark warm-up");
  if (h->flush_bytes == std::size_t(-1)) {
    const char* e = std::getenv("UCUDNN_BENCH_FLUSH_MB");
    h->flush_bytes = std::size_t(e ? std::max(0, std::atoi(e)) : 256) << 20;
    if (h->flush_bytes) cuda_check(cudaMalloc(&h->flush, h->flush_bytes), "cudaMalloc(L2 flush buffer)");
  }
  const bool want_prep = prep_ms && *prep_ms < 0;
  std::vector<float> ms[2];  // [0] steady state (kFilterReady), [1] whole call (filter prepared)
  for (int i = 0; i < (want_prep ? 2 : 1) * std::max(1, iters); ++i) {
    const int kind = want_prep ? (i & 1) : 0;
    if (h->flush_bytes) cuda_check(cudaMemsetAsync(h->flush, i & 0xff, h->flush_bytes, stream), "L2 flush");
    cuda_check(cudaEventRecord(h->ev0, stream), "cudaEventRecord");
    cuda_check(algo_run(a, op, s, ia, ib, out, h->ws, 1.f, 0.f, stream, kind ? 0 : kFilterReady), "benchmark run");
    cuda_check(cudaEventRecord(h->ev1, stream), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(h->ev1), "cudaEventSynchronize");
    float t = 0;
    cuda_check(cudaEventElapsedTime(&t, h->ev0, h->ev1), "cudaEventElapsedTime");
    ms[kind].push_back(t);
  }
  for (auto& v : ms) std::sort(v.begin(), v.end());
  const double steady = ms[0][ms[0].size() / 2];
  if (want_prep) *prep_ms = std::max(0.0, double(ms[1][ms[1].size() / 2]) - steady);
  return std::max<std::int64_t>(std::int64_t(steady * 1e6 + 0.5), 1);
}

// The cost a row charges: steady-state micro-batch time plus the filter
// preparation amortised over the ceil(B / b) micro-batches a plan of size-b
// micro-batches makes. The executor prepares the filter once per run of
// same-algorithm micro-batches (kFilterReady), so a uniform plan's summed
// cost (the reference's model, cost_provider.hpp:117-127) is exactly
// prep + k * steady.
std::int64_t row_cost_ns(std::int64_t steady_ns, double prep_ms, std::int64_t b, std::int64_t full_batch) {
  if (steady_ns < 0) return -1;
  const std::int64_t micros = std::max<std::int64_t>(1, (full_batch + b - 1) / b);
  return std::max<std::int64_t>(1, steady_ns + std::int64_t(std::max(0.0, prep_ms) * 1e6 / double(micros) + 0.5));
}

// Fill missing cost rows for every algorithm x admissible micro-batch of a
// kernel; times are exact decimals of integer nanoseconds.
// With ucudnnSetBenchmarkDevices the feasible (algorithm, micro-batch) jobs
// are spread over one host thread per listed device (an atomic job index:
// PAPER.md:472-473's parallel evaluation); rows are merged into the table
// after every thread is done, so the table never sees a partial kernel.
void benchmark_kernel(ucudnnContext* h, const Kernel& k, Policy policy) {
  ModeScope mode(h->deterministic, h->faithful);
  const ConvShape full = shape_of(k);
  struct Job {
    CostKey key;
    ConvShape s;
    std::int64_t ws;
    std::int64_t ns = 0;
  };
  std::vector<Job> jobs;
  for (std::int64_t b : micro_sizes(policy, k.batch)) {
    for (int algo = 0; algo < algo_count(); ++algo) {
      CostKey key{k.hash(), k.op, algo, b};
      if (h->table->get(key)) continue;
      ConvShape s = full;
      s.N = int(b);
      bool ok = false;
      std::int64_t ws = algo_ws(int(k.op), s, algo, &ok);
      if (ok) jobs.push_back(Job{key, s, ws});
      else h->table->put(CostRecord{key, Ratio(0), 0, false});
    }
  }
  if (jobs.empty()) return;
  const int op = int(k.op);
  // filter preparation is batch-independent: measured once per algorithm,
  // at its first (smallest) micro-batch, on the handle's own device
  std::vector<double> prep(std::size_t(algo_count()), -1.0);
  std::vector<char> done(jobs.size(), 0);
  {
    ModeScope det(h->deterministic, h->faithful);
    for (std::size_t i = 0; i < jobs.size(); ++i) {
      Job& j = jobs[i];
      if (prep[std::size_t(j.key.alg)] >= 0) continue;
      j.ns = time_once(&h->primary, h->stream, h->warmup, h->iters, op, j.s, j.key.alg, j.ws,
                       &prep[std::size_t(j.key.alg)]);
      if (j.ns < 0) prep[std::size_t(j.key.alg)] = -1.0;  // try the next size
      else done[i] = 1;
    }
  }
  if (h->slots.empty()) {
    ModeScope det(h->deterministic, h->faithful);
    // Dominance pruning (UCUDNN_BENCH_PRUNE=0 disables): one probe run per
    // row first; a row at least 25 % slower than another row of the same
    // micro-batch size that needs no more workspace can never be chosen --
    // not by the WR DP (fastest feasible per size) nor on a WD Pareto front --
    // so its probe time is recorded and only the others get the full median
    // of `iters` (AlexNet `all` planning: most (algorithm, size) rows).
    static const bool prune = [] {
      const char* e = std::getenv("UCUDNN_BENCH_PRUNE");
      return !e || std::atoi(e) != 0;
    }();
    std::vector<std::int64_t> probe(jobs.size(), -1);
    if (prune && h->iters > 1)
      for (std::size_t i = 0; i < jobs.size(); ++i)
        if (!done[i]) probe[i] = time_once(&h->primary, h->stream, h->warmup, 1, op, jobs[i].s, jobs[i].key.alg,
                                           jobs[i].ws);
    for (std::size_t i = 0; i < jobs.size(); ++i) {
      if (done[i]) continue;
      // compared as the rows' costs: steady time plus the amortised filter preparation
      auto cost = [&](std::size_t q, std::int64_t t) {
        return row_cost_ns(t, prep[std::size_t(jobs[q].key.alg)], jobs[q].key.batch, k.batch);
      };
      bool dominated = false;
      if (probe[i] > 0) {
        const std::int64_t ci = cost(i, probe[i]);
        for (std::size_t j = 0; j < jobs.size() && !dominated; ++j) {
          const std::int64_t tj = done[j] ? jobs[j].ns : probe[j];
          dominated = j != i && jobs[j].key.batch == jobs[i].key.batch && tj > 0 && cost(j, tj) * 5 < ci * 4 &&
                      jobs[j].ws <= jobs[i].ws;
        }
      }
      jobs[i].ns = dominated ? probe[i]
                             : time_once(&h->primary, h->stream, probe[i] > 0 ? 1 : h->warmup, h->iters, op,
                                         jobs[i].s, jobs[i].key.alg, jobs[i].ws);
    }
  } else {
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex err_mu;
    std::vector<std::thread> workers;
    for (auto& slot : h->slots) {
      BenchSlot* sl = slot.get();
      workers.emplace_back([&, sl] {
        try {
          ModeScope det(h->deterministic, h->faithful);
          cuda_check(cudaSetDevice(sl->device), "cudaSetDevice(benchmark device)");
          if (!sl->stream) cuda_check(cudaStreamCreateWithFlags(&sl->stream, cudaStreamNonBlocking), "cudaStreamCreate");
          for (std::size_t i = next++; i < jobs.size(); i = next++) {
            {
              std::lock_guard<std::mutex> lock(err_mu);
              if (err) return;
            }
            if (done[i]) continue;
            Job& j = jobs[i];
            j.ns = time_once(sl, sl->stream, h->warmup, h->iters, op, j.s, j.key.alg, j.ws);
          }
        } catch (...) {
          std::lock_guard<std::mutex> lock(err_mu);
          if (!err) err = std::current_exception();
        }
      });
    }
    for (auto& t : workers) t.join();
    if (err) std::rethrow_exception(err);
  }
  for (Job& j : jobs) {
    j.ns = row_cost_ns(j.ns, prep[std::size_t(j.key.alg)], j.key.batch, k.batch);
    h->table->put(j.ns < 0 ? CostRecord{j.key, Ratio(0), 0, false} : CostRecord{j.key, Ratio(j.ns, 1000), j.ws, true});
  }
}

ucudnnContext::Entry& entry_of(ucudnnContext* h, int algo) {
  int idx = algo - UCUDNN_VIRTUAL_ALGO_BASE;
  require(idx >= 0 && idx < int(h->entries.size()), "unknown virtual algorithm id");
  return h->entries[std::size_t(idx)];
}

int register_kernel(ucudnnContext* h, const Kernel& k, std::int64_t limit) {
  ucudnnContext::Entry e;
  e.kernel = k;
  e.limit = limit;
  h->entries.push_back(e);
  h->wd_stale = true;
  return UCUDNN_VIRTUAL_ALGO_BASE + int(h->entries.size() - 1);
}

void plan_wr(ucudnnContext* h, ucudnnContext::Entry& e) {
  benchmark_kernel(h, e.kernel, h->policy);
  CostSource src = CostSource::table_only(h->table.get());
  e.plan = wr_plan(src, e.kernel, e.kernel.batch, e.limit, h->policy).plan;
  e.planned = true;
}

void plan_wd(ucudnnContext* h) {
  require(!h->entries.empty(), "no kernels registered");
  std::vector<Kernel> ks;
  for (auto& e : h->entries) {
    benchmark_kernel(h, e.kernel, h->policy);
    ks.push_back(e.kernel);
  }
  CostSource src = CostSource::table_only(h->table.get());
  WdPlan wd = wd_plan(src, ks, h->total_ws, h->policy, 1);
  std::size_t off = 0;
  for (std::size_t i = 0; i < ks.size(); ++i) {
    auto& e = h->entries[i];
    e.plan = wd.chosen[i];
    e.planned = true;
    e.arena_offset = off;
    off += (std::size_t(e.plan.ws()) + 255) / 256 * 256;
  }
  h->wd_frozen = true;
  // the arena only grows (a re-plan that needs no more keeps its pointer, so
  // CUDA graphs captured over it stay valid); growing it after capture is
  // unsupported, as re-registering kernels after capture is
  if (off > h->arena_bytes) {
    if (h->arena) cudaFree(h->arena);
    h->arena = nullptr;
    h->arena_bytes = 0;
    if (off) cuda_check(cudaMalloc(&h->arena, off), "cudaMalloc(WD arena)");
    h->arena_bytes = off;
  }
  h->wd_stale = false;
}

// Runs `plan` micro-batch by micro-batch in canonical order on the handle's
// stream (reference execute_plan, reference_conv.hpp:205-278). F/BD: each
// slice gets alpha/beta; BF: user beta on the first micro-batch, then 1.
void execute(ucudnnContext* h, int op, const ConvShape& full, const Plan& plan, const float* a, const float* b,
             float* out, void* ws, std::size_t ws_bytes, float alpha, float beta) {
  require(plan.covered() == full.N, "plan does not cover the batch");
  require(std::size_t(plan.ws()) <= ws_bytes || plan.ws() == 0, "workspace smaller than the plan requires");
  const std::int64_t x_ss = std::int64_t(full.C) * full.H * full.W;
  const std::int64_t y_ss = std::int64_t(full.K) * full.OH() * full.OW();
  std::int64_t off = 0;
  const std::vector<Micro>& ms = plan.micros();
  float run_beta = beta;  // BF: beta of the current same-algorithm run (user beta if it starts the call)
  for (std::size_t i = 0; i < ms.size(); ++i) {
    const Micro& m = ms[i];
    const AlgoImpl* impl = find_algo(m.alg);
    require(impl != nullptr, "plan uses an algorithm this build does not provide");
    ConvShape s = full;
    s.N = int(m.batch);
    // the plan's workspace came from a cost table, which may predate this
    // build's kernels: never run a micro-batch on less than it really needs
    require(algo_workspace(impl, op, s) <= std::int64_t(ws_bytes) || (algo_workspace(impl, op, s) == 0),
            "micro-batch needs more workspace than its cost-table row says (stale cost table?)");
    cudaError_t e;
    const bool same_prev = i > 0 && ms[i - 1].alg == m.alg, same_next = i + 1 < ms.size() && ms[i + 1].alg == m.alg;
    int flags = same_prev ? kFilterReady : 0;
    if (op == 0) e = algo_run(impl, 0, s, a + off * x_ss, b, out + off * y_ss, ws, alpha, beta, h->stream, flags);
    else if (op == 1) e = algo_run(impl, 1, s, a + off * y_ss, b, out + off * x_ss, ws, alpha, beta, h->stream, flags);
    else {
      // user beta on the first micro-batch, 1 afterwards (the reference's
      // accumulate-into, reference_conv.hpp:257-274); an algorithm that
      // defers its finalize over a run applies the run's starting beta once
      float b_m = i == 0 ? beta : 1.f;
      if ((impl->defer_ops & (1 << 2)) && !faithful()) {
        if (!same_prev) run_beta = b_m;
        b_m = run_beta;
        if (same_prev) flags |= kAccumulate;
        if (same_next) flags |= kDeferFinal;
      }
      e = algo_run(impl, 2, s, a + off * x_ss, b + off * y_ss, out, ws, alpha, b_m, h->stream, flags);
    }
    cuda_check(e, "kernel launch");
    off += m.batch;
  }
}

Plan undivided(int algo, const ConvShape& s, int op) {
  bool ok = false;
  std::int64_t ws = algo_ws(op, s, algo, &ok);
  require(ok, "algorithm does not support this convolution");
  return Plan::one(Micro{algo, s.N, Ratio(0), ws});
}

ucudnnStatus_t run_conv(ucudnnContext* h, int op, const ConvShape& s, int algo, const float* a, const float* b,
                        float* out, void* ws, std::size_t ws_bytes, float alpha, float beta) {
  ModeScope det(h->deterministic, h->faithful);
  if (algo >= UCUDNN_VIRTUAL_ALGO_BASE) {
    auto& e = entry_of(h, algo);
    require(int(e.kernel.op) == op, "virtual algorithm belongs to another operation");
    require(shape_of(e.kernel).N == s.N && e.kernel.same_shape(kernel_from(Op(op), s, e.kernel.name)),
            "descriptors differ from the registered kernel");
    if (h->mode == Mode::WD) {
      if (h->wd_stale || !e.planned) plan_wd(h);
      execute(h, op, s, e.plan, a, b, out, static_cast<char*>(h->arena) + e.arena_offset,
              std::size_t(e.plan.ws()), alpha, beta);
    } else {
      if (!e.planned) plan_wr(h, e);
      execute(h, op, s, e.plan, a, b, out, ws, ws_bytes, alpha, beta);
    }
  } else {
    execute(h, op, s, undivided(algo, s, op), a, b, out, ws, ws_bytes, alpha, beta);
  }
  return UCUDNN_STATUS_SUCCESS;
}

Policy env_policy(Policy d) {
  if (const char* v = std::getenv("UCUDNN_BATCH_SIZE_POLICY")) {
    Policy p;
    if (parse_policy(v, &p)) return p;
  }
  return d;
}

ucudnnStatus_t copy_out(const std::string& s, char* out, std::size_t* len) {
  require(len != nullptr, "null length");
  std::size_t need = s.size() + 1;
  if (!out || *len < need) {
    *len = need;
    if (!out) return UCUDNN_STATUS_SUCCESS;
    throw std::invalid_argument("output buffer too small");
  }
  std::memcpy(out, s.c_str(), need);
  *len = need;
  return UCUDNN_STATUS_SUCCESS;
}

bool csv_file(const std::string& path) {
  std::ifstream in(path);
  std::string first;
  if (!in || !std::getline(in, first)) return false;
  if (!first.empty() && first.back() == '\r') first.pop_back();
  return first == kCsvHeader;
}

}  // namespace

extern "C" {

const char* ucudnnGetErrorString(ucudnnStatus_t s) {
  switch (s) {
    case UCUDNN_STATUS_SUCCESS: return "UCUDNN_STATUS_SUCCESS";
    case UCUDNN_STATUS_NOT_INITIALIZED: return "UCUDNN_STATUS_NOT_INITIALIZED";
    case UCUDNN_STATUS_ALLOC_FAILED: return "UCUDNN_STATUS_ALLOC_FAILED";
    case UCUDNN_STATUS_BAD_PARAM: return "UCUDNN_STATUS_BAD_PARAM";
    case UCUDNN_STATUS_INTERNAL_ERROR: return "UCUDNN_STATUS_INTERNAL_ERROR";
    case UCUDNN_STATUS_INVALID_VALUE: return "UCUDNN_STATUS_INVALID_VALUE";
    case UCUDNN_STATUS_ARCH_MISMATCH: return "UCUDNN_STATUS_ARCH_MISMATCH";
    case UCUDNN_STATUS_EXECUTION_FAILED: return "UCUDNN_STATUS_EXECUTION_FAILED";
    case UCUDNN_STATUS_NOT_SUPPORTED: return "UCUDNN_STATUS_NOT_SUPPORTED";
  }
  return "UCUDNN_STATUS_UNKNOWN";
}
const char* ucudnnGetLastError(void) { return g_last_error.c_str(); }
int64_t ucudnnGetMinTotalWorkspace(void) { return g_min_ws; }
size_t ucudnnGetVersion(void) { return UCUDNN_VERSION; }
uint64_t ucudnnGetLaunchCount(void) { return launch_count(); }

ucudnnStatus_t ucudnnDebugPrecompProfile(double* out4) {
  if (!out4) return UCUDNN_STATUS_BAD_PARAM;
  precomp_profile(out4);
  return UCUDNN_STATUS_SUCCESS;
}

ucudnnStatus_t ucudnnDebugBackwardFilterProfile(double* out4) {
  if (!out4) return UCUDNN_STATUS_BAD_PARAM;
  bf_profile(out4);
  return UCUDNN_STATUS_SUCCESS;
}

ucudnnStatus_t ucudnnDebugSetTrace(int on) {
  set_trace(on != 0);
  return UCUDNN_STATUS_SUCCESS;
}

ucudnnStatus_t ucudnnDebugGetTrace(char* buf, size_t* len) {
  return guarded([&] { return copy_out(take_trace(), buf, len); });
}

ucudnnStatus_t ucudnnCreate(UcudnnHandle_t* out) {
  return guarded([&] {
    require(out != nullptr, "null handle pointer");
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp prop;
    cuda_check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (prop.major != 10) {
      g_last_error = "this library is built for sm_100a (B200) only";
      return UCUDNN_STATUS_ARCH_MISMATCH;
    }
    auto* h = new ucudnnContext();
    h->device = dev;
    h->policy = env_policy(Policy::PowerOfTwo);
    if (const char* v = std::getenv("UCUDNN_WORKSPACE_MODE")) h->mode = std::string(v) == "wd" ? Mode::WD : Mode::WR;
    if (const char* v = std::getenv("UCUDNN_TOTAL_WORKSPACE_SIZE")) h->total_ws = std::atoll(v);
    if (const char* v = std::getenv("UCUDNN_BENCHMARK_ITERS")) h->iters = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("UCUDNN_DETERMINISTIC")) h->deterministic = std::atoi(v) != 0;
    if (const char* v = std::getenv("UCUDNN_MATH_MODE")) h->faithful = std::string(v) == "fp32";
    if (const char* v = std::getenv("UCUDNN_DATABASE")) {
      h->db_path = v;
      h->table = CostTable::open(v);
    }
    *out = h;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnDestroy(UcudnnHandle_t h) {
  return guarded([&] {
    delete h;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnSetStream(UcudnnHandle_t h, void* s) {
  return guarded([&] {
    require(h, "null handle");
    h->stream = static_cast<cudaStream_t>(s);
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnGetStream(UcudnnHandle_t h, void** s) {
  return guarded([&] {
    require(h && s, "null argument");
    *s = h->stream;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnSetBatchSizePolicy(UcudnnHandle_t h, ucudnnBatchSizePolicy_t p) {
  return guarded([&] {
    require(h && p >= 0 && p <= 2, "bad policy");
    h->policy = Policy(int(p));
    for (auto& e : h->entries) e.planned = false;
    h->wd_stale = true;
    h->wd_frozen = false;
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetWorkspaceMode(UcudnnHandle_t h, ucudnnWorkspaceMode_t m) {
  return guarded([&] {
    require(h && (m == 0 || m == 1), "bad workspace mode");
    h->mode = Mode(int(m));
    for (auto& e : h->entries) e.planned = false;
    h->wd_stale = true;
    h->wd_frozen = false;
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetTotalWorkspaceLimit(UcudnnHandle_t h, int64_t bytes) {
  return guarded([&] {
    require(h && bytes >= 0, "bad workspace limit");
    h->total_ws = bytes;
    h->wd_stale = true;
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetCostDatabase(UcudnnHandle_t h, const char* path) {
  return guarded([&] {
    require(h && path, "null argument");
    auto t = CostTable::open(path);
    for (const CostRecord& r : h->table->records())
      if (!t->get(r.key)) t->put(r);
    h->table = std::move(t);
    h->db_path = path;
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnFlushCostDatabase(UcudnnHandle_t h) {
  return guarded([&] {
    require(h, "null handle");
    require(!h->db_path.empty(), "no cost database path set");
    h->table->flush_to(h->db_path);
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetBenchmarkDevices(UcudnnHandle_t h, const int* device_ids, int n) {
  return guarded([&] {
    require(h && n >= 0 && (n == 0 || device_ids), "bad benchmark device list");
    std::vector<int> ids(device_ids, device_ids + n);
    if (n > 0) {
      int count = 0;
      cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
      for (int d : ids) require(d >= 0 && d < count, "benchmark device id out of range");
    }
    h->release_slots();
    for (int d : ids) {
      auto sl = std::make_unique<BenchSlot>();
      sl->device = d;
      h->slots.push_back(std::move(sl));
    }
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnSetDeterministic(UcudnnHandle_t h, int on) {
  return guarded([&] {
    require(h, "null handle");
    if (h->deterministic != (on != 0)) {
      // the cost rows and plans so far were timed in the other mode: start
      // from an empty table (a database file must be set again, per mode)
      h->deterministic = on != 0;
      h->table = std::make_unique<CostTable>();
      h->db_path.clear();
      for (auto& e : h->entries) e.planned = false;
      h->wd_stale = true;
    }
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnSetMathMode(UcudnnHandle_t h, ucudnnMathMode_t mode) {
  return guarded([&] {
    require(h && (mode == UCUDNN_MATH_TF32 || mode == UCUDNN_MATH_FP32_FAITHFUL), "bad math mode");
    const bool f = mode == UCUDNN_MATH_FP32_FAITHFUL;
    if (h->faithful != f) {
      h->faithful = f;
      h->table = std::make_unique<CostTable>();  // rows of the other mode: not reusable
      h->db_path.clear();
      for (auto& e : h->entries) e.planned = false;
      h->wd_stale = true;
    }
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnSetBenchmarkIterations(UcudnnHandle_t h, int warmup, int iters) {
  return guarded([&] {
    require(h && warmup >= 0 && iters >= 1, "bad iteration counts");
    h->warmup = warmup;
    h->iters = iters;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnCreateTensorDescriptor(ucudnnTensorDescriptor_t* d) {
  return guarded([&] {
    require(d, "null");
    *d = new ucudnnTensorStruct();
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetTensor4dDescriptor(ucudnnTensorDescriptor_t d, int n, int c, int h, int w) {
  return guarded([&] {
    require(d && n > 0 && c > 0 && h > 0 && w > 0, "tensor dims must be >= 1");
    *d = ucudnnTensorStruct{n, c, h, w};
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnGetTensor4dDescriptor(ucudnnTensorDescriptor_t d, int* n, int* c, int* h, int* w) {
  return guarded([&] {
    require(d && n && c && h && w, "null");
    *n = d->n; *c = d->c; *h = d->h; *w = d->w;
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnDestroyTensorDescriptor(ucudnnTensorDescriptor_t d) {
  delete d;
  return UCUDNN_STATUS_SUCCESS;
}
ucudnnStatus_t ucudnnCreateFilterDescriptor(ucudnnFilterDescriptor_t* d) {
  return guarded([&] {
    require(d, "null");
    *d = new ucudnnFilterStruct();
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetFilter4dDescriptor(ucudnnFilterDescriptor_t d, int k, int c, int r, int s) {
  return guarded([&] {
    require(d && k > 0 && c > 0 && r > 0 && s > 0, "filter dims must be >= 1");
    *d = ucudnnFilterStruct{k, c, r, s};
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnDestroyFilterDescriptor(ucudnnFilterDescriptor_t d) {
  delete d;
  return UCUDNN_STATUS_SUCCESS;
}
ucudnnStatus_t ucudnnCreateConvolutionDescriptor(ucudnnConvolutionDescriptor_t* d) {
  return guarded([&] {
    require(d, "null");
    *d = new ucudnnConvolutionStruct();
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnSetConvolution2dDescriptor(ucudnnConvolutionDescriptor_t d, int ph, int pw, int sh, int sw,
                                                int dh, int dw) {
  return guarded([&] {
    require(d && ph >= 0 && pw >= 0 && sh >= 1 && sw >= 1, "bad convolution parameters");
    if (dh != 1 || dw != 1) {
      g_last_error = "dilation != 1 is not supported";
      return UCUDNN_STATUS_NOT_SUPPORTED;
    }
    *d = ucudnnConvolutionStruct{ph, pw, sh, sw};
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnGetConvolution2dForwardOutputDim(ucudnnConvolutionDescriptor_t c, ucudnnTensorDescriptor_t x,
                                                      ucudnnFilterDescriptor_t w, int* n, int* k, int* oh, int* ow) {
  return guarded([&] {
    ConvShape s = conv_shape(x, w, c);
    require(n && k && oh && ow, "null");
    *n = s.N; *k = s.K; *oh = s.OH(); *ow = s.OW();
    return UCUDNN_STATUS_SUCCESS;
  });
}
ucudnnStatus_t ucudnnDestroyConvolutionDescriptor(ucudnnConvolutionDescriptor_t d) {
  delete d;
  return UCUDNN_STATUS_SUCCESS;
}

static ucudnnStatus_t get_algo(UcudnnHandle_t h, Op op, const ConvShape& s, int64_t limit, int* algo) {
  return guarded([&] {
    require(h && algo, "null argument");
    require(limit >= 0, "workspace limit must be >= 0");
    static int counter = 0;
    Kernel k = kernel_from(op, s, "layer" + std::to_string(counter));
    // WR: a repeated query for the same shape + limit reuses its plan. WD
    // registers every call as its own kernel (replicated layers are selected
    // independently, wd_optimizer.hpp:628-634).
    for (std::size_t i = 0; h->mode == Mode::WD && h->wd_frozen && i < h->entries.size(); ++i)
      if (h->entries[i].kernel.same_shape(k)) {
        *algo = UCUDNN_VIRTUAL_ALGO_BASE + int(i);
        return UCUDNN_STATUS_SUCCESS;
      }
    for (std::size_t i = 0; h->mode == Mode::WR && i < h->entries.size(); ++i)
      if (h->entries[i].kernel.same_shape(k) && h->entries[i].limit == limit) {
        *algo = UCUDNN_VIRTUAL_ALGO_BASE + int(i);
        if (h->mode == Mode::WR && !h->entries[i].planned) plan_wr(h, h->entries[i]);
        return UCUDNN_STATUS_SUCCESS;
      }
    ++counter;
    int id = register_kernel(h, k, limit);
    if (h->mode == Mode::WR) {
      h->report_limit = limit;
      plan_wr(h, entry_of(h, id));
    }
    *algo = id;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnGetConvolutionForwardAlgorithm(UcudnnHandle_t h, ucudnnTensorDescriptor_t x,
                                                    ucudnnFilterDescriptor_t w, ucudnnConvolutionDescriptor_t c,
                                                    ucudnnTensorDescriptor_t, int64_t limit, int* algo) {
  ConvShape s;
  ucudnnStatus_t st = guarded([&] { s = conv_shape(x, w, c); return UCUDNN_STATUS_SUCCESS; });
  return st != UCUDNN_STATUS_SUCCESS ? st : get_algo(h, Op::Forward, s, limit, algo);
}
ucudnnStatus_t ucudnnGetConvolutionBackwardDataAlgorithm(UcudnnHandle_t h, ucudnnFilterDescriptor_t w,
                                                         ucudnnTensorDescriptor_t, ucudnnConvolutionDescriptor_t c,
                                                         ucudnnTensorDescriptor_t dx, int64_t limit, int* algo) {
  ConvShape s;
  ucudnnStatus_t st = guarded([&] { s = conv_shape(dx, w, c); return UCUDNN_STATUS_SUCCESS; });
  return st != UCUDNN_STATUS_SUCCESS ? st : get_algo(h, Op::BackwardData, s, limit, algo);
}
ucudnnStatus_t ucudnnGetConvolutionBackwardFilterAlgorithm(UcudnnHandle_t h, ucudnnTensorDescriptor_t x,
                                                           ucudnnTensorDescriptor_t, ucudnnConvolutionDescriptor_t c,
                                                           ucudnnFilterDescriptor_t dw, int64_t limit, int* algo) {
  ConvShape s;
  ucudnnStatus_t st = guarded([&] { s = conv_shape(x, dw, c); return UCUDNN_STATUS_SUCCESS; });
  return st != UCUDNN_STATUS_SUCCESS ? st : get_algo(h, Op::BackwardFilter, s, limit, algo);
}

ucudnnStatus_t ucudnnGetConvolutionWorkspaceSize(UcudnnHandle_t h, int algo, ucudnnOp_t op,
                                                 ucudnnTensorDescriptor_t x, ucudnnFilterDescriptor_t w,
                                                 ucudnnConvolutionDescriptor_t c, size_t* bytes) {
  return guarded([&] {
    require(h && bytes, "null argument");
    if (algo >= UCUDNN_VIRTUAL_ALGO_BASE) {
      auto& e = entry_of(h, algo);
      if (h->mode == Mode::WD) {
        *bytes = 0;
      } else {
        if (!e.planned) plan_wr(h, e);
        *bytes = std::size_t(e.plan.ws());
      }
    } else {
      ModeScope mode(h->deterministic, h->faithful);
      ConvShape s = conv_shape(x, w, c);
      bool ok = false;
      std::int64_t ws = algo_ws(int(op), s, algo, &ok);
      require(ok, "algorithm does not support this convolution");
      *bytes = std::size_t(ws);
    }
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnOptimizeNetwork(UcudnnHandle_t h) {
  return guarded([&] {
    require(h, "null handle");
    if (h->mode == Mode::WD) plan_wd(h);
    else
      for (auto& e : h->entries)
        if (!e.planned) plan_wr(h, e);
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnGetPlan(UcudnnHandle_t h, int algo, int* n_micro, int* algs, int64_t* batches, int cap) {
  return guarded([&] {
    require(h && n_micro, "null argument");
    auto& e = entry_of(h, algo);
    if (!e.planned) {
      if (h->mode == Mode::WD) plan_wd(h);
      else plan_wr(h, e);
    }
    const auto& ms = e.plan.micros();
    *n_micro = int(ms.size());
    for (int i = 0; i < int(ms.size()) && i < cap; ++i) {
      if (algs) algs[i] = ms[std::size_t(i)].alg;
      if (batches) batches[i] = ms[std::size_t(i)].batch;
    }
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnGetMachineReport(UcudnnHandle_t h, char* buf, size_t* len) {
  return guarded([&] {
    require(h, "null handle");
    require(!h->entries.empty(), "no kernels registered");
    std::vector<Kernel> ks;
    for (auto& e : h->entries) {
      benchmark_kernel(h, e.kernel, h->policy);
      ks.push_back(e.kernel);
    }
    CostSource src = CostSource::table_only(h->table.get());
    RunConfig cfg;
    cfg.mode = h->mode;
    cfg.policy = h->policy;
    cfg.limit = h->mode == Mode::WD ? h->total_ws : h->report_limit;
    Report r = plan_network(src, "handle", ks, cfg);
    return copy_out(machine_report(r), buf, len);
  });
}

ucudnnStatus_t ucudnnConvolutionForward(UcudnnHandle_t h, const void* alpha, ucudnnTensorDescriptor_t xd,
                                        const void* x, ucudnnFilterDescriptor_t wd, const void* w,
                                        ucudnnConvolutionDescriptor_t c, int algo, void* ws, size_t ws_bytes,
                                        const void* beta, ucudnnTensorDescriptor_t, void* y) {
  return guarded([&] {
    require(h && alpha && beta && x && w && y, "null argument");
    ConvShape s = conv_shape(xd, wd, c);
    return run_conv(h, 0, s, algo, static_cast<const float*>(x), static_cast<const float*>(w),
                    static_cast<float*>(y), ws, ws_bytes, *static_cast<const float*>(alpha),
                    *static_cast<const float*>(beta));
  });
}
ucudnnStatus_t ucudnnConvolutionBackwardData(UcudnnHandle_t h, const void* alpha, ucudnnFilterDescriptor_t wd,
                                             const void* w, ucudnnTensorDescriptor_t, const void* dy,
                                             ucudnnConvolutionDescriptor_t c, int algo, void* ws, size_t ws_bytes,
                                             const void* beta, ucudnnTensorDescriptor_t dxd, void* dx) {
  return guarded([&] {
    require(h && alpha && beta && w && dy && dx, "null argument");
    ConvShape s = conv_shape(dxd, wd, c);
    return run_conv(h, 1, s, algo, static_cast<const float*>(dy), static_cast<const float*>(w),
                    static_cast<float*>(dx), ws, ws_bytes, *static_cast<const float*>(alpha),
                    *static_cast<const float*>(beta));
  });
}
ucudnnStatus_t ucudnnConvolutionBackwardFilter(UcudnnHandle_t h, const void* alpha, ucudnnTensorDescriptor_t xd,
                                               const void* x, ucudnnTensorDescriptor_t, const void* dy,
                                               ucudnnConvolutionDescriptor_t c, int algo, void* ws, size_t ws_bytes,
                                               const void* beta, ucudnnFilterDescriptor_t dwd, void* dw) {
  return guarded([&] {
    require(h && alpha && beta && x && dy && dw, "null argument");
    ConvShape s = conv_shape(xd, dwd, c);
    return run_conv(h, 2, s, algo, static_cast<const float*>(x), static_cast<const float*>(dy),
                    static_cast<float*>(dw), ws, ws_bytes, *static_cast<const float*>(alpha),
                    *static_cast<const float*>(beta));
  });
}

ucudnnStatus_t ucudnnTimeAlgorithm(UcudnnHandle_t h, ucudnnOp_t op, const int64_t* shape11, int algo,
                                   int64_t micro_batch, double* time_us, int64_t* ws_bytes, int* feasible) {
  return guarded([&] {
    require(h && shape11 && time_us && ws_bytes && feasible, "null argument");
    require(op >= 0 && op <= 2, "bad op");
    ConvShape s = shape_from11(shape11);
    s.N = int(micro_batch);
    ModeScope mode(h->deterministic, h->faithful);
    bool ok = false;
    std::int64_t ws = algo_ws(int(op), s, algo, &ok);
    *feasible = ok ? 1 : 0;
    *ws_bytes = ws;
    // a single timing charges the filter preparation in full (one micro-batch)
    double prep = -1.0;
    const std::int64_t ns =
        ok ? row_cost_ns(time_once(&h->primary, h->stream, h->warmup, h->iters, int(op), s, algo, ws, &prep), prep, 1, 1)
           : 0;
    if (ns < 0) *feasible = 0;
    *time_us = ns > 0 ? double(ns) / 1000.0 : 0.0;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnBenchmarkKernel(UcudnnHandle_t h, ucudnnOp_t op, const int64_t* shape11,
                                     ucudnnBatchSizePolicy_t policy) {
  return guarded([&] {
    require(h && shape11, "null argument");
    require(op >= 0 && op <= 2 && policy >= 0 && policy <= 2, "bad op or policy");
    benchmark_kernel(h, kernel_from(Op(int(op)), shape_from11(shape11), "bench"), Policy(int(policy)));
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnAlgorithmWorkspace(ucudnnOp_t op, const int64_t* shape11, int algo, int64_t micro_batch,
                                        int64_t* ws_bytes, int* feasible) {
  return guarded([&] {
    require(shape11 && ws_bytes && feasible, "null argument");
    ConvShape s = shape_from11(shape11);
    s.N = int(micro_batch);
    bool ok = false;
    *ws_bytes = algo_ws(int(op), s, algo, &ok);
    *feasible = ok;
    return UCUDNN_STATUS_SUCCESS;
  });
}

ucudnnStatus_t ucudnnPlanNetworkFile(const char* network_path, int64_t batch_override, const char* cost_path,
                                     const char* cache_csv, int mode, int policy, int64_t limit, unsigned jobs,
                                     int report_kind, char* out, size_t* len) {
  return guarded([&] {
    require(network_path != nullptr, "null network path");
    require(mode == 0 || mode == 1, "mode must be 0 (wr) or 1 (wd)");
    require(policy >= 0 && policy <= 2, "bad policy");
    require(limit >= 0, "workspace limit must be >= 0");
    Network net = load_network(network_path);
    std::vector<Kernel> ks = expand(net, batch_override);
    std::string cost = cost_path ? cost_path : "";
    std::unique_ptr<CostTable> meas, cache;
    std::optional<CostSource> src;
    if (!cost.empty() && cost != "builtin" && csv_file(cost)) {
      meas = CostTable::load(cost);
      src = CostSource::table_only(meas.get());
    } else {
      CostModel model = (cost.empty() || cost == "builtin") ? CostModel::builtin() : CostModel::load(cost);
      if (cache_csv && *cache_csv) cache = CostTable::open(cache_csv);
      src.emplace(std::move(model), cache.get());
    }
    RunConfig cfg;
    cfg.mode = Mode(mode);
    cfg.policy = Policy(policy);
    cfg.limit = limit;
    cfg.jobs = jobs == 0 ? 1 : jobs;
    Report r = plan_network(*src, net.name, ks, cfg);
    if (cache) cache->flush_to(cache->path());
    return copy_out(report_kind == 1 ? text_report(r) : machine_report(r), out, len);
  });
}

ucudnnStatus_t ucudnnPlanKernels(const char* network_name, const int64_t* k12, const char* const* names,
                                 int n_kernels, const char* csv_text, int mode, int policy, int64_t limit,
                                 unsigned jobs, char* out, size_t* len) {
  return guarded([&] {
    require(k12 && csv_text && n_kernels > 0, "null argument");
    require(mode == 0 || mode == 1, "mode must be 0 (wr) or 1 (wd)");
    require(policy >= 0 && policy <= 2, "bad policy");
    std::vector<Kernel> ks;
    for (int i = 0; i < n_kernels; ++i) {
      const int64_t* r = k12 + 12 * i;
      Kernel k;
      require(r[0] >= 0 && r[0] <= 2, "bad op");
      k.op = Op(r[0]); k.batch = r[1]; k.c = r[2]; k.h = r[3]; k.w = r[4]; k.k = r[5]; k.r = r[6]; k.s = r[7];
      k.pad_h = r[8]; k.pad_w = r[9]; k.stride_h = r[10]; k.stride_w = r[11];
      k.name = names && names[i] ? names[i] : "k" + std::to_string(i);
      k.check();
      ks.push_back(k);
    }
    auto table = CostTable::from_csv_text(csv_text, "cost-table");
    CostSource src = CostSource::table_only(table.get());
    RunConfig cfg;
    cfg.mode = Mode(mode);
    cfg.policy = Policy(policy);
    cfg.limit = limit;
    cfg.jobs = jobs == 0 ? 1 : jobs;
    Report r = plan_network(src, network_name ? network_name : "net", ks, cfg);
    return copy_out(machine_report(r), out, len);
  });
}

ucudnnStatus_t ucudnnCanonicalTime(const char* text, char* out, size_t* len) {
  return guarded([&] {
    require(text != nullptr, "null text");
    return copy_out(Ratio::parse(text).str(), out, len);
  });
}

ucudnnStatus_t ucudnnCanonicalCostTable(const char* csv_text, char* out, size_t* len) {
  return guarded([&] {
    require(csv_text != nullptr, "null text");
    return copy_out(CostTable::from_csv_text(csv_text, "cost-table")->to_csv(), out, len);
  });
}

uint64_t ucudnnKernelHash(const int64_t* r) {
  Kernel k;
  k.op = Op(r[0]); k.batch = r[1]; k.c = r[2]; k.h = r[3]; k.w = r[4]; k.k = r[5]; k.r = r[6]; k.s = r[7];
  k.pad_h = r[8]; k.pad_w = r[9]; k.stride_h = r[10]; k.stride_w = r[11];
  return k.hash();
}

}  // extern "C"
