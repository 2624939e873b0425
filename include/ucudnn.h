/*
 * ucudnn.h -- C ABI of the B200-native micro-batched convolution library.
 *
 * The drop-in boundary for the micro-batched convolution path (SURVEY.md
 * section 8(b)). The reference `ubatch` (/root/reference/proj) has no C ABI:
 * its seams are C++ calls, and the paper's UcudnnHandle_t wrapper
 * is described but not implemented. Each
 * entry point below names the reference interface (file:line) or paper
 * section it replaces. Plain C types only; no exception crosses this ABI --
 * every failure maps to a status code plus a per-thread message
 * (ucudnnGetLastError).
 *
 * Layout: tensors NCHW fp32, fully packed (no strided descriptors), filters
 * KCRS fp32, cross-correlation, dilation 1 -- the reference convolution's
 * semantics (reference_conv.hpp:26-55, 67-171).
 */
#ifndef UCUDNN_H_
#define UCUDNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCUDNN_VERSION 100

/* Status codes mirror cuDNN 7's numbering. Reference error mapping
 * (tools/main.cpp:420-442): invalid argument / parse error -> BAD_PARAM
 * (CLI exit 2); infeasible_error -> NOT_SUPPORTED (exit 3) with the minimum
 * total workspace queryable via ucudnnGetMinTotalWorkspace; logic / overflow
 * errors -> INTERNAL_ERROR (exit 4); CUDA failures -> EXECUTION_FAILED. */
typedef enum {
  UCUDNN_STATUS_SUCCESS = 0,
  UCUDNN_STATUS_NOT_INITIALIZED = 1,
  UCUDNN_STATUS_ALLOC_FAILED = 2,
  UCUDNN_STATUS_BAD_PARAM = 3,
  UCUDNN_STATUS_INTERNAL_ERROR = 4,
  UCUDNN_STATUS_INVALID_VALUE = 5,
  UCUDNN_STATUS_ARCH_MISMATCH = 6,
  UCUDNN_STATUS_EXECUTION_FAILED = 8,
  UCUDNN_STATUS_NOT_SUPPORTED = 9
} ucudnnStatus_t;

/* Micro-batch policies (reference BatchSizePolicy, cost_provider.hpp:32-36;
 * PAPER.md:465-470). */
typedef enum {
  UCUDNN_BATCH_SIZE_ALL = 0,
  UCUDNN_BATCH_SIZE_POWER_OF_TWO = 1,
  UCUDNN_BATCH_SIZE_UNDIVIDED = 2
} ucudnnBatchSizePolicy_t;

/* Workspace modes (reference OptMode, report.hpp:32-36). */
typedef enum { UCUDNN_WORKSPACE_WR = 0, UCUDNN_WORKSPACE_WD = 1 } ucudnnWorkspaceMode_t;

/* Math modes (cudnnMathType_t-style). TF32: every GEMM-class kernel reads its
 * fp32 operands as TF32 (10-bit mantissa) with fp32 accumulation -- normwise
 * error ~1e-3 on Gaussian data. FP32_FAITHFUL ("3xTF32"): each micro-batch
 * runs three TF32 passes over hi / lo operand splits, conv(a_hi, b_hi) +
 * conv(a_lo, b_hi) + conv(a_hi, b_lo), for fp32-level error (~1e-6) at ~3x
 * the tensor work and 2 x (|a| + |b|) extra workspace, which the cost table
 * and planner account for. */
typedef enum { UCUDNN_MATH_TF32 = 0, UCUDNN_MATH_FP32_FAITHFUL = 1 } ucudnnMathMode_t;

typedef enum {
  UCUDNN_OP_FORWARD = 0,
  UCUDNN_OP_BACKWARD_DATA = 1,
  UCUDNN_OP_BACKWARD_FILTER = 2
} ucudnnOp_t;

/* Concrete B200 algorithms (the cost-table `algorithm` column). Ids 0-2 keep
 * the reference archetype names of cost_model.hpp:165-177. */
typedef enum {
  UCUDNN_ALGO_IMPLICIT_GEMM = 0,     /* tcgen05 implicit GEMM, cp.async-gathered operands, 0 workspace */
  UCUDNN_ALGO_WINOGRAD = 1,          /* F(2x2,3x3) (3x3 s1 F/BD): transforms + 16 batched tcgen05 GEMMs */
  UCUDNN_ALGO_FFT = 2,               /* FFT-tiled (s1 F/BD, R,S <= 16): register FFTs + per-bin GEMMs */
  UCUDNN_ALGO_GEMM = 3,              /* explicit im2col / col2im + tiled tcgen05 GEMM                  */
  UCUDNN_ALGO_WINOGRAD_4x4 = 4,      /* F(4x4,3x3) (3x3 s1 F/BD): 36 batched tcgen05 GEMMs             */
  UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM = 5, /* TMA-fed implicit GEMM on re-laid copies (all ops), ws ~ b   */
  UCUDNN_ALGO_IMPLICIT_GATHER_GEMM = 6,  /* BF: cp.async-gathered NCHW operands (few-C strided: smem patch); ws O(1) */
  UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM_SLICED = 7, /* F/BD: PRECOMP over reduction-channel slices, copy <= 40 MiB */
  UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM_NHWC = 8, /* BF (stride 1): NHWC copies, TMA im2col, MN-major tcgen05 operands */
  UCUDNN_ALGO_COUNT = 9
} ucudnnAlgo_t;

/* Returned by Get*Algorithm: a plan handle, >= UCUDNN_VIRTUAL_ALGO_BASE
 * (the paper's "virtual algorithm"). Passing a value
 * < UCUDNN_ALGO_COUNT to Convolution* runs that concrete algorithm undivided. */
#define UCUDNN_VIRTUAL_ALGO_BASE 1000

typedef struct ucudnnContext* UcudnnHandle_t;
typedef struct ucudnnTensorStruct* ucudnnTensorDescriptor_t;
typedef struct ucudnnFilterStruct* ucudnnFilterDescriptor_t;
typedef struct ucudnnConvolutionStruct* ucudnnConvolutionDescriptor_t;

/* ------------------------------------------------------------ errors ----- */
const char* ucudnnGetErrorString(ucudnnStatus_t status);
/* Message of the last failing call on this host thread ("" if none). */
const char* ucudnnGetLastError(void);
/* After NOT_SUPPORTED from a WD optimisation: the smallest achievable total
 * workspace in bytes, or -1 (reference infeasible_error::min_total_workspace,
 * domain.hpp:48-58). */
int64_t ucudnnGetMinTotalWorkspace(void);
size_t ucudnnGetVersion(void);
/* Number of device kernels this library has launched in this process. */
uint64_t ucudnnGetLaunchCount(void);
/* Diagnostic: mean MMA-warp cycles {waiting for operands, issuing, waiting
 * for a free accumulator, total} per CTA of the last IMPLICIT_PRECOMP_GEMM
 * launch made with UCUDNN_TUNE=prof=1 (zeros otherwise). */
ucudnnStatus_t ucudnnDebugPrecompProfile(double* out4);
/* Same split for the last IMPLICIT_PRECOMP_GEMM BackwardFilter launch. */
ucudnnStatus_t ucudnnDebugBackwardFilterProfile(double* out4);
/* Launch-variant trace (test evidence; no reference counterpart): on != 0
 * clears and enables a process-wide log in which every main-kernel launch
 * appends one line naming its variant and tiling ("precomp2 m_tiles=...",
 * "bfn2 ...", "precomp cps=2 ..."); ucudnnDebugGetTrace copies the log out
 * (same *len convention as ucudnnGetMachineReport) and clears it. */
ucudnnStatus_t ucudnnDebugSetTrace(int on);
ucudnnStatus_t ucudnnDebugGetTrace(char* buf, size_t* len);

/* ------------------------------------------------------------ handle ----- */
/* Replaces cudnnCreate/cudnnDestroy/cudnnSetStream. The
 * handle owns: the device it was created on, a stream (default 0), the plan
 * cache, the cost table and the WD arena. One host thread per handle. */
ucudnnStatus_t ucudnnCreate(UcudnnHandle_t* handle);
ucudnnStatus_t ucudnnDestroy(UcudnnHandle_t handle);
ucudnnStatus_t ucudnnSetStream(UcudnnHandle_t handle, void* cuda_stream);
ucudnnStatus_t ucudnnGetStream(UcudnnHandle_t handle, void** cuda_stream);

/* Policy / mode / budget setters ("via an environment variable
 * or through a special library function"). Env mirrors read at ucudnnCreate:
 * UCUDNN_BATCH_SIZE_POLICY (all|powerOfTwo|undivided), UCUDNN_WORKSPACE_MODE
 * (wr|wd), UCUDNN_TOTAL_WORKSPACE_SIZE (bytes), UCUDNN_DATABASE (csv path),
 * UCUDNN_BENCHMARK_ITERS. Setters win over env (reference README.md:73-78). */
ucudnnStatus_t ucudnnSetBatchSizePolicy(UcudnnHandle_t h, ucudnnBatchSizePolicy_t policy);
ucudnnStatus_t ucudnnSetWorkspaceMode(UcudnnHandle_t h, ucudnnWorkspaceMode_t mode);
ucudnnStatus_t ucudnnSetTotalWorkspaceLimit(UcudnnHandle_t h, int64_t bytes);
/* Cost table file (reference CostDatabase::open, cost_database.hpp:72-77):
 * rows found there are not re-benchmarked; new rows are appended on
 * ucudnnFlushCostDatabase (atomic tmp+rename, cost_database.hpp:119-137). */
ucudnnStatus_t ucudnnSetCostDatabase(UcudnnHandle_t h, const char* csv_path);
ucudnnStatus_t ucudnnFlushCostDatabase(UcudnnHandle_t h);
ucudnnStatus_t ucudnnSetBenchmarkIterations(UcudnnHandle_t h, int warmup, int iters);
/* Deterministic BackwardFilter (cudnnSetConvolutionMathType-style knob; no
 * reference counterpart -- the reference's fp64 loops are deterministic by
 * construction, reference_conv.hpp:141-171). on != 0: every BackwardFilter
 * kernel gives each dW partial a single writer per launch (split-K off; the
 * few-channel patch kernel adds per-CTA slices in a fixed order), so dW is
 * bit-identical run to run on any data. Costs speed on split-K shapes; the
 * benchmarker times this mode's kernels, so keep one cost database per mode.
 * Env mirror: UCUDNN_DETERMINISTIC=1. Re-plans the handle's kernels. */
ucudnnStatus_t ucudnnSetDeterministic(UcudnnHandle_t h, int on);
/* Math mode (above). Env mirror: UCUDNN_MATH_MODE=fp32|tf32. Like
 * ucudnnSetDeterministic it starts an empty cost table (rows are mode
 * specific; set a per-mode database again) and re-plans. */
ucudnnStatus_t ucudnnSetMathMode(UcudnnHandle_t h, ucudnnMathMode_t mode);
/* Parallel benchmarking ("evaluate in parallel on multiple
 * GPUs"): the missing (algorithm x micro-batch) rows
 * of a kernel are timed by one host thread per listed device, each with its own
 * stream, scratch and L2-flush buffer, then merged into the cost table. n = 0
 * restores the default (the handle's device and stream). Ids are CUDA ordinals;
 * out of range -> BAD_PARAM. Replaces nothing in the reference (its cost
 * source is the analytic model or a CSV, cost_provider.hpp:93-106). */
ucudnnStatus_t ucudnnSetBenchmarkDevices(UcudnnHandle_t h, const int* device_ids, int n);

/* ------------------------------------------------------------ descriptors  */
ucudnnStatus_t ucudnnCreateTensorDescriptor(ucudnnTensorDescriptor_t* d);
ucudnnStatus_t ucudnnSetTensor4dDescriptor(ucudnnTensorDescriptor_t d, int n, int c, int h, int w);
ucudnnStatus_t ucudnnGetTensor4dDescriptor(ucudnnTensorDescriptor_t d, int* n, int* c, int* h, int* w);
ucudnnStatus_t ucudnnDestroyTensorDescriptor(ucudnnTensorDescriptor_t d);
ucudnnStatus_t ucudnnCreateFilterDescriptor(ucudnnFilterDescriptor_t* d);
ucudnnStatus_t ucudnnSetFilter4dDescriptor(ucudnnFilterDescriptor_t d, int k, int c, int r, int s);
ucudnnStatus_t ucudnnDestroyFilterDescriptor(ucudnnFilterDescriptor_t d);
ucudnnStatus_t ucudnnCreateConvolutionDescriptor(ucudnnConvolutionDescriptor_t* d);
ucudnnStatus_t ucudnnSetConvolution2dDescriptor(ucudnnConvolutionDescriptor_t d, int pad_h, int pad_w,
                                                int stride_h, int stride_w, int dilation_h, int dilation_w);
ucudnnStatus_t ucudnnGetConvolution2dForwardOutputDim(ucudnnConvolutionDescriptor_t conv,
                                                      ucudnnTensorDescriptor_t x, ucudnnFilterDescriptor_t w,
                                                      int* n, int* c, int* h, int* wd);
ucudnnStatus_t ucudnnDestroyConvolutionDescriptor(ucudnnConvolutionDescriptor_t d);

/* ------------------------------------------------------------ planning --- */
/* Get*Algorithm: registers the kernel (reference KernelDescriptor,
 * domain.hpp:89-121; N is the descriptor's batch) and returns a virtual
 * algorithm id. WR: plans immediately under `ws_limit_bytes` (benchmarking
 * missing cost rows on the handle's device, then wr_optimize,
 * wr_optimizer.hpp:101-117). WD: only registers; the plan is made on the
 * first Convolution* call or ucudnnOptimizeNetwork. */
ucudnnStatus_t ucudnnGetConvolutionForwardAlgorithm(UcudnnHandle_t h, ucudnnTensorDescriptor_t x,
                                                    ucudnnFilterDescriptor_t w, ucudnnConvolutionDescriptor_t conv,
                                                    ucudnnTensorDescriptor_t y, int64_t ws_limit_bytes,
                                                    int* algo);
ucudnnStatus_t ucudnnGetConvolutionBackwardDataAlgorithm(UcudnnHandle_t h, ucudnnFilterDescriptor_t w,
                                                         ucudnnTensorDescriptor_t dy,
                                                         ucudnnConvolutionDescriptor_t conv,
                                                         ucudnnTensorDescriptor_t dx, int64_t ws_limit_bytes,
                                                         int* algo);
ucudnnStatus_t ucudnnGetConvolutionBackwardFilterAlgorithm(UcudnnHandle_t h, ucudnnTensorDescriptor_t x,
                                                           ucudnnTensorDescriptor_t dy,
                                                           ucudnnConvolutionDescriptor_t conv,
                                                           ucudnnFilterDescriptor_t dw, int64_t ws_limit_bytes,
                                                           int* algo);
/* Workspace the caller must pass: the plan's max micro workspace in WR, 0 in
 * WD (library-owned arena); concrete ids report their own
 * undivided requirement. */
ucudnnStatus_t ucudnnGetConvolutionWorkspaceSize(UcudnnHandle_t h, int algo, ucudnnOp_t op,
                                                 ucudnnTensorDescriptor_t x_or_dy, ucudnnFilterDescriptor_t w,
                                                 ucudnnConvolutionDescriptor_t conv, size_t* bytes);
/* WD: optimise every registered kernel now (wd_optimize, wd_optimizer.hpp:
 * 589-649) and size the arena; the explicit form of the paper's deferred
 * first-call optimisation. */
ucudnnStatus_t ucudnnOptimizeNetwork(UcudnnHandle_t h);
/* Plan of a virtual id: n_micro and (alg, batch) pairs in canonical order. */
ucudnnStatus_t ucudnnGetPlan(UcudnnHandle_t h, int algo, int* n_micro, int* algs, int64_t* batches,
                             int capacity);
/* Machine report of every plan made on this handle (report.hpp:148-197). */
ucudnnStatus_t ucudnnGetMachineReport(UcudnnHandle_t h, char* buf, size_t* len);

/* ------------------------------------------------------------ execution -- */
/* cuDNN-style alpha/beta: out = alpha * conv + beta * out. Forward and
 * BackwardData apply them per micro-batch slice; BackwardFilter applies the
 * user's beta to the first micro-batch and beta = 1 afterwards
 * (reference execute_plan, reference_conv.hpp:205-278).
 * All micro-batches launch back to back on the handle's stream. */
ucudnnStatus_t ucudnnConvolutionForward(UcudnnHandle_t h, const void* alpha, ucudnnTensorDescriptor_t xd,
                                        const void* x, ucudnnFilterDescriptor_t wd, const void* w,
                                        ucudnnConvolutionDescriptor_t conv, int algo, void* workspace,
                                        size_t ws_bytes, const void* beta, ucudnnTensorDescriptor_t yd, void* y);
ucudnnStatus_t ucudnnConvolutionBackwardData(UcudnnHandle_t h, const void* alpha, ucudnnFilterDescriptor_t wd,
                                             const void* w, ucudnnTensorDescriptor_t dyd, const void* dy,
                                             ucudnnConvolutionDescriptor_t conv, int algo, void* workspace,
                                             size_t ws_bytes, const void* beta, ucudnnTensorDescriptor_t dxd,
                                             void* dx);
ucudnnStatus_t ucudnnConvolutionBackwardFilter(UcudnnHandle_t h, const void* alpha, ucudnnTensorDescriptor_t xd,
                                               const void* x, ucudnnTensorDescriptor_t dyd, const void* dy,
                                               ucudnnConvolutionDescriptor_t conv, int algo, void* workspace,
                                               size_t ws_bytes, const void* beta, ucudnnFilterDescriptor_t dwd,
                                               void* dw);

/* ------------------------------------------------------------ benchmarker  */
/* Times one (op, shape, algorithm, micro-batch) on the handle's stream with
 * CUDA events (medians of `iters` L2-flushed runs after `warmup`) and reports
 * the workspace it needs. *feasible = 0 when the algorithm does not support
 * the shape (or its workspace does not fit in device memory). The cost is the
 * steady-state micro-batch time plus the batch-independent filter preparation
 * amortised over the ceil(N / micro_batch) micro-batches of a uniform plan
 * (here, with no full batch known, N = micro_batch: preparation charged in
 * full); ucudnnBenchmarkKernel charges it over the kernel's batch. These are
 * the rows of the reference cost table (CostRecord, domain.hpp:300-318). */
ucudnnStatus_t ucudnnTimeAlgorithm(UcudnnHandle_t h, ucudnnOp_t op, const int64_t* shape11, int algo,
                                   int64_t micro_batch, double* time_us, int64_t* ws_bytes, int* feasible);
/* Benchmarks every algorithm x policy size for one kernel into the handle's
 * cost table (skipping rows already present). shape11 = {N,C,H,W,K,R,S,
 * pad_h,pad_w,stride_h,stride_w}. */
ucudnnStatus_t ucudnnBenchmarkKernel(UcudnnHandle_t h, ucudnnOp_t op, const int64_t* shape11,
                                     ucudnnBatchSizePolicy_t policy);
/* Workspace bytes algorithm `algo` needs for micro-batch b (0 if none);
 * *feasible = 0 if unsupported. Pure host computation. */
ucudnnStatus_t ucudnnAlgorithmWorkspace(ucudnnOp_t op, const int64_t* shape11, int algo, int64_t micro_batch,
                                        int64_t* ws_bytes, int* feasible);

/* ------------------------------------------------------------ planner ---- */
/* The reference planner seam as one call: `ubatch optimize` (reference
 * tools/main.cpp:116-155 -> harness.hpp:43-106). network_path: a .net file
 * (network.hpp:52-169); batch_override > 0 replaces its minibatch; cost_path
 * NULL/"" or "builtin" = synthetic model (cost_model.hpp:165-177), a file
 * whose first line is the cost-CSV header = measurement table only
 * (cost_provider.hpp:104-106), else a model file (cost_model.hpp:182-275);
 * cache_csv optional write-through table flushed afterwards. report_kind 0 =
 * machine report, 1 = text report. On *len too small returns BAD_PARAM and
 * sets *len to the needed size (including the NUL). */
ucudnnStatus_t ucudnnPlanNetworkFile(const char* network_path, int64_t batch_override, const char* cost_path,
                                     const char* cache_csv, int mode, int policy, int64_t limit, unsigned jobs,
                                     int report_kind, char* out, size_t* len);
/* Same, for an explicit kernel list (kinds: shape rows of 12 int64 =
 * {op,N,C,H,W,K,R,S,ph,pw,sh,sw}; names: n NUL-terminated strings) and a
 * cost table given as CSV text (table-only provider). */
ucudnnStatus_t ucudnnPlanKernels(const char* network_name, const int64_t* kernels12, const char* const* names,
                                 int n_kernels, const char* cost_csv_text, int mode, int policy, int64_t limit,
                                 unsigned jobs, char* out, size_t* len);
/* FNV-1a canonical hash of a kernel (domain.hpp:159-180). */
uint64_t ucudnnKernelHash(const int64_t* kernel12);
/* Cost-table seam utilities: parse an exact time ("27.6", "3/4") and render
 * it canonically (rational.hpp:161-230); parse a cost-table CSV and re-emit
 * it sorted and canonical (cost_database.hpp:119-222). */
ucudnnStatus_t ucudnnCanonicalTime(const char* text, char* out, size_t* len);
ucudnnStatus_t ucudnnCanonicalCostTable(const char* csv_text, char* out, size_t* len);

#ifdef __cplusplus
}
#endif
#endif /* UCUDNN_H_ */
