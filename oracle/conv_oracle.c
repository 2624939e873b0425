/*
 * TEST INFRASTRUCTURE ONLY -- not part of the product. Imported solely by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the
 * checker.
 *
 * Plain-C fp64 restatement of the reference convolution semantics
 * (/root/reference/proj/include/ubatch/reference_conv.hpp):
 *   conv_forward          reference_conv.hpp:70-100   (gather, zero padding)
 *   conv_backward_data    reference_conv.hpp:105-135  (scatter adjoint)
 *   conv_backward_filter  reference_conv.hpp:141-171  (dw += sum dy*x, no 1/N)
 *   execute_plan          reference_conv.hpp:205-278  (canonical micro order:
 *       F/BD write disjoint slices, BF accumulates into one dw)
 * The loops are reordered for speed (per-sample OpenMP, output-stationary
 * inner loops) but every output element is the same exact sum; on integer
 * data the results are bit-identical to the reference (pinned in
 * tests/test_oracle.py against oracle/_ref/ref_conv.so and tests/golden/).
 *
 * Tensors are NCHW row-major doubles; shape = {N,C,H,W,K,R,S,ph,pw,sh,sw}.
 */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef long long i64;

/* Minimal pthread fan-out over [0, n): body(i, ctx) for each i. */
typedef void (*body_fn)(i64 i, const void* ctx);
struct span { body_fn f; const void* ctx; i64 lo, hi; };
static void* run_span(void* p) {
  struct span* s = (struct span*)p;
  for (i64 i = s->lo; i < s->hi; ++i) s->f(i, s->ctx);
  return NULL;
}
static int g_threads = 0;
void oracle_set_threads(int t) { g_threads = t; }
static void par_for(i64 n, body_fn f, const void* ctx) {
  int t = g_threads > 0 ? g_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (t < 1) t = 1;
  if (t > 256) t = 256;
  if ((i64)t > n) t = (int)n;
  if (t <= 1) { for (i64 i = 0; i < n; ++i) f(i, ctx); return; }
  pthread_t th[256];
  struct span sp[256];
  i64 per = (n + t - 1) / t;
  for (int j = 0; j < t; ++j) {
    sp[j].f = f; sp[j].ctx = ctx; sp[j].lo = j * per; sp[j].hi = (j + 1) * per < n ? (j + 1) * per : n;
    pthread_create(&th[j], NULL, run_span, &sp[j]);
  }
  for (int j = 0; j < t; ++j) pthread_join(th[j], NULL);
}
struct job { const i64* sh; const double* a; const double* b; double* out; };

static i64 outdim(i64 in, i64 k, i64 p, i64 s) { return (in + 2 * p - k) / s + 1; }

/* y[n,k,oh,ow] = sum_{c,r,s} w[k,c,r,s] * x[n,c,oh*sh-ph+r, ow*sw-pw+s] */
static void fwd_sample(i64 n, const void* ctx) {
  const struct job* j = (const struct job*)ctx;
  const i64* sh = j->sh;
  const double *x = j->a, *w = j->b;
  double* y = j->out;
  i64 C = sh[1], H = sh[2], W = sh[3], K = sh[4], R = sh[5], S = sh[6];
  i64 ph = sh[7], pw = sh[8], sy = sh[9], sx = sh[10];
  i64 OH = outdim(H, R, ph, sy), OW = outdim(W, S, pw, sx);
  {
    for (i64 k = 0; k < K; ++k)
      for (i64 oh = 0; oh < OH; ++oh)
        for (i64 ow = 0; ow < OW; ++ow) {
          double acc = 0.0;
          for (i64 c = 0; c < C; ++c)
            for (i64 r = 0; r < R; ++r) {
              i64 hi = oh * sy - ph + r;
              if (hi < 0 || hi >= H) continue;
              const double* xr = x + ((n * C + c) * H + hi) * W;
              const double* wr = w + ((k * C + c) * R + r) * S;
              for (i64 s = 0; s < S; ++s) {
                i64 wi = ow * sx - pw + s;
                if (wi < 0 || wi >= W) continue;
                acc += wr[s] * xr[wi];
              }
            }
          y[((n * K + k) * OH + oh) * OW + ow] = acc;
        }
  }
}
void oracle_conv_forward(const i64* sh, const double* x, const double* w, double* y) {
  struct job j = {sh, x, w, y};
  par_for(sh[0], fwd_sample, &j);
}

/* dx[n,c,hi,wi] = sum over (k,r,s,oh,ow) with oh*sh-ph+r = hi, ow*sw-pw+s = wi
 * of w[k,c,r,s] * dy[n,k,oh,ow]  (gather form of the reference scatter) */
static void bd_sample(i64 n, const void* ctx) {
  const struct job* j = (const struct job*)ctx;
  const i64* sh = j->sh;
  const double *dy = j->a, *w = j->b;
  double* dx = j->out;
  i64 C = sh[1], H = sh[2], W = sh[3], K = sh[4], R = sh[5], S = sh[6];
  i64 ph = sh[7], pw = sh[8], sy = sh[9], sx = sh[10];
  i64 OH = outdim(H, R, ph, sy), OW = outdim(W, S, pw, sx);
  {
    for (i64 c = 0; c < C; ++c)
      for (i64 hi = 0; hi < H; ++hi)
        for (i64 wi = 0; wi < W; ++wi) {
          double acc = 0.0;
          for (i64 k = 0; k < K; ++k)
            for (i64 r = 0; r < R; ++r) {
              i64 t = hi + ph - r;
              if (t < 0 || t % sy) continue;
              i64 oh = t / sy;
              if (oh >= OH) continue;
              for (i64 s = 0; s < S; ++s) {
                i64 u = wi + pw - s;
                if (u < 0 || u % sx) continue;
                i64 ow = u / sx;
                if (ow >= OW) continue;
                acc += w[((k * C + c) * R + r) * S + s] * dy[((n * K + k) * OH + oh) * OW + ow];
              }
            }
          dx[((n * C + c) * H + hi) * W + wi] = acc;
        }
  }
}
void oracle_conv_backward_data(const i64* sh, const double* dy, const double* w, double* dx) {
  struct job j = {sh, dy, w, dx};
  par_for(sh[0], bd_sample, &j);
}

/* dw[k,c,r,s] += sum_{n,oh,ow} dy[n,k,oh,ow] * x[n,c,oh*sh-ph+r, ow*sw-pw+s] */
static void bf_filter(i64 k, const void* ctx) {
  const struct job* j = (const struct job*)ctx;
  const i64* sh = j->sh;
  const double *x = j->a, *dy = j->b;
  double* dw = j->out;
  i64 N = sh[0], C = sh[1], H = sh[2], W = sh[3], K = sh[4], R = sh[5], S = sh[6];
  i64 ph = sh[7], pw = sh[8], sy = sh[9], sx = sh[10];
  i64 OH = outdim(H, R, ph, sy), OW = outdim(W, S, pw, sx);
  {
    for (i64 c = 0; c < C; ++c)
      for (i64 r = 0; r < R; ++r)
        for (i64 s = 0; s < S; ++s) {
          double acc = 0.0;
          for (i64 n = 0; n < N; ++n)
            for (i64 oh = 0; oh < OH; ++oh) {
              i64 hi = oh * sy - ph + r;
              if (hi < 0 || hi >= H) continue;
              for (i64 ow = 0; ow < OW; ++ow) {
                i64 wi = ow * sx - pw + s;
                if (wi < 0 || wi >= W) continue;
                acc += dy[((n * K + k) * OH + oh) * OW + ow] * x[((n * C + c) * H + hi) * W + wi];
              }
            }
          dw[((k * C + c) * R + r) * S + s] += acc;
        }
  }
}
void oracle_conv_backward_filter_acc(const i64* sh, const double* x, const double* dy, double* dw) {
  struct job j = {sh, x, dy, dw};
  par_for(sh[4], bf_filter, &j);
}

static int cmp_desc(const void* a, const void* b) {
  i64 x = *(const i64*)a, y = *(const i64*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* execute_plan semantics: micro-batches in canonical (descending) order,
 * slices [off, off+b); F/BD store, BF accumulates into a zeroed dw. */
int oracle_execute_plan(int op, const i64* sh, const i64* micro, int n_micro, const double* a, const double* b,
                        double* out) {
  i64 N = sh[0], C = sh[1], H = sh[2], W = sh[3], K = sh[4], R = sh[5], S = sh[6];
  i64 OH = outdim(H, R, sh[7], sh[9]), OW = outdim(W, S, sh[8], sh[10]);
  i64* m = (i64*)malloc(sizeof(i64) * (size_t)n_micro);
  i64 total = 0;
  for (int i = 0; i < n_micro; ++i) { m[i] = micro[i]; total += micro[i]; }
  if (total != N) { free(m); return 1; }
  qsort(m, (size_t)n_micro, sizeof(i64), cmp_desc);
  i64 x_ss = C * H * W, y_ss = K * OH * OW;
  if (op == 2) memset(out, 0, sizeof(double) * (size_t)(K * C * R * S));
  i64 off = 0;
  for (int i = 0; i < n_micro; ++i) {
    i64 s2[11];
    memcpy(s2, sh, sizeof s2);
    s2[0] = m[i];
    if (op == 0) oracle_conv_forward(s2, a + off * x_ss, b, out + off * y_ss);
    else if (op == 1) oracle_conv_backward_data(s2, a + off * y_ss, b, out + off * x_ss);
    else oracle_conv_backward_filter_acc(s2, a + off * x_ss, b + off * y_ss, out);
    off += m[i];
  }
  free(m);
  return 0;
}
