// Thin inline-PTX layer for sm_100a: mbarriers, bulk async copies, TMEM and
// tcgen05.mma (kind::tf32). Everything here compiles only for
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cstdint>

namespace ucudnn {
namespace sm100 {

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Spin on try_wait without a suspend-time hint: a hinted wait parks the warp
// (NANOSLEEP.SYNCS) and its wake-up latency was a fixed ~1 us per pipeline
// step in the first profiles.
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Generic-proxy smem stores must be made visible to the async proxy (the
// tensor core reads operands through it) before the consumer is signalled.
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- TMEM
template <int kCols>
__device__ __forceinline__ void tmem_alloc(std::uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_free(std::uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---------------------------------------------------------------- UMMA
// Shared-memory matrix descriptor, no swizzle ("interleaved" canonical
// layout): core matrices of 8 rows x 16 B stored contiguously (128 B);
// `lbo` = byte distance between core matrices adjacent in K, `sbo` = byte
// distance between core matrices adjacent in M/N. Bits 46-47 = 1 (sm100
// descriptor version), layout type 0 (SWIZZLE_NONE).
__device__ __forceinline__ std::uint64_t umma_desc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= std::uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= std::uint64_t(1) << 46;
  return d;
}

// Instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major.
__host__ __device__ constexpr std::uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)            // c_format = F32
         | (2u << 7)          // a_format = TF32
         | (2u << 10)         // b_format = TF32
         | (std::uint32_t(N >> 3) << 17) | (std::uint32_t(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, M x N x 8, issued by one thread.
__device__ __forceinline__ void mma_tf32(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                         std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on `bar` once every previously issued tcgen05 op of this thread is
// complete (implicitly fences before_thread_sync).
__device__ __forceinline__ void mma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets TMEM lane
// (base lane + i), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, float (&v)[32]) {
  std::uint32_t* r = reinterpret_cast<std::uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; it must call pdl_wait() before its first global memory
// access (read or write) and may call pdl_trigger() to let its own successor
// be scheduled early. Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- clusters / 2-SM
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ std::uint32_t cluster_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ std::uint32_t mapa(std::uint32_t saddr, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(std::uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_alloc_2sm(std::uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_free_2sm(std::uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
// Warp-wide forms of the above: the whole (converged) warp executes them and
// one elected lane issues. Called that way, operands every lane computes
// from warp-uniform values (kernel parameters, loop counters, smem
// addresses, a TMEM base read through __shfl_sync) stay in uniform
// registers; issued from inside `if (lane == 0)` ptxas instead wraps every
// tcgen05 instruction in an R2UR.BROADCAST "waterfall" loop, which measured
// ~4x slower per MMA (scripts/mma_ts_probe.cu; DESIGN finding 21).
__device__ __forceinline__ void mma_tf32_w(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                           std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(std::uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_tf32_2sm_w(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                               std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_2sm_w(std::uint64_t* bar, std::uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// TMEM base address made provably warp-uniform (read from shared memory it
// is a per-thread value to the compiler).
__device__ __forceinline__ std::uint32_t tmem_base_uniform(const std::uint32_t* slot) {
  return __shfl_sync(0xffffffffu, *slot, 0);
}

// D[tmem] (+)= A * B^T over a CTA pair: M = 256 (128 rows of A per CTA), B
// split along N (N/2 rows per CTA); issued by the pair's rank-0 CTA.
__device__ __forceinline__ void mma_tf32_2sm(std::uint32_t d_tmem, std::uint64_t adesc, std::uint64_t bdesc,
                                             std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` (same smem offset) in every CTA of `mask` once the pair's
// previously issued tcgen05 ops complete
__device__ __forceinline__ void mma_commit_2sm(std::uint64_t* bar, std::uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// TMA loads into this CTA's smem whose transaction bytes count on the pair
// leader's mbarrier (`bar_cluster` = mapa(bar, 0))
__device__ __forceinline__ void tma_im2col_4d_2sm(void* dst, const void* tmap, std::uint32_t bar_cluster, int c, int w,
                                                  int h, int n, unsigned short ow, unsigned short oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_4d_2sm(void* dst, const void* tmap, std::uint32_t bar_cluster, int x, int y, int z,
                                           int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void tma_2d_2sm(void* dst, const void* tmap, std::uint32_t bar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}

// fp32 atomic add without return (RED).
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Ring position (slot, parity) stepped once per use: the kernels' hot
// producer / issuer loops used g % n and g / n with a runtime n, a software
// division each that was a large share of their issued instructions.
struct RingPos {
  int slot = 0, ph = 0;
  __device__ __forceinline__ void step(int n) {
    if (++slot == n) {
      slot = 0;
      ph ^= 1;
    }
  }
};
// ... and the producer (of np sharing the ring round-robin) that owns slot
struct RingOwner {
  int slot = 0, ph = 0, own = 0;
  __device__ __forceinline__ void step(int n, int np) {
    if (++slot == n) {
      slot = 0;
      ph ^= 1;
      own = 0;
    } else if (++own == np) {
      own = 0;
    }
  }
};

}  // namespace sm100
}  // namespace ucudnn

namespace ucudnn {
namespace sm100 {

// SWIZZLE_128B K-major smem descriptor: 8-row x 128 B atoms (1024 B apart).
__device__ __forceinline__ std::uint64_t umma_desc_sw128(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= std::uint64_t(1024 >> 4) << 32;         // SBO
  d |= std::uint64_t(1) << 46;                 // version
  d |= std::uint64_t(2) << 61;                 // SWIZZLE_128B
  return d;
}

// SWIZZLE_128B MN-major descriptor: atoms of 8 K-rows x 128 B (32 MN
// elements); `lbo` = byte stride between 32-element MN blocks, `sbo` = byte
// stride between 8-row K groups.
__device__ __forceinline__ std::uint64_t umma_desc_mn_sw128(std::uint32_t saddr, std::uint32_t lbo,
                                                            std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= std::uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(2) << 61;
  return d;
}

// Instruction descriptor, kind::tf32 with both operands MN-major.
__host__ __device__ constexpr std::uint32_t idesc_tf32_mn(int M, int N) {
  return idesc_tf32(M, N) | (1u << 15) | (1u << 16);
}

// TMA im2col load of a 4-D NHWC tensor: `pixels x channels` box starting at
// input coordinate (c, w, h, n) with filter-tap offsets (ow, oh).
__device__ __forceinline__ void tma_im2col_4d(void* dst, const void* tmap, std::uint64_t* bar, int c, int w, int h,
                                              int n, unsigned short ow, unsigned short oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}

// TMA tiled 2-D load: box at (x = inner coordinate, y).
__device__ __forceinline__ void tma_2d(void* dst, const void* tmap, std::uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

}  // namespace sm100
}  // namespace ucudnn
