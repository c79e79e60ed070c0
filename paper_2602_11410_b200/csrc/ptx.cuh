// Blackwell (sm_100a) PTX primitives used by every libcadet kernel:
// mbarrier, TMA (cp.async.bulk.tensor), tcgen05 MMA / TMEM, UMMA descriptors.
// Descriptor bit layouts follow the PTX ISA "tcgen05 shared memory descriptor"
// and "instruction descriptor" tables (same fields as CuTe's UMMA::SmemDescriptor
// and UMMA::InstrDescriptor).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

namespace cadet {

#define CADET_DEV __device__ __forceinline__

CADET_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

CADET_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
CADET_DEV uint32_t lane_id() { return threadIdx.x & 31; }

CADET_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n"
      " elect.sync r|p, 0xffffffff;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ error word
// Bit flags latched by kernels into the workspace error word (see cadet.h).
enum : uint32_t {
  ERRBIT_OFFSETS = 1u << 0,
  ERRBIT_ORDER = 1u << 1,
  ERRBIT_TOO_LONG = 1u << 2,
  ERRBIT_CAND = 1u << 3,
  ERRBIT_BUCKET = 1u << 4,
  ERRBIT_NONFINITE = 1u << 5,
  ERRBIT_TIMEOUT = 1u << 6,
  ERRBIT_CAPACITY = 1u << 7,
};

// ------------------------------------------------------------------ mbarrier
CADET_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CADET_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
CADET_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
CADET_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting thread is parked by the hardware until the phase
// completes (or the hint expires) instead of re-polling, so waiting warps stop stealing issue
// slots from the working warps on their SM sub-partition.
CADET_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}
CADET_DEV uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Bounded wait: a phase that never completes (a bug) traps after ~20 s instead of hanging the GPU.
CADET_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const uint64_t t0 = global_ns();
  // the deadline is checked every 64th unsuccessful try_wait only: a waiting warp issues as few
  // instructions as possible (it shares the scheduler with the warps doing the work)
  for (uint32_t n = 1; !mbar_try_wait(a, parity); ++n) {
    if ((n & 63u) == 0 && global_ns() - t0 > 20000000000ull) {
      printf("cadet: mbarrier timeout block %d thread %d\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

// ------------------------------------------------------------------ fences
CADET_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
CADET_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
CADET_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
CADET_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ TMA
CADET_DEV void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
CADET_DEV void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
CADET_DEV void tma_load_1d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0)
      : "memory");
}
CADET_DEV void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA store (shared -> global, bulk-group completion) and its group waits
CADET_DEV void tma_store_3d(const CUtensorMap* m, uint32_t src_smem, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src_smem), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
CADET_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
CADET_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
CADET_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// L2 eviction-priority policies for TMA loads: streamed-once data (evict_first) must not push out
// tiles that other CTAs re-read (evict_last).
CADET_DEV uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
CADET_DEV uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
CADET_DEV void tma_load_3d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// ------------------------------------------------------------------ tcgen05 / TMEM
template <uint32_t NCOLS>
CADET_DEV void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
CADET_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T-ish (per descriptors), kind::f16 (bf16 in, fp32 acc)
CADET_DEV void mma_bf16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::tf32 (fp32 storage, 10-bit mantissa products, fp32 acc):
// the 3xTF32 parity mode (CADET_FP32); K = 8 per instruction = the same 32 bytes as kind::f16's K = 16
CADET_DEV void mma_tf32_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem] (TS form): A is K-major in TMEM, lane = row, 2 bf16 per column.
CADET_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread complete.
CADET_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane (base+t).
CADET_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
CADET_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
CADET_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
CADET_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
CADET_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM address of lane quarter q (warp % 4), column c.
CADET_DEV uint32_t tmem_addr(uint32_t base, uint32_t lane_quarter, uint32_t col) {
  return base + ((lane_quarter * 32u) << 16) + col;
}

// ------------------------------------------------------------------ clusters / CTA pairs (cta_group::2)
CADET_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
CADET_DEV uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
CADET_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
CADET_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA load: the bytes complete_tx on the barrier at `bar_cluster_addr` (the leader CTA's).
CADET_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cluster_addr, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster_addr), "r"(c0), "r"(c1)
      : "memory");
}
template <uint32_t NCOLS>
CADET_DEV void tmem_alloc_pair(uint32_t* dst_smem) {  // whole warp, in BOTH CTAs of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
CADET_DEV void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
CADET_DEV void mma_bf16_ss_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once the issuing thread's prior tcgen05 ops complete) on the barrier at the same smem
// offset in every CTA of `mask`.
CADET_DEV void mma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ------------------------------------------------------------------ descriptors
enum Swz : uint32_t { SWZ_NONE = 0, SWZ_128B = 2, SWZ_64B = 4, SWZ_32B = 6 };

// Shared-memory matrix descriptor (tcgen05).  Fields: start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), base_offset=0 [49,52), lbo_mode=0 [52], layout [61,64).
CADET_DEV uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t swz) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(swz & 7u) << 61;
  return d;
}

// Instruction descriptor for kind::f16 with bf16 A/B and fp32 D.
// a_mn / b_mn: 1 = MN-major operand, 0 = K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4)            // D format F32
         | (1u << 7)          // A format BF16
         | (1u << 10)         // B format BF16
         | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// kind::tf32 instruction descriptor: D F32, A and B TF32 (format 2), K-major operands
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// Byte offset of 16-byte chunk `chunk` of row `row` inside a swizzled tile whose rows
// are `row_bytes` (= swizzle width) long.  Matches TMA SWIZZLE_{64,128}B / UMMA layouts.
CADET_DEV uint32_t swz_off(uint32_t row, uint32_t chunk, uint32_t row_bytes) {
  if (row_bytes == 128) return row * 128u + ((chunk ^ (row & 7u)) << 4);
  // 64B swizzle: chunk ^= (row >> 1) & 3
  return row * 64u + ((chunk ^ ((row >> 1) & 3u)) << 4);
}

// ------------------------------------------------------------------ small math
// Warpgroup register reallocation (all 4 warps of a warpgroup execute it).
template <uint32_t N>
CADET_DEV void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
CADET_DEV void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

CADET_DEV float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}
CADET_DEV int4 lds_i4(uint32_t saddr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}
CADET_DEV void sts_u4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
CADET_DEV uint4 lds_u4(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr) : "memory");
  return v;
}

// Row-per-lane results (lane = row of a 32-row block, as tcgen05.ld 32x32b delivers them) written
// to global memory through a per-warp shared-memory transpose, so that each store instruction
// covers whole row segments instead of 32 different lines.  XOR-swizzled 16-byte slots keep both
// shared-memory phases conflict-free.
// bf16: w = this lane's 32 columns packed (16 words); stage = 2 KB; g0 = &row0[col0], ld = row stride.
CADET_DEV void warp_store_rows_bf16(uint32_t stage, const uint32_t (&w)[16], __nv_bfloat16* g0, size_t ld,
                                    int rows_valid, int ncol) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    sts_u4(stage + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i * 8 + (lane >> 2), j = lane & 3;
    const uint4 v = lds_u4(stage + row * 64 + ((j ^ ((row >> 1) & 3)) << 4));
    if (row < rows_valid && j * 8 < ncol) *reinterpret_cast<uint4*>(g0 + (size_t)row * ld + j * 8) = v;
  }
  __syncwarp();
}
// The same store in two phases, so the global half can be deferred (e.g. past a barrier arrive):
// warp_stage_rows_bf16 writes the lane's row into the swizzled stage; warp_flush_rows_bf16 issues
// the coalesced global stores from it.
CADET_DEV void warp_stage_rows_bf16(uint32_t stage, const uint32_t (&w)[16]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    sts_u4(stage + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}
// STREAM: evict-first stores (st.global.cs) for data no later kernel re-reads soon from L2.
template <bool STREAM = false>
CADET_DEV void warp_flush_rows_bf16(uint32_t stage, __nv_bfloat16* g0, size_t ld, int rows_valid, int ncol) {
  const uint32_t lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i * 8 + (lane >> 2), j = lane & 3;
    const uint4 v = lds_u4(stage + row * 64 + ((j ^ ((row >> 1) & 3)) << 4));
    if (row < rows_valid && j * 8 < ncol) {
      uint4* dst = reinterpret_cast<uint4*>(g0 + (size_t)row * ld + j * 8);
      if (STREAM)
        __stcs(dst, v);
      else
        *dst = v;
    }
  }
  __syncwarp();
}
// fp32: u = this lane's 32 columns (scaled by f); stage = 4 KB.
CADET_DEV void warp_store_rows_f32(uint32_t stage, const uint32_t (&u)[32], float f, float* g0, size_t ld,
                                   int rows_valid, int ncol) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    sts_u4(stage + lane * 128 + ((j ^ (lane & 7)) << 4), __float_as_uint(f * __uint_as_float(u[4 * j])),
           __float_as_uint(f * __uint_as_float(u[4 * j + 1])), __float_as_uint(f * __uint_as_float(u[4 * j + 2])),
           __float_as_uint(f * __uint_as_float(u[4 * j + 3])));
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = i * 4 + (lane >> 3), j = lane & 7;
    const uint4 v = lds_u4(stage + row * 128 + ((j ^ (row & 7)) << 4));
    if (row < rows_valid && j * 4 < ncol) *reinterpret_cast<uint4*>(g0 + (size_t)row * ld + j * 4) = v;
  }
  __syncwarp();
}

CADET_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (FA4-style MUFU offload): x = n + f with n = rint(x) via the 1.5*2^23
// trick, 2^f on [-1/2, 1/2] by a degree-4 near-minimax polynomial (max rel err 2.7e-6), n added
// to the exponent field as an integer.  x < -126 (incl. -inf) returns exactly 0.
CADET_DEV float exp2_poly(float x) {
  const float xc = fmaxf(x, -127.f);
  const float t = xc + 12582912.f;
  const float f = xc - (t - 12582912.f);
  float p = fmaf(0.00957009536025538f, f, 0.05591786349494091f);
  p = fmaf(p, f, 0.24024745021653496f);
  p = fmaf(p, f, 0.6931218143849706f);
  p = fmaf(p, f, 0.99999926137738f);
  const float r = __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
  return x < -126.f ? 0.f : r;
}
// bf16x2 pack on the ALU pipe (integer round-half-up + PRMT) instead of F2FP: keeps the
// transcendental (XU) pipe free for exp2 in the softmax loops.  Differs from RNE only on exact ties.
CADET_DEV uint32_t pack_bf16_alu(float a, float b) {
  const uint32_t ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  return __byte_perm(ua, ub, 0x7632);
}
CADET_DEV uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
CADET_DEV float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }
// MUFU-only forms for the epilogues: ex2 / rcp with flush-to-zero skip the denormal fix-ups that
// __expf / __fdividef add (3 extra FMUL/FSETP per element); sigma(z) = 1 / (1 + 2^(-z log2 e))
// saturates correctly at both ends (2^+inf = inf -> rcp = 0).
CADET_DEV float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
CADET_DEV float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
CADET_DEV float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// sigma(z) = (1 + tanh(z / 2)) / 2: ONE MUFU op (tanh.approx, rel err <= 2^-10.9) instead of ex2 + rcp;
// absolute error <= ~2.5e-4, below the bf16 rounding of the gated products it feeds
CADET_DEV float sigmoid_fast(float z) { return fmaf(0.5f, tanh_approx(0.5f * z), 0.5f); }

// Warp-cooperative variants: the 32 lanes hold rows row0 .. row0 + 31 of the same 32 columns
// (tcgen05.ld 32x32b layout).  Global traffic goes through a per-warp 4 KB swizzled transpose
// (ptx.cuh) so each load / store instruction covers whole row segments instead of 32 lines.
// bf16 32 x 32 slice in two phases, so the global loads of a later slice can be issued early:
// (1) coalesced loads (8 rows x 64 B per instruction) into registers, (2) transpose to this lane's row.
CADET_DEV void warp_ldg_rows_bf16(const void* base, size_t off0, size_t ld, int rows_valid,
                                                   uint4 (&g)[4]) {
  const uint32_t lane = threadIdx.x & 31;
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(base) + off0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i * 8 + (lane >> 2), j = lane & 3;
    g[i] = row < rows_valid ? *reinterpret_cast<const uint4*>(b + (size_t)row * ld + j * 8) : make_uint4(0, 0, 0, 0);
  }
}
CADET_DEV void warp_sts_rows_bf16(uint32_t stg, const uint4 (&g)[4], float (&x)[32]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = i * 8 + (lane >> 2), j = lane & 3;
    sts_u4(stg + row * 64 + ((j ^ ((row >> 1) & 3)) << 4), g[i].x, g[i].y, g[i].z, g[i].w);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 u = lds_u4(stg + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      x[j * 8 + e * 2] = f.x;
      x[j * 8 + e * 2 + 1] = f.y;
    }
  }
  __syncwarp();
}

// fp32 32 x 32 slice in the same two phases (4 rows x 128 B per load instruction).
CADET_DEV void warp_ldg_rows_f32(const void* base, size_t off0, size_t ld, int rows_valid,
                                                  uint4 (&g)[8]) {
  const uint32_t lane = threadIdx.x & 31;
  const float* b = reinterpret_cast<const float*>(base) + off0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = i * 4 + (lane >> 3), j = lane & 7;
    g[i] = row < rows_valid ? *reinterpret_cast<const uint4*>(b + (size_t)row * ld + j * 4) : make_uint4(0, 0, 0, 0);
  }
}
CADET_DEV void warp_sts_rows_f32(uint32_t stg, const uint4 (&g)[8], float (&x)[32]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = i * 4 + (lane >> 3), j = lane & 7;
    sts_u4(stg + row * 128 + ((j ^ (row & 7)) << 4), g[i].x, g[i].y, g[i].z, g[i].w);
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 u = lds_u4(stg + lane * 128 + ((j ^ (lane & 7)) << 4));
    x[j * 4] = __uint_as_float(u.x);
    x[j * 4 + 1] = __uint_as_float(u.y);
    x[j * 4 + 2] = __uint_as_float(u.z);
    x[j * 4 + 3] = __uint_as_float(u.w);
  }
  __syncwarp();
}

CADET_DEV void warp_load_rows(uint32_t stg, const void* base, int is_f32, size_t off0, size_t ld,
                                               int rows_valid, float (&x)[32]) {
  const uint32_t lane = threadIdx.x & 31;
  if (!is_f32) {
    uint4 g[4];
    warp_ldg_rows_bf16(base, off0, ld, rows_valid, g);
    warp_sts_rows_bf16(stg, g, x);
    return;
  } else {
    uint4 g[8];
    warp_ldg_rows_f32(base, off0, ld, rows_valid, g);
    warp_sts_rows_f32(stg, g, x);
  }
}

}  // namespace cadet
