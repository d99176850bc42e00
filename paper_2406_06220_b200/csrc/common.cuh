// common.cuh -- device helpers shared by the label-looping kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ll {

typedef __nv_bfloat16 bf16;

// ---------------------------------------------------------------------------
// Packed argmax keys.  A logit v at vocabulary index i is encoded as
//   key = (ordered(v) << 32) | (0xFFFFFFFF - i)
// so that an unsigned max over keys yields the maximum logit and, among equal
// logits, the LOWEST index (tie rule of PAPER.md:141 `argmax`, reading A16).
// The max is arrival-order independent, so cross-warp / cross-CTA reductions
// are deterministic.  -0 is canonicalised to +0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ordered_f32(float v) {
  if (v == 0.0f) v = 0.0f;
  uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t pack_key(float v, int idx) {
  return ((uint64_t)ordered_f32(v) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)idx);
}
__device__ __forceinline__ int key_index(uint64_t key) {
  return (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
}
// the logit a key encodes (inverse of ordered_f32)
__device__ __forceinline__ float key_value(uint64_t key) {
  const uint32_t u = (uint32_t)(key >> 32);
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Log-sum-exp partials for the greedy scores (N2): (m, s) with s = sum exp(v - m)
// over a subset of logits, packed in 64 bits (m in the low word).  Combining
// is exact up to rounding and order-independent up to rounding; the kernels
// always combine in a fixed order, so results are deterministic.  The empty
// subset is (-inf, 0).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t lse_pack(float m, float s) {
  return ((uint64_t)__float_as_uint(s) << 32) | __float_as_uint(m);
}
__device__ __forceinline__ float lse_m(uint64_t p) { return __uint_as_float((uint32_t)p); }
__device__ __forceinline__ float lse_s(uint64_t p) { return __uint_as_float((uint32_t)(p >> 32)); }
__device__ __forceinline__ uint64_t lse_empty() { return lse_pack(-INFINITY, 0.f); }
__device__ __forceinline__ uint64_t lse_combine(uint64_t a, uint64_t b) {
  const float ma = lse_m(a), mb = lse_m(b);
  const float m = fmaxf(ma, mb);
  if (m == -INFINITY) return lse_empty();
  return lse_pack(m, lse_s(a) * __expf(ma - m) + lse_s(b) * __expf(mb - m));
}
// log sum exp of the subset
__device__ __forceinline__ float lse_value(uint64_t p) { return lse_m(p) + __logf(lse_s(p)); }
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return ((uint64_t)hi << 32) | lo;
}

// ---------------------------------------------------------------------------
// mma.sync m16n8k16 bf16 -> fp32.  Operand K order: within each 32-wide K
// block, lane q = lane%4 owns physical columns [8q, 8q+8) of both A and B; the
// two k16 steps of the block take columns [8q, 8q+4) and [8q+4, 8q+8).  The
// same permutation of K is applied to A and B, so the contraction is exact
// reordering of the dot product and both operands load with one 16-byte
// vector per row per block (no ldmatrix).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 lds128(const void *p) { return *reinterpret_cast<const uint4 *>(p); }
// 32-bit shared-window addresses (no 64-bit generic address arithmetic)
__device__ __forceinline__ uint4 lds128_u32(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a) : "memory");
  return r;
}
__device__ __forceinline__ void sts128_u32(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint2 lds64(const void *p) { return *reinterpret_cast<const uint2 *>(p); }
__device__ __forceinline__ uint4 ldg128_cg(const void *p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg128_nc(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg64_nc(const void *p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// cp.async 16 B global -> shared, L2 only (data written by other CTAs is read
// through L2; L1 is never stale).
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Thread-block cluster primitives (sm_90+ PTX, used on sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// Full cluster barrier with release/acquire semantics (all threads of all CTAs).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Address of the same shared variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t dsmem_addr(const void *smem_ptr, uint32_t rank) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem_ptr), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(s), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_u64x2(uint32_t addr, uint64_t a, uint64_t b) {
  asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_dsmem_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-async (TMA engine) copies + st.async (sm_90+ PTX on sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// CTA-scope acquire (the default): every barrier in this library completes on
// bulk copies / st.async into this CTA's own shared memory, whose complete_tx
// makes the data visible; .acquire.cluster would add an L1 invalidate
// (CCTL.IVALL) to every wait.
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking test of an mbarrier phase (debug instrumentation)
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}
// Bulk copy global -> this CTA's shared memory; completes `bytes` of tx on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 16-byte store into a (possibly remote) CTA's shared memory that completes
// 16 bytes of tx on that CTA's mbarrier (shared::cluster addresses from mapa).
__device__ __forceinline__ void st_async_u64x2(uint32_t raddr, uint64_t a, uint64_t b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(a), "l"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_u64(uint32_t raddr, uint64_t a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(a), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

// ---------------------------------------------------------------------------
// tcgen05: tensor memory (TMEM) allocation, loads/stores, fences (sm_100a).
// TMEM address = (lane << 16) | column; a warp may access lanes 32*(warp%4)..+31.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t *smem_dst, uint32_t ncols) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 32 lanes x 32 bits, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 32 lanes x 32 bits, 32 consecutive columns per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 32 bits, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// 32 lanes x 32 bits, 4 consecutive columns per thread
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint4 &v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(taddr));
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row
// core groups 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)(1) << 16;                         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;      // stride byte offset
  d |= (uint64_t)1 << 46;                           // version
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

// UMMA shared-memory descriptor, K-major operand WITHOUT swizzle: 8-row x
// 16-byte core matrices (128 contiguous bytes), `lbo` bytes between core
// matrices adjacent in K, `sbo` bytes between 8-row groups (sm_100 version 1).
__device__ __forceinline__ uint64_t umma_desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// D[tmem] (+)= A[tmem] . B[smem]^T, kind::f16 (A from TMEM: lane = row, two
// bf16 K elements per 32-bit column); issued by one thread.
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc)
      : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, kind::f16; issued by one thread.
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc)
      : "memory");
}
// four 8x8 b16 matrices (8 rows x 16 bytes each; lane 8i + r gives the address of matrix i's row r)
__device__ __forceinline__ void ldmatrix_x4(uint32_t saddr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}
// every prior tcgen05 op of this thread completes -> one arrive on `bar`
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// generic-proxy shared-memory writes -> visible to the async proxy (tensor core)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

// bf16x2(relu(lo), relu(hi)), round to nearest (the relu on the rounded value: identical)
__device__ __forceinline__ uint32_t pack_relu_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// z = bf16(relu(f + g)) for 8 elements: f bf16x8, g as two float4 (elements 0-3, 4-7)
__device__ __forceinline__ uint4 relu_add_bf16x8(uint4 f, float4 g0, float4 g1) {
  uint4 o;
  o.x = pack_relu_bf16x2(bf16_lo(f.x) + g0.x, bf16_hi(f.x) + g0.y);
  o.y = pack_relu_bf16x2(bf16_lo(f.y) + g0.z, bf16_hi(f.y) + g0.w);
  o.z = pack_relu_bf16x2(bf16_lo(f.z) + g1.x, bf16_hi(f.z) + g1.y);
  o.w = pack_relu_bf16x2(bf16_lo(f.w) + g1.z, bf16_hi(f.w) + g1.w);
  return o;
}

// as relu_add_bf16x8 with g as raw float4 words; the adds as FADD2 (f32x2)
__device__ __forceinline__ uint32_t add_relu_pack(uint32_t fw, uint32_t g_lo, uint32_t g_hi) {
  const uint64_t fv = ((uint64_t)(fw & 0xffff0000u) << 32) | (uint64_t)(fw << 16);
  const uint64_t gv = ((uint64_t)g_hi << 32) | g_lo;
  uint64_t sv;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(sv) : "l"(fv), "l"(gv));
  return pack_relu_bf16x2(__uint_as_float((uint32_t)sv), __uint_as_float((uint32_t)(sv >> 32)));
}
__device__ __forceinline__ uint4 relu_add_bf16x8_2(uint4 f, uint4 g0, uint4 g1) {
  uint4 o;
  o.x = add_relu_pack(f.x, g0.x, g0.y);
  o.y = add_relu_pack(f.y, g0.z, g0.w);
  o.z = add_relu_pack(f.z, g1.x, g1.y);
  o.w = add_relu_pack(f.w, g1.z, g1.w);
  return o;
}

// dot product of two bf16x8 vectors in fp32 (each product exact in fp32), in element order
__device__ __forceinline__ float dot_bf16x8(uint4 a, uint4 b) {
  float d = bf16_lo(a.x) * bf16_lo(b.x);
  d = fmaf(bf16_hi(a.x), bf16_hi(b.x), d);
  d = fmaf(bf16_lo(a.y), bf16_lo(b.y), d);
  d = fmaf(bf16_hi(a.y), bf16_hi(b.y), d);
  d = fmaf(bf16_lo(a.z), bf16_lo(b.z), d);
  d = fmaf(bf16_hi(a.z), bf16_hi(b.z), d);
  d = fmaf(bf16_lo(a.w), bf16_lo(b.w), d);
  return fmaf(bf16_hi(a.w), bf16_hi(b.w), d);
}

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<bf16>(bf16 v) { return __bfloat162float(v); }

// logistic: fast reciprocal (MUFU.RCP), no IEEE-division slow path; relative error ~1e-7
__device__ __forceinline__ float sigmoidf_(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
// tanh x = 2 s(2x) - 1: absolute error ~1e-7 (a MUFU.EX2 + MUFU.RCP; tanhf is a longer sequence)
__device__ __forceinline__ float tanhf_(float x) { return 2.0f * sigmoidf_(2.0f * x) - 1.0f; }

}  // namespace ll
