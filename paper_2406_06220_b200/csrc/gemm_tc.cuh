// gemm_tc.cuh -- Y[M,N] = X[M,K] . W[N,K]^T + bias[N] (+ bias2[N]) on the
// 5th-generation tensor cores (sm_100a): TMA (cp.async.bulk.tensor, 128-byte
// swizzle) stages 128x64 tiles of X and W through a 4-stage shared-memory ring;
// a producer warp, an MMA warp (tcgen05.mma kind::f16, M=128, N=128, K=16,
// fp32 accumulators in TMEM, double-buffered) and four epilogue warps
// (tcgen05.ld, bias, conversion, store) run as a persistent pipeline.
//
// Used for the throughput-bound projections of PAPER.md §3.4 (:216-222): the
// encoder projection f = W_enc enc + b_enc over all B*T_max frames (Alg. 3
// line 2) and the model tables (E' = Emb W_ih^T + b_ih + b_hh, G_k).  Shapes
// it does not cover (K % 64, N % 128, misaligned rows) fall back to the
// mma.sync kernel of linear.cuh.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace ll {

// Output tiles are 128 x 256 (the last tile of a row 128 x (N % 256)): the
// wider B tile halves the operand bytes staged per MMA cycle against 128 x 128.
constexpr int TC_BM = 128, TC_BN = 256, TC_BNQ = 128, TC_BK = 64, TC_STAGES = 4;   // N % TC_BNQ == 0
constexpr int TC_TILE_A = TC_BM * TC_BK * 2;   // 16 KB
constexpr int TC_TILE_B = TC_BN * TC_BK * 2;   // 32 KB (rows past N are zero-filled by the TMA)
constexpr int TC_SMEM = TC_STAGES * (TC_TILE_A + TC_TILE_B) + 1024;   // + alignment slack

struct TcGemmArgs {
  const void *bias, *bias2;   // bf16 [N] or nullptr
  void *Y;
  int64_t ldy;
  int M, N, K;
  // Rows are Bu SEGMENTS of T rows (row r = b * T + t; without lengths: one
  // segment, T = M).  Optional ragged rows (the encoder projection): row
  // b * T + t is used only if t < lengths[b].  M tiles never straddle a
  // segment (X is read as a 3-D tensor {K, T, Bu}, rows past T zero-filled)
  // and only the tiles of used rows exist: ceil(min(lengths[b], T) / 128) per
  // segment, dealt round-robin to the persistent CTAs, so padding frames cost
  // neither MMAs nor load imbalance (frames t >= lengths[b] are never read).
  const int *lengths;
  int T, Bu;
  int bn;   // output tile width: TC_BN (256) or TC_BNQ (128, small problems: more tiles than SMs)
};

// Walks the segments' M tiles in order (tile index mi -> segment b, first row
// t0); every role of a CTA walks the same sequence.
struct TileCursor {
  int b = 0, cum = 0, cb = 0, L = 0;   // segment b: used rows L, its first tile index cum, tile count cb
  __device__ __forceinline__ void load(const TcGemmArgs &a) {
    L = 0;
    if (b < a.Bu) {
      L = a.lengths ? a.lengths[b] : a.T;
      L = L < 0 ? 0 : (L > a.T ? a.T : L);
    }
    cb = (L + TC_BM - 1) / TC_BM;
  }
  __device__ __forceinline__ void init(const TcGemmArgs &a) {
    b = 0;
    cum = 0;
    load(a);
  }
  // position on tile index mi (non-decreasing across calls); false past the end
  __device__ __forceinline__ bool seek(const TcGemmArgs &a, int mi) {
    while (b < a.Bu && mi >= cum + cb) {
      cum += cb;
      ++b;
      load(a);
    }
    return b < a.Bu;
  }
  __device__ __forceinline__ int t0(int mi) const { return (mi - cum) * TC_BM; }
};

// Instruction descriptor: D fp32, A/B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Persistent, warp-specialized: grid = number of SMs (one CTA each); CTA c
// takes output tiles c, c + gridDim.x, ... of the used tiles (tile = (m-tile,
// n-tile), n fastest; TileCursor maps m-tile indices to segments).
//   warp 0:    TMA producer (lane 0): A/B 128x64 k-blocks into a TC_STAGES ring
//   warp 1:    MMA issuer (lane 0): tcgen05.mma into one of TWO TMEM
//              accumulators (128 columns each), tcgen05.commit per k-block
//              (frees the stage) and per tile (accumulator full)
//   warps 2-5: epilogue (TMEM lane quarter = warp % 4): accumulator -> bias ->
//              global, then release the accumulator, so the MMAs of tile i+1
//              overlap the epilogue of tile i.
constexpr int TC_THREADS = 192;

template <typename OutT>
__global__ void __launch_bounds__(TC_THREADS, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                                                                const __grid_constant__ CUtensorMap map_w,
                                                                const __grid_constant__ TcGemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);   // SW128 atoms: 1024-B aligned
  __shared__ __align__(8) uint64_t full[TC_STAGES], empty[TC_STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = a.K / TC_BK;
  const int nt = (a.N + a.bn - 1) / a.bn;
  const uint32_t stage_tx = (uint32_t)(TC_TILE_A + a.bn * TC_BK * 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);   // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&s_tmem, 2 * TC_BN);   // two 128x256 fp32 accumulators (all 512 columns)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    if (lane == 0) {   // producer
      int it = 0;
      TileCursor cur;
      cur.init(a);
      for (int tile = blockIdx.x;; tile += gridDim.x) {
        const int mi = tile / nt, n0 = (tile % nt) * a.bn;
        if (!cur.seek(a, mi)) break;
        const int t0 = cur.t0(mi);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % TC_STAGES;
          if (it >= TC_STAGES) mbar_wait(&empty[s], ((it / TC_STAGES) - 1) & 1);
          uint8_t *sa = smem + s * (TC_TILE_A + TC_TILE_B), *sb = sa + TC_TILE_A;
          mbar_arrive_expect_tx(&full[s], stage_tx);
          tma_load_3d(sa, &map_x, kb * TC_BK, t0, cur.b, &full[s]);
          tma_load_2d(sb, &map_w, kb * TC_BK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      int it = 0, t = 0;
      TileCursor cur;
      cur.init(a);
      for (int tile = blockIdx.x;; tile += gridDim.x) {
        const int mi = tile / nt, n0 = (tile % nt) * a.bn, nw = min(a.bn, a.N - n0);
        if (!cur.seek(a, mi)) break;
        const int ab = t & 1;
        if (t >= 2) mbar_wait(&acc_empty[ab], ((t >> 1) - 1) & 1);   // the epilogue drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(ab * TC_BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % TC_STAGES;
          mbar_wait(&full[s], (it / TC_STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * (TC_TILE_A + TC_TILE_B)), sb = sa + TC_TILE_A;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)   // K = 16 per MMA: +32 bytes inside the swizzle atom
            umma_ss(acc, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), tc_idesc(nw), kb > 0 || k > 0);
          umma_commit(&empty[s]);   // the stage is free once these MMAs have read it
        }
        umma_commit(&acc_full[ab]);
        ++t;
      }
    }
  } else {
    // epilogue: warp w reads accumulator rows 32 (w % 4) .. + 31 (TMEM lane = row)
    const int qd = warp & 3;
    const bf16 *bias = (const bf16 *)a.bias, *bias2 = (const bf16 *)a.bias2;
    int t = 0;
    TileCursor cur;
    cur.init(a);
    for (int tile = blockIdx.x;; tile += gridDim.x) {
      const int mi = tile / nt, n0 = (tile % nt) * a.bn, nw = min(a.bn, a.N - n0);
      if (!cur.seek(a, mi)) break;
      const int ab = t & 1;
      mbar_wait(&acc_full[ab], (t >> 1) & 1);
      tc_fence_after();
      const int tr = cur.t0(mi) + qd * 32 + lane;   // row within segment cur.b
      const bool used = tr < cur.L;
      const int64_t row = (int64_t)cur.b * a.T + tr;
#pragma unroll 1
      for (int c0 = 0; c0 < nw; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ab * TC_BN + c0), r);
        tmem_wait_ld();
        if (used) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + c0 + j;
            float x = __uint_as_float(r[j]);
            if (bias) x += __bfloat162float(bias[n]);
            if (bias2) x += __bfloat162float(bias2[n]);
            v[j] = x;
          }
          OutT *y = (OutT *)a.Y + (int64_t)row * a.ldy + n0 + c0;
          if constexpr (sizeof(OutT) == 2) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint4 o;
              o.x = pack_bf16x2(v[j], v[j + 1]);
              o.y = pack_bf16x2(v[j + 2], v[j + 3]);
              o.z = pack_bf16x2(v[j + 4], v[j + 5]);
              o.w = pack_bf16x2(v[j + 6], v[j + 7]);
              *reinterpret_cast<uint4 *>(y + j) = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4 *>(y + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      ++t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * TC_BN);
}

}  // namespace ll
