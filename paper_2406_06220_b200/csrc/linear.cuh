// linear.cuh -- Y[M,N] = X[M,K] . W[N,K]^T + bias[N] (+ bias2[N]).
//
// Used for the precomputed projections of PAPER.md §3.4 (:216-222):
//   * encoder projection f = W_enc enc + b_enc over all B*T_max frames
//     (Alg. 3 line 2, :134) -- the dominant GEMM of a call;
//   * model tables that turn per-step predictor work into lookups:
//     LSTM input part  E'[v] = W_ih Emb[v] + b_ih + b_hh       [V+1, 4P]
//     stateless        G_k[v] = W_pred[:, k-slice] Emb_k[v] (+ b_pred, k=0) [V+1, H]
//
// bf16 path: 128x64x32 CTA tiles, 8 warps (each 32x32 = 2 m16 x 4 n8
// mma.sync tiles), cp.async double buffering, K permuted per 32-block as in
// common.cuh so every fragment is one 16-byte shared load.
// f32 path: SIMT 64x64 tiles, 4x4 per thread, fp32 accumulation.
#pragma once
#include "common.cuh"

namespace ll {

struct LinearArgs {
  const void *X;
  int64_t ldx;
  const void *W;
  int64_t ldw;
  const void *bias;   // [N] in input dtype, or nullptr
  const void *bias2;  // [N] in input dtype, or nullptr
  void *Y;
  int64_t ldy;
  int M, N, K;
};

constexpr int LB_M = 128, LB_N = 64, LB_K = 32;
constexpr int LB_STRIDE = LB_K * 2;  // 64 B per smem row (== 64 mod 128: conflict-free LDS.128)

template <typename OutT>
__global__ void __launch_bounds__(256) linear_bf16_kernel(LinearArgs a) {
  __shared__ __align__(16) uint8_t xs[2][LB_M * LB_STRIDE];
  __shared__ __align__(16) uint8_t wsm[2][LB_N * LB_STRIDE];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * LB_M, n0 = blockIdx.x * LB_N;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const bf16 *X = (const bf16 *)a.X, *W = (const bf16 *)a.W;
  const int nk = (a.K + LB_K - 1) / LB_K;

  auto load_stage = [&](int stage, int kb) {
    const int k0 = kb * LB_K;
    // X tile: 128 rows x 4 chunks of 16 B = 512 chunks, 2 per thread
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      int idx = tid + c * 256, r = idx >> 2, ch = idx & 3;
      int gm = m0 + r, gk = k0 + ch * 8;
      void *dst = xs[stage] + r * LB_STRIDE + ch * 16;
      if (gm < a.M && gk < a.K)
        cp_async16(dst, X + (int64_t)gm * a.ldx + gk);
      else
        *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
    }
    {
      int r = tid >> 2, ch = tid & 3;
      int gn = n0 + r, gk = k0 + ch * 8;
      void *dst = wsm[stage] + r * LB_STRIDE + ch * 16;
      if (gn < a.N && gk < a.K)
        cp_async16(dst, W + (int64_t)gn * a.ldw + gk);
      else
        *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
    }
    cp_async_commit();
  };

  float acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;

  const int g = lane >> 2, q = lane & 3;
  load_stage(0, 0);
  for (int kb = 0; kb < nk; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nk) {
      load_stage(st ^ 1, kb + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    uint4 af[2][2], bfr[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      af[i][0] = lds128(xs[st] + (wm + i * 16 + g) * LB_STRIDE + q * 16);
      af[i][1] = lds128(xs[st] + (wm + i * 16 + g + 8) * LB_STRIDE + q * 16);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) bfr[j] = lds128(wsm[st] + (wn + j * 8 + g) * LB_STRIDE + q * 16);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        mma_bf16_16816(acc[i][j], af[i][0].x, af[i][1].x, af[i][0].y, af[i][1].y, bfr[j].x, bfr[j].y);
        mma_bf16_16816(acc[i][j], af[i][0].z, af[i][1].z, af[i][0].w, af[i][1].w, bfr[j].z, bfr[j].w);
      }
    __syncthreads();
  }
  const bf16 *b1 = (const bf16 *)a.bias, *b2 = (const bf16 *)a.bias2;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int r = m0 + wm + i * 16 + g + (e >= 2 ? 8 : 0);
        int c = n0 + wn + j * 8 + 2 * q + (e & 1);
        if (r < a.M && c < a.N) {
          float v = acc[i][j][e];
          if (b1) v += __bfloat162float(b1[c]);
          if (b2) v += __bfloat162float(b2[c]);
          OutT *Y = (OutT *)a.Y;
          if constexpr (sizeof(OutT) == 2)
            Y[(int64_t)r * a.ldy + c] = __float2bfloat16_rn(v);
          else
            Y[(int64_t)r * a.ldy + c] = v;
        }
      }
}

// fp32 SIMT path (LL_F32): 64x64 tile, 256 threads, 4x4 outputs per thread.
__global__ void __launch_bounds__(256) linear_f32_kernel(LinearArgs a) {
  __shared__ float xs[16][64 + 4];
  __shared__ float ws[16][64 + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const float *X = (const float *)a.X, *W = (const float *)a.W;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += 16) {
    for (int idx = tid; idx < 64 * 16; idx += 256) {
      int r = idx >> 4, kk = idx & 15;
      int gm = m0 + r, gn = n0 + r, gk = k0 + kk;
      xs[kk][r] = (gm < a.M && gk < a.K) ? X[(int64_t)gm * a.ldx + gk] : 0.f;
      ws[kk][r] = (gn < a.N && gk < a.K) ? W[(int64_t)gn * a.ldw + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const float *b1 = (const float *)a.bias, *b2 = (const float *)a.bias2;
  float *Y = (float *)a.Y;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      if (r < a.M && c < a.N) {
        float v = acc[i][j];
        if (b1) v += b1[c];
        if (b2) v += b2[c];
        Y[(int64_t)r * a.ldy + c] = v;
      }
    }
}

}  // namespace ll
