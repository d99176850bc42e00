// tc_probe.cu -- checks the tcgen05 operand layouts the decode kernel relies on
// (and times the small-N MMA chains it issues), on the B200 itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tcp tools/tc_probe.cu && /tmp/tcp
//
// 1. SS mode, M=64: A K-major 128-byte swizzle, B K-major no-swizzle with
//    (LBO, SBO) = (K-direction core-matrix stride, N-direction 8-row stride);
//    prints which TMEM lane holds D row m.
// 2. TS mode, M=128: A in TMEM (lane = row, two bf16 per 32-bit column).
// 3. TMA 3-D box {8 elems, 8 rows, 80 chunks} of a row-major [T, 640] bf16
//    matrix lands as [chunk][row][8 elems] (the no-swizzle K-major layout).
// 4. clock64 latency of MMA chains (issue -> commit mbarrier) for the shapes used.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#include "../paper_2406_06220_b200/csrc/common.cuh"
using namespace ll;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;   // layout type 0 = SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// A: [M][K] bf16 global, B: [N][K] bf16 global.  mode 0: SS (A sw128), 1: TS (A in TMEM).
// lbo/sbo: B descriptor fields.  Out: D[128][N] fp32 (all TMEM lanes), cyc.
__global__ void probe_mma(const bf16 *A, const bf16 *B, float *D, long long *cyc, int mode, int M, int N, int K,
                          uint32_t lbo_sel, int reps) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t *sa = sm;                                  // A sw128: K/64 chunks of [M rows][128 B]
  const int KC = K / 64;
  uint8_t *sb = sm + (size_t)KC * (M < 64 ? 64 : M) * 128;   // B no-swizzle [K/8][N][16 B] or [N/8][K/8][8][16B]
  // A -> sw128
  for (int i = tid; i < M * (K / 8); i += blockDim.x) {
    const int r = i / (K / 8), c = i % (K / 8);      // 16-B chunk c of row r
    const int kc = c / 8, cc = c % 8;
    uint4 v = *reinterpret_cast<const uint4 *>(A + (size_t)r * K + c * 8);
    *reinterpret_cast<uint4 *>(sa + (size_t)kc * M * 128 + (r / 8) * 1024 + (r % 8) * 128 + ((cc ^ (r % 8)) * 16)) = v;
  }
  // B -> no swizzle.  layout sel 0: (n,k) at (k/8)*(N*16) + n*16  [K-chunk major, N-groups contiguous]
  //                   layout sel 1: (n,k) at (n/8)*(K/8*128) + (k/8)*128 + (n%8)*16
  for (int i = tid; i < N * (K / 8); i += blockDim.x) {
    const int n = i / (K / 8), c = i % (K / 8);
    uint4 v = *reinterpret_cast<const uint4 *>(B + (size_t)n * K + c * 8);
    size_t off = (lbo_sel == 0 || lbo_sel == 2) ? (size_t)c * N * 16 + n * 16 : (size_t)(n / 8) * (K / 8) * 128 + c * 128 + (n % 8) * 16;
    *reinterpret_cast<uint4 *>(sb + off) = v;
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t dcol = 256;   // D at columns 256..
  if (mode == 1) {
    // A into TMEM columns 0 .. K/2-1: lane = row, column j = (k = 2j, 2j+1)
    const int row = warp * 32 + lane;
    for (int j0 = 0; j0 < K / 2; j0 += 16) {
      uint32_t r[16];
      for (int e = 0; e < 16; ++e) {
        const int k = 2 * (j0 + e);
        uint32_t lo = 0, hi = 0;
        if (row < M) {
          lo = *reinterpret_cast<const uint16_t *>(A + (size_t)row * K + k);
          hi = *reinterpret_cast<const uint16_t *>(A + (size_t)row * K + k + 1);
        }
        r[e] = lo | (hi << 16);
      }
      tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j0, r);
    }
    tmem_wait_st();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // B descriptor strides
  uint32_t LBO, SBO;
  if (lbo_sel == 0) { LBO = N * 16; SBO = 128; }                 // K-chunk stride N*16, 8-row group stride 128
  else if (lbo_sel == 1) { LBO = 128; SBO = (K / 8) * 128; }     // K-chunk stride 128, group stride K/8*128
  else if (lbo_sel == 2) { LBO = 128; SBO = N * 16; }            // swapped (wrong for sel 0) -> probe meaning
  else { LBO = (K / 8) * 128; SBO = 128; }                       // swapped for layout 1
  const uint32_t id = idesc(M, N);
  long long t0 = 0, t1 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    if (tid == 0) {
      t0 = clock64();
      for (int kk = 0; kk < K / 16; ++kk) {
        const uint32_t boff = (lbo_sel == 0 || lbo_sel == 2) ? (uint32_t)kk * 2 * N * 16 : (uint32_t)kk * 256;
        const uint64_t db = desc_ns(smem_u32(sb) + boff, LBO, SBO);
        if (mode == 0) {
          const uint64_t da = desc_sw128(smem_u32(sa) + (kk / 4) * M * 128 + (kk % 4) * 32);
          mma_ss(tmem + dcol, da, db, id, kk > 0);
        } else {
          mma_ts(tmem + dcol, tmem + (uint32_t)(kk * 8), db, id, kk > 0);
        }
      }
      commit(&bar);
      mbar_wait(&bar, rep & 1);
      t1 = clock64();
    }
  }
  __syncthreads();
  tc_fence_after();
  if (tid == 0) *cyc = t1 - t0;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + dcol + c0, r);
    tmem_wait_ld();
    for (int e = 0; e < 8; ++e) D[(size_t)(warp * 32 + lane) * N + c0 + e] = __uint_as_float(r[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// TMA 3-D box test
__global__ void probe_tma(const __grid_constant__ CUtensorMap map, bf16 *out, int t0) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    // poison
  }
  for (int i = threadIdx.x; i < 10240 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0xDEADBEEFu;
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 10240);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(sm)), "l"(&map), "r"(0), "r"(t0), "r"(0), "r"(smem_u32(&bar))
        : "memory");
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 5120; i += blockDim.x) out[i] = reinterpret_cast<bf16 *>(sm)[i];
}

static float bf(const bf16 &x) { return __bfloat162float(x); }

int main() {
  srand(1);
  const int MAXM = 128, MAXN = 64, MAXK = 640;
  std::vector<bf16> hA(MAXM * MAXK), hB(MAXN * MAXK);
  for (auto &x : hA) x = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (auto &x : hB) x = __float2bfloat16((rand() % 13 - 6) / 4.0f);
  bf16 *dA, *dB; float *dD; long long *dc;
  CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dD, 128 * MAXN * 4)); CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  struct Case { const char *name; int mode, M, N, K, sel; };
  Case cases[] = {
      {"SS M=64 N=40 K=64 B-sel0(LBO=N*16,SBO=128)", 0, 64, 40, 64, 0},
      {"SS M=64 N=40 K=64 B-sel2(LBO=128,SBO=N*16)", 0, 64, 40, 64, 2},
      {"SS M=64 N=40 K=64 B-sel1(LBO=128,SBO=K/8*128)", 0, 64, 40, 64, 1},
      {"SS M=64 N=40 K=64 B-sel3(LBO=K/8*128,SBO=128)", 0, 64, 40, 64, 3},
      {"SS M=128 N=40 K=64 sel1", 0, 128, 40, 64, 1},
      {"TS M=128 N=8 K=64 sel1", 1, 128, 8, 64, 1},
      {"TS M=128 N=32 K=64 sel1", 1, 128, 32, 64, 1},
      {"TS M=128 N=8 K=64 sel3", 1, 128, 8, 64, 3},
      {"SS M=64 N=40 K=640 sel1", 0, 64, 40, 640, 1},
      {"SS M=64 N=32 K=640 sel1", 0, 64, 32, 640, 1},
      {"SS M=64 N=64 K=640 sel1", 0, 64, 64, 640, 1},
      {"SS M=64 N=8 K=640 sel1", 0, 64, 8, 640, 1},
      {"SS M=128 N=40 K=640 sel1", 0, 128, 40, 640, 1},
      {"TS M=128 N=8 K=640 sel1", 1, 128, 8, 640, 1},
      {"TS M=128 N=16 K=640 sel1", 1, 128, 16, 640, 1},
      {"TS M=128 N=32 K=160 sel1", 1, 128, 32, 160, 1},
      {"TS M=128 N=40 K=640 sel1", 1, 128, 40, 640, 1},
  };
  for (const Case &c : cases) {
    CK(cudaMemset(dD, 0, 128 * MAXN * 4));
    probe_mma<<<1, 128, 220 * 1024>>>(dA, dB, dD, dc, c.mode, c.M, c.N, c.K, c.sel, 4);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(128 * c.N);
    long long cyc;
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    // reference rows; find the lane of each row
    int ok_rows = 0;
    std::vector<int> lane_of(c.M, -1);
    for (int m = 0; m < c.M; ++m) {
      std::vector<double> ref(c.N);
      for (int n = 0; n < c.N; ++n) {
        double s = 0;
        for (int k = 0; k < c.K; ++k) s += (double)bf(hA[m * c.K + k]) * bf(hB[n * c.K + k]);
        ref[n] = s;
      }
      for (int l = 0; l < 128; ++l) {
        double err = 0;
        for (int n = 0; n < c.N; ++n) err = fmax(err, fabs(D[l * c.N + n] - ref[n]));
        if (err < 1e-3) { lane_of[m] = l; break; }
      }
      if (lane_of[m] >= 0) ++ok_rows;
    }
    printf("%-48s rows matched %3d/%3d  chain %5lld cyc  lanes:", c.name, ok_rows, c.M, cyc);
    for (int m = 0; m < c.M; m += (c.M > 64 ? 16 : 4)) printf(" %d->%d", m, lane_of[m]);
    printf("\n");
  }
  // TMA 3-D
  {
    const int T = 20;
    std::vector<bf16> f(T * 640);
    for (int i = 0; i < T * 640; ++i) f[i] = __float2bfloat16((float)(i % 997));
    bf16 *df, *dout;
    CK(cudaMalloc(&df, f.size() * 2)); CK(cudaMalloc(&dout, 5120 * 2));
    CK(cudaMemcpy(df, f.data(), f.size() * 2, cudaMemcpyHostToDevice));
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap map;
    const cuuint64_t dims[3] = {8, (cuuint64_t)T, 80};
    const cuuint64_t strides[2] = {1280, 16};
    const cuuint32_t box[3] = {8, 8, 80};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, df, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("TMA 3-D encode: %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
      CK(cudaFuncSetAttribute(probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 1024));
      for (int t0 : {3, 15}) {
        probe_tma<<<1, 128, 12 * 1024>>>(map, dout, t0);
        CK(cudaDeviceSynchronize());
        std::vector<bf16> o(5120);
        CK(cudaMemcpy(o.data(), dout, 5120 * 2, cudaMemcpyDeviceToHost));
        int bad = 0, zeros = 0;
        for (int c = 0; c < 80; ++c)
          for (int rr = 0; rr < 8; ++rr)
            for (int e = 0; e < 8; ++e) {
              const float got = bf(o[(c * 8 + rr) * 8 + e]);
              const int t = t0 + rr;
              const float want = t < T ? bf(f[t * 640 + c * 8 + e]) : 0.f;
              if (got != want) ++bad;
              if (t >= T && got == 0.f) ++zeros;
            }
        printf("TMA 3-D box t0=%d: mismatches %d (OOB zero-filled elems %d)\n", t0, bad, zeros);
      }
    }
  }
  return 0;
}
