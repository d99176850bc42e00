// tc_probe3.cu -- can several warps issue tcgen05.mma concurrently (separate
// accumulators) to beat the ~50-cycle single-thread issue interval?
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "../paper_2406_06220_b200/csrc/common.cuh"
using namespace ll;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)
__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// NW issuing warps (lane 0 of warps 0..NW-1), each NPER MMAs into its own D; M x N x 16.
template <int NW, int NPER, int M, int N, int TS>
__global__ void multi(long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
  if (tid == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t sa = smem_u32(sm), sb = sa + 80 * 1024;
  for (int rep = 0; rep < 4; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (warp < NW && lane == 0) {
#pragma unroll
      for (int i = 0; i < NPER; ++i) {
        const int kk = (warp * NPER + i) % 40;
        const uint64_t db = desc_ns(sb + kk * 256, 128, 2048);
        const uint32_t d = tmem + 320 + warp * N;
        if (TS) {
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(d), "r"(tmem + (uint32_t)(kk * 8)), "l"(db), "r"(idesc(M, N)), "r"((uint32_t)(i > 0)) : "memory");
        } else {
          const uint64_t da = desc_ns(sa + kk * 256, 128, 2048);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(d), "l"(da), "l"(db), "r"(idesc(M, N)), "r"((uint32_t)(i > 0)) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])) : "memory");
      mbar_wait(&bar[warp], rep & 1);
      long long t1 = clock64();
      if (rep == 3) cyc[warp] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
template <int NW, int NPER, int M, int N, int TS>
void run(const char *nm) {
  long long *d, h[8] = {};
  CK(cudaMalloc(&d, 64));
  CK(cudaMemset(d, 0, 64));
  CK(cudaFuncSetAttribute(multi<NW, NPER, M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  multi<NW, NPER, M, N, TS><<<1, 256, 200 * 1024>>>(d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost));
  long long mx = 0; for (int i = 0; i < NW; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s M=%3d N=%3d warps=%d mmas/warp=%2d : max %5lld cyc  (total mmas %d, %.1f cyc/mma)\n", nm, M, N, NW, NPER, mx,
         NW * NPER, (double)mx / (NW * NPER));
  cudaFree(d);
}
int main() {
  run<1, 40, 128, 32, 0>("SS");
  run<2, 20, 128, 32, 0>("SS");
  run<4, 10, 128, 32, 0>("SS");
  run<8, 5, 128, 32, 0>("SS");
  run<4, 10, 64, 40, 0>("SS");
  run<1, 40, 128, 8, 1>("TS");
  run<2, 20, 128, 8, 1>("TS");
  run<4, 10, 128, 8, 1>("TS");
  run<8, 5, 128, 8, 1>("TS");
  run<4, 10, 128, 32, 1>("TS");
  run<4, 40, 128, 8, 1>("TS");
  return 0;
}
