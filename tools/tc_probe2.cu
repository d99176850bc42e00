// tc_probe2.cu -- tcgen05.mma issue/latency behaviour for small N (B200):
// dependent chains vs independent accumulators, per-instruction cost vs N.
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
// nmma MMAs split over nchain accumulators (round robin), M x N x 16 each, A and B no-swizzle in smem
template <int NMMA, int NCH, int M, int N, int TS>
__global__ void chain(long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t sa = smem_u32(sm), sb = sa + 96 * 1024;
  long long t0 = 0, t1 = 0;
  for (int rep = 0; rep < 4; ++rep) {
    __syncthreads();
    if (tid == 0) {
      t0 = clock64();
#pragma unroll
      for (int i = 0; i < NMMA; ++i) {
        const int ch = i % NCH, kk = i / NCH;
        const uint64_t db = desc_ns(sb + kk * 256, 128, (N / 8 > 1 ? 2048 : 128));
        const uint32_t d = tmem + 256 + ch * N;
        if (TS) {
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(d), "r"(tmem + (uint32_t)((kk * 8) & 255)), "l"(db), "r"(idesc(M, N)), "r"((uint32_t)(kk > 0)) : "memory");
        } else {
          const uint64_t da = desc_ns(sa + kk * 256, 128, 2048);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(d), "l"(da), "l"(db), "r"(idesc(M, N)), "r"((uint32_t)(kk > 0)) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      const long long ti = clock64();
      mbar_wait(&bar, rep & 1);
      t1 = clock64();
      if (rep == 3) { cyc[0] = t1 - t0; cyc[1] = ti - t0; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
template <int NMMA, int NCH, int M, int N, int TS>
void run(const char *nm) {
  long long *d, h[2];
  CK(cudaMalloc(&d, 16));
  CK(cudaFuncSetAttribute(chain<NMMA, NCH, M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  chain<NMMA, NCH, M, N, TS><<<1, 128, 200 * 1024>>>(d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  printf("%-6s M=%3d N=%3d mmas=%3d chains=%d : total %6lld cyc (issue %5lld)  per mma %.1f\n", nm, M, N, NMMA, NCH, h[0], h[1],
         (double)h[0] / NMMA);
  cudaFree(d);
}
int main() {
  run<1, 1, 128, 32, 0>("SS");
  run<2, 1, 128, 32, 0>("SS");
  run<4, 1, 128, 32, 0>("SS");
  run<8, 1, 128, 32, 0>("SS");
  run<16, 1, 128, 32, 0>("SS");
  run<40, 1, 128, 32, 0>("SS");
  run<40, 2, 128, 32, 0>("SS");
  run<40, 4, 128, 32, 0>("SS");
  run<40, 8, 128, 32, 0>("SS");
  run<40, 1, 64, 32, 0>("SS");
  run<40, 1, 128, 8, 0>("SS");
  run<40, 1, 128, 64, 0>("SS");
  run<40, 1, 128, 128, 0>("SS");
  run<40, 1, 128, 256, 0>("SS");
  run<40, 4, 128, 64, 0>("SS");
  run<40, 1, 128, 8, 1>("TS");
  run<40, 4, 128, 8, 1>("TS");
  run<40, 1, 128, 32, 1>("TS");
  run<40, 4, 128, 32, 1>("TS");
  run<40, 1, 128, 256, 1>("TS");
  run<160, 4, 128, 256, 0>("SS");
  return 0;
}
