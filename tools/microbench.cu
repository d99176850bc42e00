// microbench.cu -- latency / throughput of the primitives the decode kernel is built from,
// measured on the B200 itself (clock64 cycles).  Build + run on a GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2406_06220_b200/csrc/common.cuh"
using namespace ll;

__global__ void hmma_latency(float *out, long long *cyc, int n) {
  float d[4] = {0, 0, 0, 0};
  uint32_t a = 0x3f803f80u, b = 0x3f803f80u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) mma_bf16_16816(d, a, a, a, a, b, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x * blockDim.x / 32 + threadIdx.x / 32] = t1 - t0;
  out[threadIdx.x] = d[0] + d[1] + d[2] + d[3];
}

template <int CH>
__global__ void hmma_tput(float *out, long long *cyc, int n) {
  float d[CH][4] = {};
  uint32_t a = 0x3f803f80u, b = 0x3f803f80u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) mma_bf16_16816(d[c], a, a, a, a, b, b);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void lds_latency(long long *cyc, int n) {
  __shared__ uint32_t buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
  __syncthreads();
  uint32_t idx = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = buf[idx];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (idx == 12345) cyc[1] = idx;
}

__global__ void syncthreads_cost(long long *cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// cluster: ping-pong between rank 0 and rank r via st.async + mbarrier
__global__ void __cluster_dims__(16, 1, 1) dsmem_pingpong(long long *cyc, int n) {
  __shared__ __align__(8) uint64_t bar[1];
  __shared__ __align__(16) uint64_t slot[2];
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync_all();
  const uint32_t peer = (rank == 0) ? 15 : 0;
  uint32_t ph = 0;
  long long t0 = clock64();
  if (threadIdx.x == 0 && (rank == 0 || rank == 15)) {
    for (int i = 0; i < n; ++i) {
      mbar_arrive_expect_tx(bar, 16);
      if (rank == 0) {
        st_async_u64x2(mapa_u32(smem_u32(slot), peer), i, i, mapa_u32(smem_u32(bar), peer));
        mbar_wait(bar, ph);
      } else {
        mbar_wait(bar, ph);
        st_async_u64x2(mapa_u32(smem_u32(slot), peer), i, i, mapa_u32(smem_u32(bar), peer));
      }
      ph ^= 1;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) cyc[0] = t1 - t0;
  cluster_sync_all();
}

__global__ void __cluster_dims__(16, 1, 1) cluster_barrier_cost(long long *cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) cluster_sync_all();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cluster_rank() == 0) cyc[0] = t1 - t0;
}

__global__ void bulk_latency(const uint8_t *src, long long *cyc, int n, int bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[1];
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(sm, src + (size_t)(i % 64) * bytes, bytes, bar);
      mbar_wait(bar, ph);
      ph ^= 1;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void ldg_latency(const uint32_t *src, long long *cyc, int n) {
  uint32_t idx = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = __ldcg(src + idx);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (idx == 0xFFFFFFFF) cyc[1] = 1;
}

int main1() {
  float *out;
  long long *cyc, h[64];
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 4096);
  const int N = 4096;
  hmma_latency<<<1, 32>>>(out, cyc, N);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("HMMA m16n8k16 bf16 dependent latency: %.1f cycles\n", (double)h[0] / N);
  for (int warps : {1, 4, 8, 16}) {
    hmma_tput<4><<<1, 32 * warps>>>(out, cyc, N);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)h[0] / (N * 4.0 * warps);
    printf("HMMA throughput, %2d warps x 4 chains: %.2f cycles/HMMA/SM -> %.0f MAC/clk/SM\n", warps, per,
           2048.0 / per);
  }
  lds_latency<<<1, 32>>>(cyc, N);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.1f cycles\n", (double)h[0] / N);
  syncthreads_cost<<<1, 288>>>(cyc, N);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (288 thr): %.1f cycles\n", (double)h[0] / N);
  dsmem_pingpong<<<16, 32>>>(cyc, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("st.async+mbarrier ping-pong round trip (rank0<->15): %.1f cycles (%s)\n", (double)h[0] / 1000,
         cudaGetErrorString(e));
  cluster_barrier_cost<<<16, 288>>>(cyc, 1000);
  e = cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("barrier.cluster (16 CTAs x 288 thr): %.1f cycles (%s)\n", (double)h[0] / 1000, cudaGetErrorString(e));
  uint8_t *src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0, 64 << 20);
  for (int bytes : {1280, 10240, 40960}) {
    cudaFuncSetAttribute(bulk_latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
    bulk_latency<<<1, 32, 64 << 10>>>(src, cyc, 200, bytes);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("bulk copy %6d B L2->smem + mbarrier: %.1f cycles\n", bytes, (double)h[0] / 200);
  }
  uint32_t *chain;
  cudaMalloc(&chain, 4 << 20);
  uint32_t *hc = (uint32_t *)malloc(4 << 20);
  for (int i = 0; i < (1 << 20); ++i) hc[i] = (uint32_t)((i * 4099 + 97) & ((1 << 20) - 1)) & ~31u;
  cudaMemcpy(chain, hc, 4 << 20, cudaMemcpyHostToDevice);
  ldg_latency<<<1, 1>>>(chain, cyc, 2000);
  ldg_latency<<<1, 1>>>(chain, cyc, 2000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDG.cg dependent latency (4 MB chain, L2): %.1f cycles\n", (double)h[0] / 2000);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}

// ---------------------------------------------------------------------------
// joint-style MMA loop in isolation: W fragments in registers (20 x uint4),
// A (32 rows x 640) from smem with the decode kernel's padded stride.
// ---------------------------------------------------------------------------
template <int MT>
__global__ void joint_loop(long long *cyc, float *out, int iters, int spin_warp) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ volatile int flag;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int zstride = 1344;
  for (int i = threadIdx.x; i < 32 * zstride / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0x3f803f80u ^ i;
  if (threadIdx.x == 0) flag = 0;
  uint4 wreg[20];
#pragma unroll
  for (int k = 0; k < 20; ++k) wreg[k] = make_uint4(0x3f80u + k, lane, warp, k);
  __syncthreads();
  if (spin_warp && warp == blockDim.x / 32 - 1) {
    // a warp spinning on a volatile smem flag, like an idle producer
    while (flag == 0) {
    }
    return;
  }
  float acc[2][2][4] = {};
  const uint8_t *a0 = sm + g * zstride + q * 16, *a1 = a0 + 8 * zstride, *a2 = a0 + 16 * zstride, *a3 = a0 + 24 * zstride;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kb = 0; kb < 20; ++kb) {
      const uint4 b = wreg[kb];
      const uint4 x0 = lds128(a0 + kb * 64), x1 = lds128(a1 + kb * 64);
      mma_bf16_16816(acc[0][kb & 1], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
      mma_bf16_16816(acc[0][kb & 1], x0.z, x1.z, x0.w, x1.w, b.z, b.w);
      if (MT > 1) {
        const uint4 x2 = lds128(a2 + kb * 64), x3 = lds128(a3 + kb * 64);
        mma_bf16_16816(acc[1][kb & 1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
        mma_bf16_16816(acc[1][kb & 1], x2.z, x3.z, x2.w, x3.w, b.z, b.w);
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  float s = 0;
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 2; ++c)
      for (int e = 0; e < 4; ++e) s += acc[a][c][e];
  out[threadIdx.x] = s;
  if (lane == 0) cyc[warp] = t1 - t0;
  if (threadIdx.x == 0) flag = 1;
}

int main2() {
  float *out;
  long long *cyc, h[64];
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 4096);
  cudaFuncSetAttribute(joint_loop<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(joint_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  for (int warps : {1, 9}) {
    for (int spin : {0, 1}) {
      const int nthr = (warps + spin) * 32;
      joint_loop<2><<<1, nthr, 64 << 10>>>(cyc, out, 100, spin);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 8 * warps, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      printf("joint loop MT=2 (80 HMMA + 80 LDS.128): %d warps%s: %.0f cycles/iter (max warp)\n", warps,
             spin ? " + 1 spinning warp" : "", (double)mx / 100);
    }
    joint_loop<1><<<1, warps * 32, 64 << 10>>>(cyc, out, 100, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * warps, cudaMemcpyDeviceToHost);
    printf("joint loop MT=1 (40 HMMA + 40 LDS.128): %d warps: %.0f cycles/iter\n", warps, (double)h[0] / 100);
  }
  return 0;
}


// many outstanding bulk copies: n copies of `bytes` from rows `stride` apart, one mbarrier
__global__ void bulk_multi(const uint8_t *src, long long *cyc, int reps, int ncopies, int bytes, int stride) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[1];
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, ncopies * bytes);
    __syncwarp();
    for (int i = threadIdx.x; i < ncopies; i += 32)
      bulk_g2s(sm + (size_t)i * bytes, src + (size_t)((r * 7 + i) % 512) * stride, bytes, bar);
    mbar_wait(bar, ph);
    ph ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main3() {
  long long *cyc, h[8];
  cudaMalloc(&cyc, 4096);
  uint8_t *src;
  cudaMalloc(&src, 256 << 20);
  cudaMemset(src, 1, 256 << 20);
  cudaFuncSetAttribute(bulk_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  struct { int n, bytes, stride; } cs[] = {{1, 1280, 1280 * 640}, {8, 1280, 1280 * 640}, {40, 1280, 1280 * 640},
                                           {80, 1280, 1280 * 640}, {1, 10240, 10240}, {8, 10240, 10240},
                                           {1, 40960, 40960}, {4, 40960, 40960}};
  for (auto c : cs) {
    bulk_multi<<<1, 32, 200 << 10>>>(src, cyc, 50, c.n, c.bytes, c.stride);  // warm L2
    bulk_multi<<<1, 32, 200 << 10>>>(src, cyc, 200, c.n, c.bytes, c.stride);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / 200;
    printf("bulk %3d x %6d B (stride %7d): %7.0f cycles per batch, %6.1f B/cycle (%s)\n", c.n, c.bytes, c.stride, per,
           c.n * c.bytes / per, cudaGetErrorString(e));
  }
  return 0;
}



// TMEM -> register load bandwidth: every warp reads `cols` columns of its lane quarter
__global__ void tmem_bw(long long *cyc, float *out, int iters, int cols) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&taddr_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
  if (warp < 4)
    for (int c = 0; c < 512; c += 16) tmem_st16(base + c, r);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < cols; c += 16) {
      tmem_ld16(base + ((c + it * 16) & 511), r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += r[i];
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = (float)acc;
  if ((threadIdx.x & 31) == 0) cyc[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(taddr_s, 512);
}

int main4() {
  long long *cyc, h[32];
  float *out;
  cudaMalloc(&cyc, 4096);
  cudaMalloc(&out, 1 << 20);
  for (int warps : {1, 4, 8, 10}) {
    tmem_bw<<<1, 32 * warps>>>(cyc, out, 100, 80);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * warps, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = 100.0 * 80 * 32 * 4 * warps;
    printf("tcgen05.ld 32x32b.x16 (wait each), %2d warps x 80 cols: %.0f cycles/iter, %.0f B/cycle/SM (%s)\n", warps,
           (double)mx / 100, bytes / mx, cudaGetErrorString(e));
  }
  return 0;
}

int main(int argc, char **argv) {
  if (argc > 1 && argv[1][0] == '3') return main3();
  if (argc > 1 && argv[1][0] == '4') return main4();
  if (argc > 1) return main2();
  return main1();
}
