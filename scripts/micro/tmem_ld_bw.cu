// TMEM -> register read bandwidth per SM (tcgen05.ld.32x32b.x32), the path
// the prefill softmax reads S through.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2512_16391_b200/csrc scripts/micro/tmem_ld_bw.cu -o /tmp/tmem_bw && /tmp/tmem_bw
#include <cstdio>
#include "sm100.cuh"
using namespace kscd::sm100;

template <int COLS_PER_WAIT>
__global__ void tmem_bw(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t col0 = (warp >> 2) * 128 % 512;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < COLS_PER_WAIT / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(lane_base + ((col0 + c * 32) & 511), r);
      tmem_ld_wait();
      uint32_t x[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // 8 independent chains: the consumer never paces the loads
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i & 7] ^= r[i];
      acc += __uint_as_float((x[0] ^ x[1]) ^ (x[2] ^ x[3]) ^ ((x[4] ^ x[5]) ^ (x[6] ^ x[7])));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// all four 32-col loads in flight before one wait (the prefill softmax pattern)
__global__ void tmem_bw_batched(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t col0 = (warp >> 2) * 128 % 512;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[128];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(lane_base + col0 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[c * 32]));
    tmem_ld_wait();
    uint32_t x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 128; ++i) x[i & 7] ^= r[i];
    acc += __uint_as_float((x[0] ^ x[1]) ^ (x[2] ^ x[3]) ^ ((x[4] ^ x[5]) ^ (x[6] ^ x[7])));
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  const int iters = 2000;
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) tmem_bw<128><<<148, warps * 32>>>(iters, cyc, sink);
        else tmem_bw_batched<<<148, warps * 32>>>(iters, cyc, sink);
      }
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += h[i];
      mean /= 148;
      const double bytes = (double)iters * warps * 32 * 128 * 4;
      printf("warps=%2d %-26s %s: %.1f B/clk/SM (%.0f clk per warp-iteration of 16 KB)\n", warps,
             mode == 0 ? "ld x32 + wait, 4x" : "4 x ld x32, one wait", cudaGetErrorString(e), bytes / mean,
             mean / iters);
    }
  }
  return 0;
}
