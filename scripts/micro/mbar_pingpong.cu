// mbarrier handoff latency between two warps of a CTA (the softmax <-> MMA
// handoffs of the prefill pipeline): warp 0 arrives on A and waits on B,
// warp 1 waits on A and arrives on B.  Variants: try_wait (default suspend),
// test_wait spin.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_16391_b200/csrc
#include <cstdio>
#include "sm100.cuh"
using namespace kscd;
using namespace kscd::sm100;

__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

template <int MODE>
__global__ void pingpong(int iters, long long* out, int nthreads_arrive) {
  __shared__ uint64_t bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], nthreads_arrive);
    mbar_init(&bars[1], nthreads_arrive);
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const bool all = nthreads_arrive == 32;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (warp == 0) {
      if (all || (threadIdx.x & 31) == 0) mbar_arrive(&bars[0]);
      if (MODE == 0) mbar_wait(&bars[1], i & 1);
      else while (!test_wait(&bars[1], i & 1)) {}
    } else if (warp == 1) {
      if (MODE == 0) mbar_wait(&bars[0], i & 1);
      else while (!test_wait(&bars[0], i & 1)) {}
      if (all || (threadIdx.x & 31) == 0) mbar_arrive(&bars[1]);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (int arr : {1, 32}) {
    for (int mode = 0; mode < 2; ++mode) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) pingpong<0><<<1, 64>>>(20000, d, arr);
        else pingpong<1><<<1, 64>>>(20000, d, arr);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-10s arrivals/phase=%2d: %lld clk per round trip (2 handoffs)\n", mode == 0 ? "try_wait" : "test_wait", arr, h);
    }
  }
  return 0;
}
