// Microbenchmark (dev tool): the reuse-layer decode gather with 1-D bulk
// copies (cp.async.bulk global -> shared, 256 B per K / V row, completion on
// an mbarrier) instead of 16-B cp.async / LDG per lane.  Same workload as
// hbm_gather.cu: B*Hkv lists of k sorted random rows of K and V caches
// [B][Hkv][n][128] bf16; reports GB/s of K+V rows + index bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_16391_b200/csrc \
//     scripts/micro/bulk_gather.cu -o /tmp/bg && /tmp/bg
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "sm100.cuh"
using namespace kscd;
using namespace kscd::sm100;

constexpr int kEnt = 32;                 // entries (K row + V row) per stage
constexpr int kStageBytes = kEnt * 512;  // 16 KB

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int S>
__global__ void __launch_bounds__(160) bulk_gather(const char* kc, const char* vc, const int* idx, int lists, int k,
                                                   long long n, int per, int* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * kStageBytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long total = (long long)lists * k;
  const long long e0 = (long long)blockIdx.x * per, e1 = min(total, e0 + per);
  const int nst = (int)((e1 - e0 + kEnt - 1) / kEnt);
  if (warp == 0) {
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      const long long e = e0 + (long long)i * kEnt + lane;
      const int cnt = (int)min((long long)kEnt, e1 - (e0 + (long long)i * kEnt));
      if (lane == 0) mbar_expect_tx(&full[s], cnt * 512);
      __syncwarp();
      if (lane < cnt) {
        const long long list = e / k;
        const long long row = list * n + __ldg(idx + e);
        const uint32_t dst = smem_u32(sm + s * kStageBytes + lane * 512);
        bulk_g2s(dst, kc + row * 256, 256, &full[s]);
        bulk_g2s(dst + 256, vc + row * 256, 256, &full[s]);
      }
    }
  } else {
    int acc = 0;
    const int c = warp - 1;
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      acc ^= reinterpret_cast<const int*>(sm + s * kStageBytes)[c * 1024 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

template <int S>
static void run(const char* kc, const char* vc, const int* idx, int lists, int k, long long n, int* sink, int grid,
                double bytes) {
  const long long total = (long long)lists * k;
  const int per = (int)((total + grid - 1) / grid);
  const int smem = S * kStageBytes + 2 * S * 8;
  cudaFuncSetAttribute(bulk_gather<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(a);
    bulk_gather<S><<<grid, 160, smem>>>(kc, vc, idx, lists, k, n, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0) best = std::min(best, ms);
  }
  printf("stages=%d (%d KB) grid=%d: %.1f us  %.0f GB/s  (%s)\n", S, smem / 1024, grid, best * 1e3, bytes / best / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int B = 8, H = 8, k = 13107;
  const long long n = 131072;
  const int lists = B * H;
  const size_t cache = (size_t)lists * n * 256;
  char *kc, *vc;
  int *idx, *sink;
  cudaMalloc(&kc, cache);
  cudaMalloc(&vc, cache);
  cudaMemset(kc, 1, cache);
  cudaMemset(vc, 2, cache);
  cudaMalloc(&sink, 16);
  std::vector<int> h((size_t)lists * k);
  std::mt19937 rng(7);
  std::vector<int> perm(n);
  for (int l = 0; l < lists; ++l) {
    for (long long i = 0; i < n; ++i) perm[i] = (int)i;
    for (int i = 0; i < k; ++i) std::swap(perm[i], perm[i + rng() % (n - i)]);
    std::sort(perm.begin(), perm.begin() + k);
    std::copy(perm.begin(), perm.begin() + k, h.begin() + (size_t)l * k);
  }
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const double bytes = (double)lists * k * (512 + 4);
  printf("lists=%d n=%lld k=%d, algorithmic %.1f MB\n", lists, n, k, bytes / 1e6);
  for (int g : {148, 296, 592}) {
    run<4>(kc, vc, idx, lists, k, n, sink, g, bytes);
    run<8>(kc, vc, idx, lists, k, n, sink, g, bytes);
    run<12>(kc, vc, idx, lists, k, n, sink, g, bytes);
  }
  return 0;
}
