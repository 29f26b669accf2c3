// Microbenchmark (dev tool): the HBM ceiling of the reuse-layer decode
// gather.  K and V caches [B][Hkv][n][128] bf16 (separate arrays, 2 GB each
// at the bench shape, far beyond L2); each (sequence, kv head) row list holds
// k sorted random positions (Top-k lists).  Plain coalesced 16-B loads, 16
// lanes per 256-B row, U rows per half-warp in flight, no shared memory and
// no math: the best random-row read rate this access pattern gets from HBM.
// Reports GB/s of K+V rows + index bytes (the decode sparse kernel's
// algorithmic bytes, B*Hkv*k*(512 + 4)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/micro/hbm_gather.cu -o /tmp/hg
//   /tmp/hg [B=8] [Hkv=8] [n=131072] [k=13107]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) gather_rows(const int4* __restrict__ kc, const int4* __restrict__ vc,
                                                   const int* __restrict__ idx, int lists, int k, long long n,
                                                   int4* sink, int rs) {
  const int half = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;   // one half-warp per row group
  const int nhalf = (gridDim.x * blockDim.x) >> 4;
  const int sub = threadIdx.x & 15;
  int4 acc = make_int4(0, 0, 0, 0);
  const long long total = (long long)lists * k;
  for (long long base = (long long)half * U; base < total; base += (long long)nhalf * U) {
    int4 kr[U], vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = base + u;
      if (e < total) {
        const long long list = e / k;
        const long long row = list * n + __ldg(idx + e);
        kr[u] = __ldcs(kc + row * rs + sub);
        vr[u] = __ldcs(vc + row * rs + sub);
      } else {
        kr[u] = vr[u] = make_int4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x ^= kr[u].x ^ vr[u].x;
      acc.y ^= kr[u].y ^ vr[u].y;
      acc.z ^= kr[u].z ^ vr[u].z;
      acc.w ^= kr[u].w ^ vr[u].w;
    }
  }
  if ((acc.x & acc.y & acc.z & acc.w) == 0x7fffffff) sink[0] = acc;   // never true; keeps the loads
}

template <int U>
static void run(const int4* kc, const int4* vc, const int* idx, int lists, int k, long long n, int4* sink, int grid,
                double bytes, int rs = 16) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(a);
    gather_rows<U><<<grid, 256>>>(kc, vc, idx, lists, k, n, sink, rs);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0) best = std::min(best, ms);
  }
  printf("U=%d grid=%d: %.1f us  %.0f GB/s  (%s)\n", U, grid, best * 1e3, bytes / best / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 8, H = argc > 2 ? atoi(argv[2]) : 8;
  const long long n = argc > 3 ? atoll(argv[3]) : 131072;
  const int k = argc > 4 ? atoi(argv[4]) : 13107;
  const int lists = B * H;
  const size_t cache = (size_t)lists * n * 256;
  int4 *kc, *vc, *sink;
  int* idx;
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
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)lists * k * (512 + 4);
  printf("lists=%d n=%lld k=%d cache=%.2f GB x2, algorithmic %.1f MB\n", lists, n, k, cache / 1e9, bytes / 1e6);
  for (int g : {sms * 4, sms * 8}) {
    run<1>(kc, vc, idx, lists, k, n, sink, g, bytes);
    run<2>(kc, vc, idx, lists, k, n, sink, g, bytes);
    run<4>(kc, vc, idx, lists, k, n, sink, g, bytes);
    run<8>(kc, vc, idx, lists, k, n, sink, g, bytes);
  }
  // interleaved layout: K and V rows of one position adjacent ([n][2][128]),
  // one 512-B contiguous read per selected key instead of two 256-B reads
  printf("interleaved K|V rows (one 512-B read per key):\n");
  {
    int4* kv;
    cudaMalloc(&kv, 2 * cache);
    cudaMemset(kv, 3, 2 * cache);
    for (int g : {sms * 4, sms * 8}) {
      run<2>(kv, kv + 16, idx, lists, k, n, sink, g, bytes, 32);
      run<4>(kv, kv + 16, idx, lists, k, n, sink, g, bytes, 32);
      run<8>(kv, kv + 16, idx, lists, k, n, sink, g, bytes, 32);
    }
    cudaFree(kv);
  }
  // sequential read of the same byte count for reference (contiguous rows)
  {
    std::vector<int> seq((size_t)lists * k);
    for (int l = 0; l < lists; ++l)
      for (int i = 0; i < k; ++i) seq[(size_t)l * k + i] = i;
    cudaMemcpy(idx, seq.data(), seq.size() * 4, cudaMemcpyHostToDevice);
    printf("contiguous rows:\n");
    run<4>(kc, vc, idx, lists, k, n, sink, sms * 8, bytes);
    run<8>(kc, vc, idx, lists, k, n, sink, sms * 8, bytes);
  }
  return 0;
}
