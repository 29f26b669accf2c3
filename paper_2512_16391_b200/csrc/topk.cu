// Post-softmax pooling for decode tiles and exact Top-k selection.
//
// pool_decode:  pooled[b][g][j] = sum_{h in group g} exp(s[b][h][j] - lse[b][h])
//               -- _post_pooled for a one-row decode tile (runner.py:148-152)
//               up to the constant 1/G, which does not change the ranking.
// topk:         oracle_topk_indices (attention.py:147-174): the k largest
//               values of a row, ties to the SMALLER index, emitted in
//               ascending index order.  Radix select on order-preserving
//               uint32 keys (12 + 12 + 8 bits) finds the exact k-th key T;
//               one ordered compaction pass then keeps every key > T and the
//               (k - #>T) lowest-index keys == T.
//
// A row is split over a thread-block cluster of CL CTAs (CL = 4 when there
// are few rows, as in decode where rows = batch x kv heads): each CTA
// histograms its segment with shared-memory atomics, the cluster reduces the
// histograms through distributed shared memory, and the compaction offsets
// of the segments are exchanged the same way.  HBM/L2-bound integer work; no
// tensor cores.  The first radix pass is shared-atomic bound (~0.5 atomic /
// clk / SM), which is why splitting a row across SMs pays.
#include <stdlib.h>

#include "kscd_internal.h"
#include "topk_select.cuh"

namespace kscd {

constexpr int kPoolThreads = 256;
constexpr int kPoolKeysPerThread = 4;

__global__ void __launch_bounds__(kPoolThreads) pool_decode_kernel(const PoolDecodeArgs a) {
  const int g = blockIdx.y, b = blockIdx.z;
  const int j0 = (blockIdx.x * kPoolThreads + threadIdx.x) * kPoolKeysPerThread;
  if (j0 >= a.n) return;
  float acc[kPoolKeysPerThread] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < a.G; ++i) {
    const int64_t h = (int64_t)b * a.Hq + (int64_t)g * a.G + i;
    const float lse2 = __ldg(a.lse + h) * kLog2e;
    const float* s = a.scores + h * a.score_stride + j0;
    if (j0 + kPoolKeysPerThread <= a.n) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(s));
      acc[0] += exp2f(v.x - lse2);
      acc[1] += exp2f(v.y - lse2);
      acc[2] += exp2f(v.z - lse2);
      acc[3] += exp2f(v.w - lse2);
    } else {
      for (int c = 0; c < kPoolKeysPerThread && j0 + c < a.n; ++c) acc[c] += exp2f(s[c] - lse2);
    }
  }
  float* out = a.pooled + ((int64_t)b * a.Hkv + g) * a.pool_stride + j0;
  if (j0 + kPoolKeysPerThread <= a.n) {
    *reinterpret_cast<float4*>(out) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  } else {
    for (int c = 0; c < kPoolKeysPerThread && j0 + c < a.n; ++c) out[c] = acc[c];
  }
}

cudaError_t launch_pool_decode(const PoolDecodeArgs& a, cudaStream_t st) {
  const int per_block = kPoolThreads * kPoolKeysPerThread;
  dim3 grid((a.n + per_block - 1) / per_block, a.Hkv, a.B);
  pool_decode_kernel<<<grid, kPoolThreads, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Top-k
template <int CL>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const TopkArgs a) {
  __shared__ TopkShared sh;
  const int r = blockIdx.x / CL;
  int n = a.lens ? a.lens[r] : a.len;
  int k = a.ks ? a.ks[r] : a.k;
  if (a.seq_div > 0) {
    // ragged decode batch: this row's sequence length and its k_budget
    n = min(a.len, __ldg(a.seq_lens + r / a.seq_div));
    k = k_budget_dev(a.fraction, a.k_min, n);
  } else if (a.tile > 0) {
    // k_budget (tiles.py:81-89) of the tile's causal bound, in the same fp64
    n = min(a.len, a.tile * (r % a.T + 1));
    k = k_budget_dev(a.fraction, a.k_min, n);
  }
  const int take = n < k ? n : k;
  topk_select<CL, kTopkThreads>(a.vals + (int64_t)r * a.val_stride,
                                a.vals2 ? a.vals2 + (int64_t)r * a.val_stride : nullptr, n, take,
                                a.idx + (int64_t)r * a.k_cap, a.k_cap, a.counts + r, sh);
}

template <int CL>
static cudaError_t launch_topk_cl(const TopkArgs& a, cudaStream_t st) {
  if (CL == 1) {
    topk_kernel<1><<<a.rows, kTopkThreads, 0, st>>>(a);
    return cudaGetLastError();
  }
  if (CL > 8) {
    static const cudaError_t np = cudaFuncSetAttribute(topk_kernel<CL>,
                                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (np != cudaSuccess) return np;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.rows * CL);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, topk_kernel<CL>, a);
}

cudaError_t launch_topk(const TopkArgs& a, cudaStream_t st) {
  if (a.rows <= 0) return cudaSuccess;
  // Few long rows (decode: batch x kv heads) -> a cluster of CTAs per row.
  // Measured on B200 at 128K: 64 rows: 1 CTA 141 us, 2: 83, 4: 65, 8: 85;
  // 16 rows: 4: 64, 8: 54; 8 rows: 4: 62, 8: 44.  Warp-aggregated
  // (match_any) histogram atomics and a sample-bracketed single-CTA select
  // were measured slower and removed.
  // (16-CTA non-portable clusters for <= 9 rows measured 60 us vs 32 us for 8)
  const int cl = a.len < 8192 ? 1 : (a.rows * 8 <= 148 ? 8 : (a.rows <= 148 ? 4 : 1));
  if (cl == 8) return launch_topk_cl<8>(a, st);
  if (cl == 4) return launch_topk_cl<4>(a, st);
  return launch_topk_cl<1>(a, st);
}

}  // namespace kscd
