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
//               (k - #>T) lowest-index keys == T.  HBM/L2-bound integer work.
#include "common.cuh"
#include "kscd_internal.h"

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
constexpr int kTopkThreads = 1024;
constexpr int kTopkItems = 8;  // elements per thread per compaction chunk

KSCD_DEV uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0: equal values tie
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Exclusive prefix sum over the 1024 threads of the block (thread order).
KSCD_DEV uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = warp_tot[lane];
    uint32_t wx = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
      if (lane >= o) wx += y;
    }
    warp_tot[lane] = wx - w;  // exclusive warp offsets
    if (lane == 31) warp_tot[32] = wx;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const TopkArgs a) {
  __shared__ uint32_t hist[4096];
  __shared__ uint32_t scan_buf[33];
  __shared__ uint32_t sel_bin, sel_above;
  const int r = blockIdx.x, tid = threadIdx.x;
  int n = a.lens ? a.lens[r] : a.len;
  int k = a.ks ? a.ks[r] : a.k;
  if (a.tile > 0) {
    // k_budget (tiles.py:81-89) of the tile's causal bound, in the same fp64
    n = min(a.len, a.tile * (r % a.T + 1));
    long long kk = (long long)floor(a.fraction * (double)n);
    kk = kk < a.k_min ? a.k_min : kk;
    k = (int)(kk > n ? n : kk);
  }
  const int take = n < k ? n : k;
  const float* vals = a.vals + (int64_t)r * a.val_stride;
  int* out = a.idx + (int64_t)r * a.k_cap;
  if (tid == 0) a.counts[r] = take;
  for (int j = take + tid; j < a.k_cap; j += kTopkThreads) out[j] = 0x7fffffff;
  if (take <= 0) return;
  if (take == n) {
    for (int j = tid; j < n; j += kTopkThreads) out[j] = j;
    return;
  }

  // ---- radix select of the take-th largest key -------------------------
  uint32_t prefix = 0, pmask = 0, remaining = (uint32_t)take;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 20 : (pass == 1 ? 8 : 0);
    const int nb = pass == 2 ? 256 : 4096;
    for (int i = tid; i < nb; i += kTopkThreads) hist[i] = 0;
    __syncthreads();
    for (int j = tid; j < n; j += kTopkThreads) {
      const uint32_t key = order_key(__ldcg(vals + j));
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & (nb - 1)], 1u);
    }
    __syncthreads();
    // thread t owns bins nb-1-4t .. nb-4-4t (descending); exclusive scan in
    // thread order = number of keys in strictly higher bins
    uint32_t local = 0;
    const int top = nb - 1 - 4 * tid;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (top - i >= 0) local += hist[top - i];
    uint32_t tot;
    uint32_t above = block_excl_scan(local, scan_buf, tot);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int bin = top - i;
      if (bin >= 0) {
        const uint32_t c = hist[bin];
        if (above < remaining && above + c >= remaining) {
          sel_bin = bin;
          sel_above = above;
        }
        above += c;
      }
    }
    __syncthreads();
    prefix |= sel_bin << shift;
    pmask |= (uint32_t)(nb - 1) << shift;
    remaining -= sel_above;
    __syncthreads();
  }
  const uint32_t T = prefix;       // exact key of the take-th largest
  const uint32_t r_eq = remaining; // how many keys == T to keep (lowest indices)

  // ---- ordered compaction ------------------------------------------------
  uint32_t gt_carry = 0, eq_carry = 0;
  const int chunk = kTopkThreads * kTopkItems;
#pragma unroll 1
  for (int base = 0; base < n; base += chunk) {
    uint32_t keys[kTopkItems];
    uint32_t gt = 0, eq = 0;
    const int j0 = base + tid * kTopkItems;
#pragma unroll
    for (int i = 0; i < kTopkItems; ++i) {
      const int j = j0 + i;
      keys[i] = j < n ? order_key(__ldcg(vals + j)) : 0u;
      gt += (j < n && keys[i] > T);
      eq += (j < n && keys[i] == T);
    }
    uint32_t tot;
    const uint32_t pre = block_excl_scan((eq << 16) | gt, scan_buf, tot);
    uint32_t g_before = gt_carry + (pre & 0xffffu);
    uint32_t e_before = eq_carry + (pre >> 16);
#pragma unroll
    for (int i = 0; i < kTopkItems; ++i) {
      const int j = j0 + i;
      if (j >= n) break;
      const bool is_gt = keys[i] > T, is_eq = keys[i] == T;
      if (is_gt || (is_eq && e_before < r_eq)) out[g_before + min(e_before, r_eq)] = j;
      g_before += is_gt;
      e_before += is_eq;
    }
    gt_carry += tot & 0xffffu;
    eq_carry += tot >> 16;
  }
}

cudaError_t launch_topk(const TopkArgs& a, cudaStream_t st) {
  if (a.rows <= 0) return cudaSuccess;
  topk_kernel<<<a.rows, kTopkThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace kscd
