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
#include <cooperative_groups.h>
#include <stdlib.h>

#include "common.cuh"
#include "kscd_internal.h"

namespace cg = cooperative_groups;

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
constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
#ifndef KSCD_TOPK_BATCH
#define KSCD_TOPK_BATCH 2
#endif
// float4 loads in flight per thread in the counting passes.  Measured on
// B200 (scripts/perf_topk.py, same box): 1 -> 2 cuts the decode select
// 65.5 -> 62.2 us (64 rows x 128K) and the 128K prefill select 2658 -> 2426
// us; 4 is equal on decode and slower on prefill; 8 drops occupancy.
constexpr int kTopkBatch = KSCD_TOPK_BATCH;
#ifndef KSCD_TOPK_ITEMS
#define KSCD_TOPK_ITEMS 8
#endif
constexpr int kTopkItems = KSCD_TOPK_ITEMS;  // consecutive elements per thread per compaction chunk

KSCD_DEV uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0: equal values tie
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Exclusive prefix sum over the threads of the block (thread order).
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
    const uint32_t w = lane < kTopkWarps ? warp_tot[lane] : 0u;
    uint32_t wx = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
      if (lane >= o) wx += y;
    }
    if (lane < kTopkWarps) warp_tot[lane] = wx - w;  // exclusive warp offsets
    if (lane == 31) warp_tot[32] = wx;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return res;
}

// Four consecutive values of a row; out-of-range -> 0.
KSCD_DEV void load4_plane(const float* vals, int j, int end, bool vec, float (&v)[4]) {
  if (vec && j + 3 < end) {
    const float4 f = __ldcg(reinterpret_cast<const float4*>(vals + j));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = j + i < end ? __ldcg(vals + j + i) : 0.f;
  }
}

// NB groups of four values at j0 + b*step (plus the second partial plane
// when the row is stored as two sums, see pool_prefill.cu).  Every load is
// issued before the first add: an add right behind its own load (even a
// predicated-off one) waits on the load's scoreboard and serialises the
// loads -- the dominant stall of the counting passes (ncu, decode shapes).
template <int NB>
KSCD_DEV void load_groups(const float* vals, const float* vals2, int j0, int step, int end, bool vec,
                          float (&v)[NB][4]) {
#pragma unroll
  for (int b = 0; b < NB; ++b) load4_plane(vals, j0 + b * step, end, vec, v[b]);
  if (vals2) {
    float w[NB][4];
#pragma unroll
    for (int b = 0; b < NB; ++b) load4_plane(vals2, j0 + b * step, end, vec, w[b]);
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int i = 0; i < 4; ++i) v[b][i] += w[b][i];
  }
}

// Keys of the threshold bin of the first digit that a CTA keeps on chip
// (candidate mode, see the kernel); more than this in any CTA of a cluster
// and the row takes the full-segment passes instead.
#ifndef KSCD_TOPK_CAND
#define KSCD_TOPK_CAND 6144
#endif
constexpr int kRadixCandCap = KSCD_TOPK_CAND;

struct TopkShared {
  uint32_t hist[4096];
  uint32_t range_tot[16];     // per-CTA bin-range totals (valid in CTA 0)
  uint32_t seg_cnt[16][2];    // per-CTA (gt, eq) counts (valid in CTA 0)
  uint32_t scan_buf[33];
  uint32_t sel_bin, sel_above, sel_cnt;   // threshold bin, keys above it, keys in it (cluster-wide)
  uint32_t ncand;             // candidates appended by this CTA
  uint32_t ovf[16];           // per-CTA candidate overflow flags (every CTA holds all)
  uint32_t cand[kRadixCandCap];    // candidate keys (threshold bin of digit 0)
};

template <int CL>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const TopkArgs a) {
  __shared__ TopkShared sh;
  cg::cluster_group cluster = cg::this_cluster();
  const int c = CL > 1 ? (int)cluster.block_rank() : 0;
  const int r = blockIdx.x / CL;
  const int tid = threadIdx.x, lane = tid & 31;
  int n = a.lens ? a.lens[r] : a.len;
  int k = a.ks ? a.ks[r] : a.k;
  if (a.seq_div > 0) {
    // ragged decode batch: this row's sequence length and its k_budget
    n = min(a.len, __ldg(a.seq_lens + r / a.seq_div));
    long long kk = (long long)floor(a.fraction * (double)n);
    kk = kk < a.k_min ? a.k_min : kk;
    k = (int)(kk > n ? n : kk);
  } else if (a.tile > 0) {
    // k_budget (tiles.py:81-89) of the tile's causal bound, in the same fp64
    n = min(a.len, a.tile * (r % a.T + 1));
    long long kk = (long long)floor(a.fraction * (double)n);
    kk = kk < a.k_min ? a.k_min : kk;
    k = (int)(kk > n ? n : kk);
  }
  const int take = n < k ? n : k;
  const float* vals = a.vals + (int64_t)r * a.val_stride;
  const float* vals2 = a.vals2 ? a.vals2 + (int64_t)r * a.val_stride : nullptr;
  int* out = a.idx + (int64_t)r * a.k_cap;
  // segment of this CTA (multiple of 8 elements so float4 loads stay aligned)
  const int seg_len = ((n + CL - 1) / CL + 7) & ~7;
  const int seg0 = min(n, c * seg_len), seg1 = min(n, seg0 + seg_len);
  const bool vec = ((reinterpret_cast<uintptr_t>(vals) & 15) == 0);

  if (c == 0) {
    if (tid == 0) a.counts[r] = take;
    for (int j = take + tid; j < a.k_cap; j += kTopkThreads) out[j] = 0x7fffffff;
  }
  if (take <= 0) return;                      // uniform across the cluster
  if (take == n) {
    for (int j = seg0 + tid; j < seg1; j += kTopkThreads) out[j] = j;
    return;
  }

  // ---- radix select of the take-th largest key -------------------------
  uint32_t prefix = 0, pmask = 0, remaining = (uint32_t)take;
  const int iters = (seg1 - seg0 + 4 * kTopkThreads - 1) / (4 * kTopkThreads);
  // Candidate mode: after the first digit, the keys of its threshold bin
  // are copied to shared memory in one more pass over the segment, and the
  // two remaining digits and the (gt, eq) counts of the compaction run on
  // that copy -- three passes over the row from L2 instead of five.
  bool cand_mode = false;
  uint32_t above_bin = 0;     // this CTA's keys above digit 0's threshold bin
  if (tid == 0) sh.ncand = 0;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 20 : (pass == 1 ? 8 : 0);
    const int nb = pass == 2 ? 256 : 4096;
    for (int i = tid; i < nb; i += kTopkThreads) sh.hist[i] = 0;
    __syncthreads();
    if (cand_mode) {
      const int nc = (int)sh.ncand;
      for (int i = tid; i < nc; i += kTopkThreads) {
        const uint32_t key = sh.cand[i];
        if ((key & pmask) == prefix) atomicAdd(&sh.hist[(key >> shift) & (nb - 1)], 1u);
      }
    } else
    // kTopkBatch float4 loads in flight per thread before any atomic: the
    // row streams from L2 and one outstanding load per thread leaves the
    // pass latency-bound (few CTAs per SM at decode shapes)
#pragma unroll 1
    for (int it0 = 0; it0 < iters; it0 += kTopkBatch) {
      float v[kTopkBatch][4];
      load_groups<kTopkBatch>(vals, vals2, seg0 + (it0 * kTopkThreads + tid) * 4, kTopkThreads * 4, seg1, vec, v);
#pragma unroll
      for (int b = 0; b < kTopkBatch; ++b) {
        const int j = seg0 + ((it0 + b) * kTopkThreads + tid) * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t key = order_key(v[b][i]);
          const bool m = (j + i < seg1) && ((key & pmask) == prefix);
          const uint32_t bin = (key >> shift) & (nb - 1);
          if (m) atomicAdd(&sh.hist[bin], 1u);
        }
      }
    }
    if (CL > 1) cluster.sync(); else __syncthreads();
    // CTA c owns bins [c*per, (c+1)*per): sum them over the cluster
    const int per = nb / CL;
    const int b0 = c * per;
    uint32_t mine = 0;
    for (int i = tid; i < per; i += kTopkThreads) {
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const uint32_t* h = CL > 1 ? cluster.map_shared_rank(sh.hist, q) : sh.hist;
        s += h[b0 + i];
      }
      mine += s;
    }
    // range total -> CTA 0
    uint32_t tot_unused;
    const uint32_t pre = block_excl_scan(mine, sh.scan_buf, tot_unused);
    (void)pre;
    if (tid == 0) {
      uint32_t* dst = CL > 1 ? cluster.map_shared_rank(sh.range_tot, 0) : sh.range_tot;
      dst[c] = tot_unused;
    }
    if (CL > 1) cluster.sync(); else __syncthreads();
    uint32_t above_range = 0;
    {
      const uint32_t* rt = CL > 1 ? cluster.map_shared_rank(sh.range_tot, 0) : sh.range_tot;
      for (int q = c + 1; q < CL; ++q) above_range += rt[q];
      const uint32_t my_tot = rt[c];
      if (above_range < remaining && above_range + my_tot >= remaining) {
        // the threshold bin lies in this CTA's range: descending scan of it,
        // thread t owning bins top-bpt*t ... (bpt = 1 in a cluster, 8 alone)
        constexpr int kMaxBpt = 4096 / kTopkThreads;
        const int bpt = (per + kTopkThreads - 1) / kTopkThreads;
        uint32_t local = 0;
        const int top = b0 + per - 1 - bpt * tid;
        uint32_t cnts[kMaxBpt];
#pragma unroll
        for (int i = 0; i < kMaxBpt; ++i) {
          const int bin = top - i;
          uint32_t s = 0;
          if (i < bpt && bin >= b0) {
#pragma unroll
            for (int q = 0; q < CL; ++q) {
              const uint32_t* h = CL > 1 ? cluster.map_shared_rank(sh.hist, q) : sh.hist;
              s += h[bin];
            }
          }
          cnts[i] = s;
          local += s;
        }
        uint32_t tot2;
        uint32_t above = above_range + block_excl_scan(local, sh.scan_buf, tot2);
#pragma unroll
        for (int i = 0; i < kMaxBpt; ++i) {
          const int bin = top - i;
          if (i < bpt && bin >= b0) {
            if (above < remaining && above + cnts[i] >= remaining) {
              for (int q = 0; q < CL; ++q) {
                TopkShared* dst = CL > 1 ? cluster.map_shared_rank(&sh, q) : &sh;
                dst->sel_bin = (uint32_t)bin;
                dst->sel_above = above;
                dst->sel_cnt = cnts[i];
              }
            }
            above += cnts[i];
          }
        }
      }
    }
    if (CL > 1) cluster.sync(); else __syncthreads();
    prefix |= sh.sel_bin << shift;
    pmask |= (uint32_t)(nb - 1) << shift;
    remaining -= sh.sel_above;
    if (CL > 1) cluster.sync(); else __syncthreads();   // hist / sel reuse in the next pass
    // only when the bin's cluster-wide count says the copy will (very
    // likely) fit: long prefill rows of near-uniform attention put most of a
    // row in one bin, and a wasted copy pass costs more than it saves
    if (pass == 0 && sh.sel_cnt <= (uint32_t)(CL == 1 ? kRadixCandCap : kRadixCandCap * CL / 2)) {
      // copy the threshold bin's keys on chip and count the keys above it
      const uint32_t hi_key = prefix | 0x000fffffu;
      uint32_t ab = 0;
#pragma unroll 1
      for (int it0 = 0; it0 < iters; it0 += kTopkBatch) {
        float v[kTopkBatch][4];
        load_groups<kTopkBatch>(vals, vals2, seg0 + (it0 * kTopkThreads + tid) * 4, kTopkThreads * 4, seg1, vec, v);
#pragma unroll
        for (int b = 0; b < kTopkBatch; ++b) {
          const int j = seg0 + ((it0 + b) * kTopkThreads + tid) * 4;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t key = order_key(v[b][i]);
            const bool ok = j + i < seg1;
            ab += ok && key > hi_key;
            const bool isc = ok && (key & pmask) == prefix;
            const uint32_t m = __ballot_sync(0xffffffffu, isc);
            if (m) {
              const int leader = __ffs(m) - 1;
              uint32_t base = 0;
              if (lane == leader) base = atomicAdd(&sh.ncand, (uint32_t)__popc(m));
              base = __shfl_sync(0xffffffffu, base, leader);
              const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
              if (isc && pos < (uint32_t)kRadixCandCap) sh.cand[pos] = key;
            }
          }
        }
      }
      uint32_t ab_tot;
      block_excl_scan(ab, sh.scan_buf, ab_tot);    // (its barriers also publish ncand)
      above_bin = ab_tot;
      const uint32_t my_ovf = sh.ncand > (uint32_t)kRadixCandCap;
      if (tid < CL) {
        uint32_t* dst = CL > 1 ? cluster.map_shared_rank(sh.ovf, tid) : sh.ovf;
        dst[c] = my_ovf;
      }
      if (CL > 1) cluster.sync(); else __syncthreads();
      uint32_t any = 0;
#pragma unroll
      for (int q = 0; q < CL; ++q) any |= sh.ovf[q];
      cand_mode = any == 0;
    }
  }
  const uint32_t T = prefix;       // exact key of the take-th largest
  const uint32_t r_eq = remaining; // how many keys == T to keep (lowest indices)

  // ---- ordered compaction ------------------------------------------------
  const int chunk = kTopkThreads * kTopkItems;
  uint32_t gt_seg = 0, eq_seg = 0;
  if (cand_mode) {
    const int nc = (int)sh.ncand;
    for (int i = tid; i < nc; i += kTopkThreads) {
      const uint32_t key = sh.cand[i];
      gt_seg += key > T;
      eq_seg += key == T;
    }
    if (tid == 0) gt_seg += above_bin;
  } else
#pragma unroll 1
  for (int base = seg0; base < seg1; base += kTopkThreads * 4 * kTopkBatch) {
    float v[kTopkBatch][4];
    load_groups<kTopkBatch>(vals, vals2, base + tid * 4, kTopkThreads * 4, seg1, vec, v);
#pragma unroll
    for (int b = 0; b < kTopkBatch; ++b) {
      const int j = base + (b * kTopkThreads + tid) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t key = order_key(v[b][i]);
        gt_seg += (j + i < seg1 && key > T);
        eq_seg += (j + i < seg1 && key == T);
      }
    }
  }
  uint32_t tg, te;
  block_excl_scan(gt_seg, sh.scan_buf, tg);
  block_excl_scan(eq_seg, sh.scan_buf, te);
  if (tid == 0) {
    uint32_t* dst = CL > 1 ? &cluster.map_shared_rank(&sh, 0)->seg_cnt[c][0] : &sh.seg_cnt[c][0];
    dst[0] = tg;
    dst[1] = te;
  }
  if (CL > 1) cluster.sync(); else __syncthreads();
  uint32_t gt_carry = 0, eq_carry = 0;
  {
    const TopkShared* s0 = CL > 1 ? cluster.map_shared_rank(&sh, 0) : &sh;
    for (int q = 0; q < c; ++q) {
      gt_carry += s0->seg_cnt[q][0];
      eq_carry += s0->seg_cnt[q][1];
    }
  }
  if (CL > 1) cluster.sync();   // CTA 0's seg_cnt stays readable until all have read it
#pragma unroll 1
  for (int base = seg0; base < seg1; base += chunk) {
    uint32_t keys[kTopkItems];
    uint32_t gt = 0, eq = 0;
    const int j0 = base + tid * kTopkItems;
    {
      float v[kTopkItems / 4][4];
      load_groups<kTopkItems / 4>(vals, vals2, j0, 4, seg1, vec, v);
#pragma unroll
      for (int h = 0; h < kTopkItems; ++h) keys[h] = order_key(v[h / 4][h % 4]);
    }
#pragma unroll
    for (int i = 0; i < kTopkItems; ++i) {
      const bool ok = j0 + i < seg1;
      gt += (ok && keys[i] > T);
      eq += (ok && keys[i] == T);
    }
    uint32_t tot;
    const uint32_t pre = block_excl_scan((eq << 16) | gt, sh.scan_buf, tot);
    uint32_t g_before = gt_carry + (pre & 0xffffu);
    uint32_t e_before = eq_carry + (pre >> 16);
#pragma unroll
    for (int i = 0; i < kTopkItems; ++i) {
      const int j = j0 + i;
      if (j >= seg1) break;
      const bool is_gt = keys[i] > T, is_eq = keys[i] == T;
      if (is_gt || (is_eq && e_before < r_eq)) out[g_before + min(e_before, r_eq)] = j;
      g_before += is_gt;
      e_before += is_eq;
    }
    gt_carry += tot & 0xffffu;
    eq_carry += tot >> 16;
  }
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
  // 16-CTA (non-portable) clusters when even 8 per row leave half the SMs idle
  const int cl = a.len < 8192 ? 1 : (a.rows * 16 <= 148 ? 16 : (a.rows * 8 <= 148 ? 8 : (a.rows <= 148 ? 4 : 1)));
  if (cl == 16) return launch_topk_cl<16>(a, st);
  if (cl == 8) return launch_topk_cl<8>(a, st);
  if (cl == 4) return launch_topk_cl<4>(a, st);
  return launch_topk_cl<1>(a, st);
}

}  // namespace kscd
