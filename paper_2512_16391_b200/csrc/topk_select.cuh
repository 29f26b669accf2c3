// Exact Top-k of one row (order keys, radix select, ordered compaction) as a
// device function: used by topk_kernel (topk.cu) and by the fused
// anchor-selection tail of the prefill pass B (pool_prefill.cu).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace kscd {

namespace cg = cooperative_groups;

constexpr int kTopkThreads = 512;
#ifndef KSCD_TOPK_BATCH
#define KSCD_TOPK_BATCH 2
#endif
// float4 loads in flight per thread in the counting passes.  Measured on
// B200 (scripts/perf_topk.py, same box): 1 -> 2 cuts the decode select
// 65.5 -> 62.2 us (64 rows x 128K) and the 128K prefill select 2658 -> 2426
// us; 4 is equal on decode and slower on prefill; 8 drops occupancy.
constexpr int kTopkBatchDefault = KSCD_TOPK_BATCH;
#ifndef KSCD_TOPK_ITEMS
#define KSCD_TOPK_ITEMS 8
#endif
constexpr int kTopkItems = KSCD_TOPK_ITEMS;  // consecutive elements per thread per compaction chunk

KSCD_DEV uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0: equal values tie
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Barrier of the NT threads taking part: the whole CTA (TID0 = 0), or the
// warps from thread TID0 on through named barrier 1 (the fused prefill
// selection runs on the pass-B column-sum warpgroups only).
template <int NT, int TID0>
KSCD_DEV void tk_sync() {
  if (TID0 == 0) __syncthreads();
  else asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
}

// Exclusive prefix sum over the NT threads (thread order).
template <int NT = kTopkThreads, int TID0 = 0>
KSCD_DEV uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  constexpr int kTopkWarps = NT / 32;
  const int lane = threadIdx.x & 31, warp = (threadIdx.x - TID0) >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  tk_sync<NT, TID0>();
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
  tk_sync<NT, TID0>();
  const uint32_t res = warp_tot[warp] + x - v;
  total = warp_tot[32];
  tk_sync<NT, TID0>();
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

// Exact Top-k of one row (values vals[j] (+ vals2[j]), j < n): the take
// largest, ties to the smaller index, ascending, INT32_MAX-padded to k_cap;
// counts_out (written by CTA 0 of the cluster) = take.  NT threads of the CTA
// take part; CL CTAs of a cluster split the row.  Used by topk_kernel and by
// the fused anchor-selection tail of pool_prefill_kernel (NT = 384, CL = 1).
template <int CL, int NT, int TID0 = 0, int kTopkBatch = kTopkBatchDefault>
KSCD_DEV void topk_select(const float* vals, const float* vals2, int n, int take, int* out, int k_cap,
                          int* counts_out, TopkShared& sh) {
  static_assert(CL == 1 || TID0 == 0, "a cluster-split row runs on whole CTAs");
  cg::cluster_group cluster = cg::this_cluster();
  const int c = CL > 1 ? (int)cluster.block_rank() : 0;
  const int tid = threadIdx.x - TID0, lane = threadIdx.x & 31;
  constexpr int kTopkThreads = NT;
  // segment of this CTA (multiple of 8 elements so float4 loads stay aligned)
  const int seg_len = ((n + CL - 1) / CL + 7) & ~7;
  const int seg0 = min(n, c * seg_len), seg1 = min(n, seg0 + seg_len);
  const bool vec = ((reinterpret_cast<uintptr_t>(vals) & 15) == 0) &&
                   (vals2 == nullptr || (reinterpret_cast<uintptr_t>(vals2) & 15) == 0);

  if (c == 0) {
    if (tid == 0) *counts_out = take;
    for (int j = take + tid; j < k_cap; j += kTopkThreads) out[j] = 0x7fffffff;
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
    tk_sync<NT, TID0>();
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
    if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();
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
    const uint32_t pre = block_excl_scan<NT, TID0>(mine, sh.scan_buf, tot_unused);
    (void)pre;
    if (tid == 0) {
      uint32_t* dst = CL > 1 ? cluster.map_shared_rank(sh.range_tot, 0) : sh.range_tot;
      dst[c] = tot_unused;
    }
    if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();
    uint32_t above_range = 0;
    {
      const uint32_t* rt = CL > 1 ? cluster.map_shared_rank(sh.range_tot, 0) : sh.range_tot;
      for (int q = c + 1; q < CL; ++q) above_range += rt[q];
      const uint32_t my_tot = rt[c];
      if (above_range < remaining && above_range + my_tot >= remaining) {
        // the threshold bin lies in this CTA's range: descending scan of it,
        // thread t owning bins top-bpt*t ... (bpt = 1 in a cluster, 8 alone)
        constexpr int kMaxBpt = (4096 + kTopkThreads - 1) / kTopkThreads;
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
        uint32_t above = above_range + block_excl_scan<NT, TID0>(local, sh.scan_buf, tot2);
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
    if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();
    prefix |= sh.sel_bin << shift;
    pmask |= (uint32_t)(nb - 1) << shift;
    remaining -= sh.sel_above;
    if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();   // hist / sel reuse in the next pass
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
      block_excl_scan<NT, TID0>(ab, sh.scan_buf, ab_tot);    // (its barriers also publish ncand)
      above_bin = ab_tot;
      const uint32_t my_ovf = sh.ncand > (uint32_t)kRadixCandCap;
      if (tid < CL) {
        uint32_t* dst = CL > 1 ? cluster.map_shared_rank(sh.ovf, tid) : sh.ovf;
        dst[c] = my_ovf;
      }
      if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();
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
  block_excl_scan<NT, TID0>(gt_seg, sh.scan_buf, tg);
  block_excl_scan<NT, TID0>(eq_seg, sh.scan_buf, te);
  if (tid == 0) {
    uint32_t* dst = CL > 1 ? &cluster.map_shared_rank(&sh, 0)->seg_cnt[c][0] : &sh.seg_cnt[c][0];
    dst[0] = tg;
    dst[1] = te;
  }
  if (CL > 1) cluster.sync(); else tk_sync<NT, TID0>();
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
    const uint32_t pre = block_excl_scan<NT, TID0>((eq << 16) | gt, sh.scan_buf, tot);
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

}  // namespace kscd
