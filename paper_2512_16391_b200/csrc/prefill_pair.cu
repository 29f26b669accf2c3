// Prefill attention on CTA PAIRS (tcgen05 cta_group::2): the four query heads
// of one kv group at one 128-row tile share a cluster of two CTAs, and every
// S = Q K^T and O += P V is ONE 2-SM UMMA (M = 256: 128 query rows from each
// CTA) issued by the even CTA.  Each CTA stages only HALF of every K/V block:
//
//   K block (128 keys x 128 d): CTA r holds keys [64r, 64r+64)   (B split on N = keys)
//   V block (128 keys x 128 d): CTA r holds d-columns [64r, 64r+64) (B split on N = d)
//
// so the pair reads each K/V block from L2 once instead of twice, and every
// SM streams half the operand bytes per FLOP out of shared memory -- the two
// limits the single-CTA kernel (prefill.cu) runs into (measured ~17 B/clk/SM
// of L2 gather bandwidth; SMEM operand reads at the tensor rate).  Per CTA the
// pipeline is the same warp-specialised design as prefill.cu:
//
//   warp 0 (lane 0)  TMA producer (dense): its K/V halves, 2-SM TMA whose
//                    transaction bytes land on the leader's full barriers
//   warps 0-2        cp.async gather producers (sparse): its halves of the
//                    selected rows; one arrive per CTA on the leader's barrier
//   warp 3 (lane 0)  leader only: MMA issuer for the pair
//   warps 4-7 / 8-11 softmax warpgroups of tile slots 0 / 1 (its own TMEM
//                    lanes), P written over S in its own TMEM, lazy O rescale
//
// Barriers live at the same offsets in both CTAs.  Full barriers (q, k, v, p)
// are waited on by the leader only and receive arrivals from both CTAs;
// s_full / o_done / k_empty / kv_empty are multicast-committed by the
// leader's MMA to both CTAs.  Modes: DENSE and SPARSE (prefill.cu documents
// the reference semantics they implement).  Clusters pair CTAs along x (a
// (1, 2) cluster is rejected for cta_group::2 at launch).
//
// Measured on B200 (Llama-8B heads): correct (the GPU parity
// suite passes with it forced on), but its MMA skeleton runs at the same rate
// as the single-CTA kernel's (5.75 ms at 32K, 100.8 ms at 128K) and the
// cross-CTA P-ready round trip lengthens the S -> softmax -> PV chain: dense
// 128K 142 ms vs 126, sparse 19.0 vs 15.4.  Opt-in (KSCD_PREFILL_PAIR=1).
#include <stdio.h>
#include <stdlib.h>

#include "sm100.cuh"
#include "kscd_internal.h"

namespace kscd {
using namespace sm100;

namespace pp2 {
constexpr int kTileM = 128;
constexpr int kBlockN = 128;
constexpr int kStages = 4;
constexpr int kThreads = 384;
constexpr int kQTileBytes = 128 * 256;     // 128 rows x 128 bf16 (one head's Q tile)
constexpr int kQHalf = 16384;              // one 64-column half of it
constexpr int kKHalfBytes = 64 * 256;      // 64 keys x 128 d  [2 d-halves][64 rows][128 B]
constexpr int kKDHalf = 8192;              // one d-half of it
constexpr int kVHalfBytes = 128 * 128;     // 128 keys x 64 d  [128 rows][128 B]
constexpr int kPosBufs = kStages + 2;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + 2 * kQTileBytes;
constexpr int kOffV = kOffK + kStages * kKHalfBytes;
constexpr int kOffPos = kOffV + kStages * kVHalfBytes;
constexpr int kOffBar = kOffPos + kPosBufs * 128 * 4;
constexpr int kNumBars = 32;
constexpr int kOffTmem = kOffBar + kNumBars * 8;
constexpr int kSmemBytes = kOffTmem + 16 + 1024;
constexpr uint32_t kIdescS = idesc_bf16(256, 128, false, false);
constexpr uint32_t kIdescPV = idesc_bf16(256, 128, false, true);
constexpr float kRescaleThreshold = 8.0f;
// barrier slots
constexpr int kQFull = 0;
constexpr int kKFull = 1;        // + stage
constexpr int kVFull = 5;        // + stage
constexpr int kKVEmpty = 9;      // + stage
constexpr int kKEmpty = 13;      // + stage (sparse)
constexpr int kSFull = 17;       // + tile
constexpr int kPFull = 19;       // + tile
constexpr int kODone = 21;       // + tile
}  // namespace pp2

struct PairTmaps {
  CUtensorMap q, k, v;   // q/k: box {64, 128 or 64, 1}; v: box {64, 128, 1}
};

template <int MODE>
__global__ void __launch_bounds__(pp2::kThreads, 1)
    prefill_pair_kernel(const __grid_constant__ PairTmaps tm, const PrefillArgs a) {
  using namespace pp2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  int* posbuf = reinterpret_cast<int*>(smem + kOffPos);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();               // 0 = leader (issues the pair's MMAs)
  const int num_tiles = (a.N + kTileM - 1) / kTileM;
  const int ti = num_tiles - 1 - (int)blockIdx.y;      // heavy (late) tiles first
  const int r0 = ti * kTileM;
  const int h0 = blockIdx.x * 2;                       // this CTA's two heads (cluster pairs along x)
  const int g = h0 / a.G;                              // same kv head for both CTAs (G % 4 == 0)

  int count = 0;
  const int* sel = nullptr;
  int nb;
  if (MODE == PMODE_SPARSE) {
    const int src = a.head_map ? __ldg(a.head_map + g) : g;
    sel = a.idx + (int64_t)src * a.idx_sg + (int64_t)ti * a.idx_st;
    count = min(__ldg(a.cnt + (int64_t)src * a.cnt_sg + ti), a.k_cap);
    nb = (count + kBlockN - 1) / kBlockN;
  } else {
    const int kend = a.causal ? min(a.N, r0 + kTileM) : a.N;
    nb = (kend + kBlockN - 1) / kBlockN;
  }

  if (threadIdx.x == 0) {
    mbar_init(&bars[kQFull], 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars[kKFull + s], MODE == PMODE_SPARSE ? 2 : 1);
      mbar_init(&bars[kVFull + s], MODE == PMODE_SPARSE ? 2 : 1);
      mbar_init(&bars[kKVEmpty + s], 1);
      mbar_init(&bars[kKEmpty + s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars[kSFull + t], 1);
      mbar_init(&bars[kPFull + t], 8);     // 4 softmax warps x 2 CTAs
      mbar_init(&bars[kODone + t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();                                  // barriers + TMEM visible pair-wide
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t leader_bar0 = cluster_addr(smem_u32(&bars[0]), 0);
  auto leader_bar = [&](int i) { return leader_bar0 + 8u * (uint32_t)i; };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n");
    if (warp == 3) {
      if (rank == 0 && lane == 0 && nb > 0) {
        // ------------------------------------------ MMA issuer (leader)
        const uint32_t qaddr = smem_u32(smem + kOffQ);
        const uint32_t kaddr = smem_u32(smem + kOffK);
        const uint32_t vaddr = smem_u32(smem + kOffV);
        auto issue_s = [&](int t, int st) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t qoff = (ks >> 2) * kQHalf + (ks & 3) * 32;
            const uint32_t koff = (ks >> 2) * kKDHalf + (ks & 3) * 32;
            mma_ss_pair(tmem + t * 256, sw128_desc(qaddr + t * kQTileBytes + qoff, 16, 1024),
                        sw128_desc(kaddr + st * kKHalfBytes + koff, 16, 1024), kIdescS, ks > 0);
          }
          mma_commit_pair(&bars[kSFull + t]);
        };
        auto issue_pv = [&](int t, int st, int j) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            mma_ts_pair(tmem + t * 256 + 128, tmem + t * 256 + ks * 8,
                        sw128_desc(vaddr + st * kVHalfBytes + ks * 2048, 8192, 1024), kIdescPV,
                        (j > 0 || ks > 0) ? 1u : 0u);
        };
        mbar_wait(&bars[kQFull], 0);
        mbar_wait(&bars[kKFull], 0);
        tc_fence_after();
        issue_s(0, 0);
        issue_s(1, 0);
        if (MODE == PMODE_SPARSE) mma_commit_pair(&bars[kKEmpty]);
        for (int j = 0; j < nb; ++j) {
          const int st = j % kStages;
          const bool more = j + 1 < nb;
          const int st1 = (j + 1) % kStages;
          mbar_wait(&bars[kVFull + st], (j / kStages) & 1);
          mbar_wait(&bars[kPFull + 0], j & 1);
          tc_fence_after();
          issue_pv(0, st, j);
          if (j == nb - 1) mma_commit_pair(&bars[kODone + 0]);
          if (more) {
            mbar_wait(&bars[kKFull + st1], ((j + 1) / kStages) & 1);
            tc_fence_after();
            issue_s(0, st1);
          }
          mbar_wait(&bars[kPFull + 1], j & 1);
          tc_fence_after();
          issue_pv(1, st, j);
          if (j == nb - 1) mma_commit_pair(&bars[kODone + 1]);
          mma_commit_pair(&bars[kKVEmpty + st]);     // K/V stage of block j free in both CTAs
          if (more) {
            issue_s(1, st1);
            if (MODE == PMODE_SPARSE) mma_commit_pair(&bars[kKEmpty + st1]);
          }
        }
      }
    } else if (MODE != PMODE_SPARSE) {
      if (warp == 0 && lane == 0 && nb > 0) {
        // ------------------------------------------ TMA producer (both CTAs)
        tma_prefetch(&tm.q);
        tma_prefetch(&tm.k);
        tma_prefetch(&tm.v);
        if (rank == 0) mbar_expect_tx(&bars[kQFull], 2 * 2 * kQTileBytes);   // both CTAs' two tiles
        for (int t = 0; t < 2; ++t)
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d_pair(smem + kOffQ + t * kQTileBytes + hf * kQHalf, &tm.q, &bars[kQFull], hf * 64, r0, h0 + t);
        for (int j = 0; j < nb; ++j) {
          const int st = j % kStages;
          if (j >= kStages) mbar_wait(&bars[kKVEmpty + st], ((j / kStages) - 1) & 1);
          if (rank == 0) {
            mbar_expect_tx(&bars[kKFull + st], 2 * kKHalfBytes);
            mbar_expect_tx(&bars[kVFull + st], 2 * kVHalfBytes);
          }
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d_pair(smem + kOffK + st * kKHalfBytes + hf * kKDHalf, &tm.k, &bars[kKFull + st], hf * 64,
                             j * kBlockN + 64 * (int)rank, g);
          tma_load_3d_pair(smem + kOffV + st * kVHalfBytes, &tm.v, &bars[kVFull + st], 64 * (int)rank, j * kBlockN, g);
        }
      }
    } else {
      // ------------------------------------- sparse gather producers (96)
      const int pt = threadIdx.x;
      if (pt == 0 && nb > 0) {
        tma_prefetch(&tm.q);
        if (rank == 0) mbar_expect_tx(&bars[kQFull], 2 * 2 * kQTileBytes);
        for (int t = 0; t < 2; ++t)
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d_pair(smem + kOffQ + t * kQTileBytes + hf * kQHalf, &tm.q, &bars[kQFull], hf * 64, r0, h0 + t);
      }
      const __nv_bfloat16* kg = a.k + (int64_t)g * a.kv_sh;
      const __nv_bfloat16* vg = a.v + (int64_t)g * a.kv_sh + 64 * rank;
      const int r1 = pt + 96;
      auto load_sel = [&](int j, int& p0, int& p1) {
        const int e0 = j * kBlockN + pt, e1 = j * kBlockN + r1;
        p0 = e0 < count ? __ldg(sel + e0) : 0x7fffffff;
        p1 = (r1 < kBlockN && e1 < count) ? __ldg(sel + e1) : 0x7fffffff;
      };
      int p0 = 0x7fffffff, p1 = 0x7fffffff;
      if (nb > 0) load_sel(0, p0, p1);
      // K half: keys [64 rank, 64 rank + 64) of the block, all 128 d (16 x 16 B per row)
      auto gather_k = [&](uint32_t dst, const int* pos) {
#pragma unroll 2
        for (int c = pt; c < 64 * 16; c += 96) {
          const int r = c >> 4, ch = c & 15;
          const int p = pos[64 * rank + r];
          const bool valid = p != 0x7fffffff;
          const uint32_t off = (ch >> 3) * kKDHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
          cp_async16_zfill(dst + off, kg + (int64_t)(valid ? p : 0) * 128 + ch * 8, valid);
        }
        cp_async_commit();
      };
      // V half: all 128 keys, d-columns [64 rank, 64 rank + 64) (8 x 16 B per row)
      auto gather_v = [&](uint32_t dst, const int* pos) {
#pragma unroll 2
        for (int c = pt; c < 128 * 8; c += 96) {
          const int r = c >> 3, ch = c & 7;
          const int p = pos[r];
          const bool valid = p != 0x7fffffff;
          const uint32_t off = r * 128 + ((ch ^ (r & 7)) << 4);
          cp_async16_zfill(dst + off, vg + (int64_t)(valid ? p : 0) * 128 + ch * 8, valid);
        }
        cp_async_commit();
      };
      // publish: every producer thread's copies landed -> proxy fence -> one
      // arrive per CTA on the leader's barrier
      auto publish = [&](int bar) {
        fence_proxy_async_smem();
        named_bar_sync(1, 96);
        if (pt == 0) mbar_arrive_remote(leader_bar(bar));
      };
      for (int j = 0; j < nb; ++j) {
        const int st = j % kStages;
        const uint32_t ph_free = ((j / kStages) - 1) & 1;
        if (j >= kStages) mbar_wait(&bars[kKEmpty + st], ph_free);   // every S of block j - kStages retired
        int* pos = posbuf + (j % kPosBufs) * 128;
        pos[pt] = p0;
        if (r1 < kBlockN) pos[r1] = p1;
        if (j + 1 < nb) load_sel(j + 1, p0, p1);
        named_bar_sync(1, 96);
        gather_k(smem_u32(smem + kOffK + st * kKHalfBytes), pos);
        if (j > 0) {                                              // V_{j-1} landed
          cp_async_wait<1>();
          publish(kVFull + (j - 1) % kStages);
        }
        if (j >= kStages) mbar_wait(&bars[kKVEmpty + st], ph_free);  // PV of block j - kStages retired
        gather_v(smem_u32(smem + kOffV + st * kVHalfBytes), pos);
        cp_async_wait<1>();                                       // K_j landed
        publish(kKFull + st);
      }
      if (nb > 0) {
        cp_async_wait<0>();
        publish(kVFull + (nb - 1) % kStages);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n");
    // ================================================== softmax warpgroups
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;
    const int row = r0 + q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t s_col = t * 256, o_col = t * 256 + 128;
    const int h = h0 + t;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nb; ++j) {
      mbar_wait(&bars[kSFull + t], j & 1);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32(lane_base + s_col + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
      if (MODE == PMODE_SPARSE) {
        const int* pos = posbuf + (j % kPosBufs) * 128;
        if (pos[127] > r0) {
#pragma unroll
          for (int c = 0; c < 128; c += 4) {
            const int4 p = *reinterpret_cast<const int4*>(pos + c);
            if (p.x > row) s[c] = -INFINITY;   // also pads (INT32_MAX)
            if (p.y > row) s[c + 1] = -INFINITY;
            if (p.z > row) s[c + 2] = -INFINITY;
            if (p.w > row) s[c + 3] = -INFINITY;
          }
        }
      } else {
        const int k0 = j * kBlockN;
        const int lim = a.causal ? min(row, a.N - 1) : a.N - 1;
        if (k0 + kBlockN - 1 > lim) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (k0 + c > lim) s[c] = -INFINITY;
        }
      }
      const float mx_raw = max_tree<128>(s);
      const float mx = mx_raw * a.scale_log2;
      const bool need = mx > m_used + kRescaleThreshold;
      const float alpha = (need && m_used != -INFINITY) ? exp2f(m_used - mx) : 1.f;
      if (__any_sync(0xffffffffu, alpha != 1.f)) {
        // O_t holds blocks < j: PV_t(j-1) retired before S_t(j) was committed
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(lane_base + o_col + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(lane_base + o_col + c * 32, r);
        }
        tmem_st_wait();
      }
      l *= alpha;
      if (need) m_used = mx;
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
      const float2 nm2 = make_float2(-mu, -mu);
      float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2);
          const float2 p = exp2_pair(x, c * 16 + i);
          sum4[i & 3] = __fadd2_rn(sum4[i & 3], p);
          r[i] = pack_bf16(p.x, p.y);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
            ::"r"(lane_base + s_col + c * 16), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
            "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
            "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
      }
      tmem_st_wait();
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sum4[0], sum4[1]), __fadd2_rn(sum4[2], sum4[3]));
      l += sum2.x + sum2.y;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_bar(kPFull + t));   // P_t(j) of this warp's rows
    }
    // ------------------------------------------------------------ epilogue
    const bool live = row < a.N;
    if (nb > 0) {
      mbar_wait(&bars[kODone + t], 0);
      tc_fence_after();
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = a.out + ((int64_t)h * a.N + row) * 128;
    const bool fallback = (MODE == PMODE_SPARSE) && l == 0.f;
    uint32_t o[128];
    if (nb > 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32(lane_base + o_col + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 128; ++i) o[i] = 0u;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t* r = o + c * 32;
      if (live) {
        uint4 w[4];
        uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          wp[i] = pack_bf16(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
        if (fallback) {
          const uint4* vrow = reinterpret_cast<const uint4*>(a.v + (int64_t)g * a.kv_sh + (int64_t)row * 128 + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] = __ldg(vrow + i);
        }
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = w[i];
      }
    }
    if (live && a.lse) a.lse[(int64_t)h * a.N + row] = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();          // the peer is done with the leader's barriers, the leader's MMAs with both TMEMs
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

// ------------------------------------------------------------------- host
bool make_prefill_map(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride);
bool make_prefill_map_box(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride, int box_rows);

template <int MODE>
static cudaError_t launch_pair_mode(const PrefillArgs& a, cudaStream_t st) {
  PairTmaps tm;
  if (!make_prefill_map(&tm.q, a.q, a.Hq, a.N, a.q_sh)) return cudaErrorInvalidValue;
  if (!make_prefill_map_box(&tm.k, a.k, a.Hkv, a.Nk, a.kv_sh, 64)) return cudaErrorInvalidValue;
  if (!make_prefill_map(&tm.v, a.v, a.Hkv, a.Nk, a.kv_sh)) return cudaErrorInvalidValue;
  static const cudaError_t attr = cudaFuncSetAttribute(prefill_pair_kernel<MODE>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, pp2::kSmemBytes);
  if (attr != cudaSuccess) return attr;
  const int tiles = (a.N + pp2::kTileM - 1) / pp2::kTileM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.Hq / 2, tiles);
  cfg.blockDim = dim3(pp2::kThreads);
  cfg.dynamicSmemBytes = pp2::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr_cl[1];
  attr_cl[0].id = cudaLaunchAttributeClusterDimension;
  attr_cl[0].val.clusterDim.x = 2;
  attr_cl[0].val.clusterDim.y = 1;
  attr_cl[0].val.clusterDim.z = 1;
  cfg.attrs = attr_cl;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, prefill_pair_kernel<MODE>, tm, a);
}

bool prefill_pair_supported(int mode, const PrefillArgs& a) {
  return (mode == PMODE_DENSE || mode == PMODE_SPARSE) && a.slots == 2 && a.G % 4 == 0 && (a.Hq / 2) % 2 == 0;
}

cudaError_t launch_prefill_pair(int mode, const PrefillArgs& a, cudaStream_t st) {
  return mode == PMODE_SPARSE ? launch_pair_mode<PMODE_SPARSE>(a, st) : launch_pair_mode<PMODE_DENSE>(a, st);
}

}  // namespace kscd
