// Prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA = two query tiles of 128 rows -- two query heads of the same kv
// group at the same token range, so every K/V block is loaded once and used
// by both -- and a warp-specialised pipeline:
//
//   warp 0 (lane 0)  TMA producer: Q tiles once, K/V blocks through a
//                    2-stage ring (dense modes)
//   warps 0-2        cp.async gather producers (sparse mode): K/V rows at
//                    the selected positions into the same 128B-swizzled
//                    layout TMA would produce
//   warp 3 (lane 0)  MMA issuer: S_t = Q_t K^T (SS, fp32 in TMEM), then
//                    O_t += P_t V (TS: P read back from TMEM as bf16)
//   warps 4-7 / 8-11 softmax warpgroups of tile 0 / tile 1: one thread per
//                    row (TMEM lane), so the row max / sum need no shuffles;
//                    P is written over S in TMEM; O is rescaled lazily (only
//                    when the running max grows by > 2^8), so the correction
//                    step is rare.
//
// The two tiles ping-pong: while one warpgroup exponentiates block j, the
// tensor core runs the other tile's PV / next S.  TMEM: S0|P0, O0, S1|P1,
// O1 = 4 x 128 columns (all 512).
//
// Modes (reference semantics):
//   DENSE   causal (or full) attention over keys [0, N): O, LSE
//           dense_attention, attention.py:106-144 (never materialising P)
//   SPARSE  keys = the (kv head, tile) selection routed through head_map;
//           row r sees the selected keys <= r (the staircase), a row with
//           none falls back to V[r]: topk_attention, attention.py:185-253,
//           _routed_selections, runner.py:210-225.  O, LSE
//   LSE     QK^T + online softmax statistics only (anchor pass A)
#include <stdlib.h>

#include "sm100.cuh"
#include "kscd_internal.h"

namespace kscd {
using namespace sm100;

namespace pf {
constexpr int kTileM = 128;          // rows per query tile (= Kascade prefill tile)
constexpr int kBlockN = 128;         // keys per block
constexpr int kStages = 2;
constexpr int kThreads = 384;
constexpr int kTileBytes = 128 * 256;  // 128 rows x 128 bf16
constexpr int kHalf = 16384;           // one 64-column 128B-swizzled half tile
// smem layout (bytes, 1024-aligned where needed)
constexpr int kOffQ = 0;                                   // 2 tiles
constexpr int kOffK = kOffQ + 2 * kTileBytes;              // stages
constexpr int kOffV = kOffK + kStages * kTileBytes;
constexpr int kPosBufs = 4;                               // sparse: positions of blocks j..j+3
constexpr int kOffPos = kOffV + kStages * kTileBytes;      // int[kPosBufs][128]
constexpr int kOffBar = kOffPos + kPosBufs * 128 * 4;
constexpr int kNumBars = 16;
constexpr int kOffTmem = kOffBar + kNumBars * 8;
constexpr int kSmemBytes = kOffTmem + 16 + 1024;           // + alignment slack
constexpr uint32_t kIdescS = idesc_bf16(128, 128, false, false);
constexpr uint32_t kIdescPV = idesc_bf16(128, 128, false, true);
constexpr float kRescaleThreshold = 8.0f;                  // log2 units
}  // namespace pf

struct PrefillTmaps {
  CUtensorMap q, k, v;
};

#ifdef KSCD_PF_TRACE
// dev instrumentation (variant builds only): clock64 stamps of one CTA's
// pipeline events per key block -- see scripts/pf_trace.py
__device__ long long g_pf_trace[256][8];
#define PF_TRACE(e, j)                                                                                   \
  do {                                                                                                   \
    if (blockIdx.y == 0 && (int)blockIdx.x == (int)gridDim.x / 2 && (j) < 256) g_pf_trace[(j)][(e)] = clock64(); \
  } while (0)
#else
#define PF_TRACE(e, j) \
  do {                 \
  } while (0)
#endif

// bars: 0 q_full | 1-2 k_full[s] | 3-4 v_full[s] | 5-6 kv_empty[s] |
//       7-8 s_full[t] | 9-10 p_full[t] | 11-12 o_done[t] |
//       13-14 k_empty[s] (sparse: the K half of a stage frees once S of
//       both tiles retired, long before PV frees the V half)
template <int MODE>
__global__ void __launch_bounds__(pf::kThreads, 1)
    prefill_attn_kernel(const __grid_constant__ PrefillTmaps tm, const PrefillArgs a) {
  using namespace pf;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round
  // trip would hide the address space and turn shared loads into generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  int* posbuf = reinterpret_cast<int*>(smem + kOffPos);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = (a.N + kTileM - 1) / kTileM;
  const int ti = num_tiles - 1 - (int)blockIdx.x;     // heavy (late) tiles first
  const int r0 = ti * kTileM;
  const int nslots = a.slots;                          // 2 (G even) or 1
  const int h0 = blockIdx.y * nslots;
  const int g = h0 / a.G;

  // key blocks this tile visits
  int count = 0;                                       // sparse: selected entries
  const int* sel = nullptr;
  int nb;
  if (MODE == PMODE_SPARSE) {
    // Programmatic dependent launch between consecutive reuse layers: the
    // next layer's CTAs may take SMs as ours retire.  Inputs are complete at
    // launch (per-layer Q/K/V; index lists from a select launch that never
    // triggers early) and each layer writes its own output, so only the
    // optional LSE side output (shared) waits for the previous grid.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int src = a.head_map ? __ldg(a.head_map + g) : g;
    sel = a.idx + (int64_t)src * a.idx_sg + (int64_t)ti * a.idx_st;
    count = min(__ldg(a.cnt + (int64_t)src * a.cnt_sg + ti), a.k_cap);
    nb = (count + kBlockN - 1) / kBlockN;
  } else {
    const int kend = a.causal ? min(a.N, r0 + kTileM) : a.N;
    nb = (kend + kBlockN - 1) / kBlockN;
  }

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars[1 + s], MODE == PMODE_SPARSE ? 96 : 1);
      mbar_init(&bars[3 + s], MODE == PMODE_SPARSE ? 96 : 1);
      mbar_init(&bars[5 + s], 1);
      if (MODE == PMODE_SPARSE) mbar_init(&bars[13 + s], 1);
    }
    if (MODE == PMODE_LSE) {
      // no O: each tile double-buffers S; s_full(t,b) = 7+t+2b, p_full(t,b) = 11+t+2b
      for (int i = 0; i < 4; ++i) {
        mbar_init(&bars[7 + i], 1);
        mbar_init(&bars[11 + i], 128);
      }
    } else {
      for (int t = 0; t < 2; ++t) {
        mbar_init(&bars[7 + t], 1);
        mbar_init(&bars[9 + t], 128);
        mbar_init(&bars[11 + t], 1);
      }
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;\n");
    // ================================================ producers / MMA
    if (warp == 3) {
      if (lane == 0 && nb > 0) {
        // --------------------------------------------------- MMA issuer
        const uint32_t qaddr = smem_u32(smem + kOffQ);
        const uint32_t kaddr = smem_u32(smem + kOffK);
        const uint32_t vaddr = smem_u32(smem + kOffV);
        auto issue_s = [&](int t, int st) {
          const uint32_t d = tmem + t * 256;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t off = (ks >> 2) * kHalf + (ks & 3) * 32;
            mma_ss(d, sw128_desc(qaddr + t * kTileBytes + off, 16, 1024),
                   sw128_desc(kaddr + st * kTileBytes + off, 16, 1024), kIdescS, ks > 0);
          }
          mma_commit(&bars[7 + t]);
        };
        auto issue_pv = [&](int t, int st, int j) {
          const uint32_t d = tmem + t * 256 + 128;
          const uint32_t p = tmem + t * 256;
          mbar_wait(&bars[9 + t], j & 1);          // P_t(j) written
          PF_TRACE(2 * t, j);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            mma_ts(d, p + ks * 8, sw128_desc(vaddr + st * kTileBytes + ks * 2048, kHalf, 1024), kIdescPV,
                   (j > 0 || ks > 0) ? 1u : 0u);
          }
        };
        mbar_wait(&bars[0], 0);
        if (MODE == PMODE_LSE) {
          // S only: block j goes to buffer j&1 of each tile as soon as the
          // softmax has drained that buffer (block j-2), so the tensor core
          // runs a block ahead of the exponentials.
          for (int j = 0; j < nb; ++j) {
            const int st = j % kStages, b = j & 1;
            mbar_wait(&bars[1 + st], (j / kStages) & 1);
            for (int t = 0; t < nslots; ++t) {
              if (j >= 2) mbar_wait(&bars[11 + t + 2 * b], ((j >> 1) - 1) & 1);
              tc_fence_after();
              const uint32_t d = tmem + t * 256 + b * 128;
#pragma unroll
              for (int ks = 0; ks < 8; ++ks) {
                const uint32_t off = (ks >> 2) * kHalf + (ks & 3) * 32;
                mma_ss(d, sw128_desc(qaddr + t * kTileBytes + off, 16, 1024),
                       sw128_desc(kaddr + st * kTileBytes + off, 16, 1024), kIdescS, ks > 0);
              }
              mma_commit(&bars[7 + t + 2 * b]);
            }
            mma_commit(&bars[5 + st]);
          }
        }
        if (MODE != PMODE_LSE) {
        mbar_wait(&bars[1], 0);
        tc_fence_after();
        for (int t = 0; t < nslots; ++t) issue_s(t, 0);
        if (MODE == PMODE_SPARSE) mma_commit(&bars[13]);
        for (int j = 0; j < nb; ++j) {
          const int st = j % kStages;
          const uint32_t ph = (j / kStages) & 1;
          const bool more = j + 1 < nb;
          const int st1 = (j + 1) % kStages;
          const uint32_t ph1 = ((j + 1) / kStages) & 1;
          if (MODE != PMODE_LSE) mbar_wait(&bars[3 + st], ph);
          // tile 0: PV_j, then S_{j+1}
          if (MODE != PMODE_LSE) {
            issue_pv(0, st, j);
            if (j == nb - 1) mma_commit(&bars[11]);
          }
          if (more) {
            mbar_wait(&bars[1 + st1], ph1);
            tc_fence_after();
            issue_s(0, st1);
            PF_TRACE(1, j);
          }
          if (nslots == 2) {
            if (MODE != PMODE_LSE) {
              issue_pv(1, st, j);
              if (j == nb - 1) mma_commit(&bars[12]);
            }
          }
          mma_commit(&bars[5 + st]);   // K/V stage free once everything so far retires
          if (more && nslots == 2) {
            issue_s(1, st1);
            PF_TRACE(3, j);
          }
          if (MODE == PMODE_SPARSE && more) mma_commit(&bars[13 + st1]);   // K_{j+1} consumed by both S
        }
        }  // MODE != PMODE_LSE
      }
    } else if (MODE != PMODE_SPARSE) {
      if (warp == 0 && lane == 0 && nb > 0) {
        // ----------------------------------------------- TMA producer
        tma_prefetch(&tm.q);
        tma_prefetch(&tm.k);
        tma_prefetch(&tm.v);
        mbar_expect_tx(&bars[0], nslots * kTileBytes);
        for (int t = 0; t < nslots; ++t)
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d(smem + kOffQ + t * kTileBytes + hf * kHalf, &tm.q, &bars[0], hf * 64, r0, h0 + t);
        for (int j = 0; j < nb; ++j) {
          const int st = j % kStages;
          if (j >= kStages) mbar_wait(&bars[5 + st], ((j / kStages) - 1) & 1);
          mbar_expect_tx(&bars[1 + st], kTileBytes);
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d(smem + kOffK + st * kTileBytes + hf * kHalf, &tm.k, &bars[1 + st], hf * 64, j * kBlockN, g);
          if (MODE != PMODE_LSE) {
            mbar_expect_tx(&bars[3 + st], kTileBytes);
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d(smem + kOffV + st * kTileBytes + hf * kHalf, &tm.v, &bars[3 + st], hf * 64,
                          j * kBlockN, g);
          }
        }
      }
    } else {
      // ------------------------------------- sparse gather producers (96)
      const int pt = threadIdx.x;  // 0..95
      if (pt == 0 && nb > 0) {
        tma_prefetch(&tm.q);
        mbar_expect_tx(&bars[0], nslots * kTileBytes);
        for (int t = 0; t < nslots; ++t)
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d(smem + kOffQ + t * kTileBytes + hf * kHalf, &tm.q, &bars[0], hf * 64, r0, h0 + t);
      }
      // Block j's rows are gathered while the tensor core and the softmax
      // warpgroups work on block j-1 (double buffering); completion is
      // published per block (wait_group, proxy fence, mbarrier arrive) so the
      // tensor core reads coherent shared memory.
      const __nv_bfloat16* kg = a.k + (int64_t)g * a.kv_sh;
      const __nv_bfloat16* vg = a.v + (int64_t)g * a.kv_sh;
      // The selection entries of block j+1 are loaded into registers while
      // block j's rows are in flight, so the dependent index load never sits
      // on the stage-free -> gather -> publish critical path.
      const int r1 = pt + 96;                       // second row of threads 0..31
      auto load_sel = [&](int j, int& p0, int& p1) {
        const int e0 = j * kBlockN + pt, e1 = j * kBlockN + r1;
        p0 = e0 < count ? __ldg(sel + e0) : 0x7fffffff;
        p1 = (r1 < kBlockN && e1 < count) ? __ldg(sel + e1) : 0x7fffffff;
      };
      int p0 = 0x7fffffff, p1 = 0x7fffffff;
      if (nb > 0) load_sel(0, p0, p1);
      // Cp.async groups retire in order K_0, V_0, K_1, V_1, ...: K_j is
      // gathered as soon as S_{j-2} released its half-stage and is published
      // first; V_{j-1} is published while K_j is in flight.
      // 128 rows x 16 chunks over 96 threads: thread pt always copies chunk
      // pt % 16 (96 is a multiple of 16) of rows pt / 16 + 6 i.  Its <= 22
      // positions are read from shared memory once per block, all loads in
      // flight together, and reused by the K and the V gather -- a position
      // load per copy (dependent LDS -> address -> LDGSTS) was the gather's
      // dominant stall (ncu: short scoreboard; 14.3 -> 12.6 ms at 128K).
      constexpr int kRowsPer = (kBlockN + 5) / 6;               // 22
      const int gch = pt & 15, grow0 = pt >> 4;
      int prow[kRowsPer];
      auto load_rows = [&](const int* pos) {
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          const int r = grow0 + 6 * i;
          prow[i] = r < kBlockN ? pos[r] : 0x7fffffff;
        }
      };
      auto gather = [&](uint32_t dst, const __nv_bfloat16* src) {
#pragma unroll
        for (int i = 0; i < kRowsPer; ++i) {
          const int r = grow0 + 6 * i;
          if (r < kBlockN) {
            const int p = prow[i];
            const bool valid = p != 0x7fffffff;
            const uint32_t off = (gch >> 3) * kHalf + r * 128 + (((gch & 7) ^ (r & 7)) << 4);
            cp_async16_zfill(dst + off, src + (int64_t)(valid ? p : 0) * 128 + gch * 8, valid);
          }
        }
        cp_async_commit();
      };
      for (int j = 0; j < nb; ++j) {
        const int st = j % kStages;
        const uint32_t ph_free = ((j / kStages) - 1) & 1;
        if (j >= kStages) mbar_wait(&bars[13 + st], ph_free);    // K half of the stage free
        int* pos = posbuf + (j % kPosBufs) * 128;
        pos[pt] = p0;
        if (r1 < kBlockN) pos[r1] = p1;
        if (j + 1 < nb) load_sel(j + 1, p0, p1);
        named_bar_sync(1, 96);
        load_rows(pos);
        gather(smem_u32(smem + kOffK + st * kTileBytes), kg);
        if (j > 0) {                                              // V_{j-1} landed
          cp_async_wait<1>();
          fence_proxy_async_smem();
          mbar_arrive(&bars[3 + (j - 1) % kStages]);
        }
        if (j >= kStages) mbar_wait(&bars[5 + st], ph_free);     // V half free (PV_{j-2} retired)
        gather(smem_u32(smem + kOffV + st * kTileBytes), vg);
        cp_async_wait<1>();                                       // K_j landed
        fence_proxy_async_smem();
        mbar_arrive(&bars[1 + st]);
      }
      if (nb > 0) {
        cp_async_wait<0>();
        fence_proxy_async_smem();
        mbar_arrive(&bars[3 + (nb - 1) % kStages]);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n");
    // ================================================== softmax warpgroups
    const int t = (warp - 4) >> 2;          // tile slot
    const int q = warp & 3;                 // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;
    const int row = r0 + row_in_tile;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t s_col = t * 256, o_col = t * 256 + 128;
    if (t < nslots) {
      const int h = h0 + t;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        // LSE mode: S double-buffered (buffer j&1, its own barrier pair)
        const int sb = MODE == PMODE_LSE ? 7 + t + 2 * (j & 1) : 7 + t;
        const uint32_t s_off = MODE == PMODE_LSE ? 128 * (j & 1) : 0;
        mbar_wait(&bars[sb], MODE == PMODE_LSE ? (j >> 1) & 1 : j & 1);
        if (lane == 0 && q == 0) PF_TRACE(4 + 2 * t, j);
        tc_fence_after();
        // the whole 128-key row of S in one batch of TMEM loads, one wait
        float s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld32(lane_base + s_col + s_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
        tmem_ld_wait();
        // masking on raw scores: keys past the end / after the row (causal) /
        // unselected.  Sorted selections only reach the tile's own rows in
        // their last block(s), so earlier blocks skip the per-key test.
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
          const int lim = a.causal ? min(row, a.N - 1) : a.N - 1;   // last visible key
          if (k0 + kBlockN - 1 > lim) {
#pragma unroll
            for (int c = 0; c < 128; ++c)
              if (k0 + c > lim) s[c] = -INFINITY;
          }
        }
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
        float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};   // 4 independent FADD2 chains
        // p = exp2(s*scale*log2e - m): one packed FFMA2 per key pair + MUFU,
        // P (bf16 pairs) over S in TMEM; the row sum into sum4
        auto exps = [&](float mu) {
          const float2 nm2 = make_float2(-mu, -mu);
#pragma unroll
          for (int i = 0; i < 4; ++i) sum4[i] = make_float2(0.f, 0.f);
          if (MODE == PMODE_LSE) {
#pragma unroll
            for (int c = 0; c < 128; c += 2) {
              const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sc2, nm2);
              sum4[(c >> 1) & 3] = __fadd2_rn(sum4[(c >> 1) & 3], exp2_pair_sum<KSCD_LSE_POLY>(x, c >> 1));
            }
          } else {
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
              // 16 packed columns: the key pairs of this 32-key chunk
              asm volatile(
                  "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                  ::"r"(lane_base + s_col + c * 16), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
                  "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
                  "r"(r[13]), "r"(r[14]), "r"(r[15])
                  : "memory");
            }
          }
        };
        // Lazy rescale: a row moves its reference max only when the block max
        // exceeds it by > 2^8.  The exponentials are taken against the current
        // reference first; every p <= 2^8 (sum <= 2^8 proves it) means no key
        // exceeded the reference by > 2^8, which is exactly the no-rescale
        // case, so the block max is never formed then (no FMNMX on the
        // per-tile chain).  Otherwise -- and while a row has no reference --
        // the warp takes the exact path: block max, the same rescale rule,
        // the block redone.  tcgen05.ld/st are warp-collective, so the O
        // correction runs for the whole warp (alpha = 1 for the other rows).
        bool slow = m_used == -INFINITY;
        if (!__all_sync(0xffffffffu, slow)) {
          exps(m_used == -INFINITY ? 0.f : m_used);
          const float2 t2 = __fadd2_rn(__fadd2_rn(sum4[0], sum4[1]), __fadd2_rn(sum4[2], sum4[3]));
          slow = slow || t2.x + t2.y > 256.f;
        }
        if (__any_sync(0xffffffffu, slow)) {
          const float mx = max_tree<128>(s) * a.scale_log2;   // scale > 0: max commutes
          const bool need = mx > m_used + kRescaleThreshold;
          const float alpha = (need && m_used != -INFINITY) ? exp2f(m_used - mx) : 1.f;
          if (MODE != PMODE_LSE) tmem_st_wait();              // speculative P landed before it is redone
          if (MODE != PMODE_LSE && __any_sync(0xffffffffu, alpha != 1.f)) {
            // O_t holds blocks < j (their PV completed before S_j was committed)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t r[32];
              tmem_ld32(lane_base + o_col + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              tmem_st32(lane_base + o_col + c * 32, r);
            }
          }
          l *= alpha;
          if (need) m_used = mx;
          exps(m_used == -INFINITY ? 0.f : m_used);
        }
        if (MODE != PMODE_LSE) tmem_st_wait();
        const float2 sum2 = __fadd2_rn(__fadd2_rn(sum4[0], sum4[1]), __fadd2_rn(sum4[2], sum4[3]));
        l += sum2.x + sum2.y;
        tc_fence_before();
        if (lane == 0 && q == 0) PF_TRACE(5 + 2 * t, j);
        mbar_arrive(&bars[MODE == PMODE_LSE ? 11 + t + 2 * (j & 1) : 9 + t]);
      }
      // ---------------------------------------------------------- epilogue
      const bool live = row < a.N;
      if (MODE != PMODE_LSE && nb > 0) {
        mbar_wait(&bars[11 + t], 0);
        tc_fence_after();
      }
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (MODE != PMODE_LSE) {
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
              // attention.py:248-252: no selected key visible -> V[g][row]
              const uint4* vrow = reinterpret_cast<const uint4*>(a.v + (int64_t)g * a.kv_sh + (int64_t)row * 128 + c * 32);
#pragma unroll
              for (int i = 0; i < 4; ++i) w[i] = __ldg(vrow + i);
            }
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = w[i];
          }
        }
      }
      if (MODE == PMODE_SPARSE && a.lse) asm volatile("griddepcontrol.wait;\n" ::: "memory");
      if (live && a.lse) a.lse[(int64_t)h * a.N + row] = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool make_prefill_map_box(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride, int box_rows);

// [heads][rows][128] bf16 with row stride 128 and head stride `head_stride`
// elements, box {64, 128, 1}, 128B swizzle.
bool make_prefill_map(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride) {
  return make_prefill_map_box(m, base, heads, rows, head_stride, 128);
}

bool make_prefill_map_box(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)heads};
  cuuint64_t strides[2] = {256, (cuuint64_t)head_stride * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE>
static cudaError_t launch_prefill_mode(const PrefillArgs& a, cudaStream_t st) {
  PrefillTmaps tm;
  if (!make_prefill_map(&tm.q, a.q, a.Hq, a.N, a.q_sh)) return cudaErrorInvalidValue;
  if (!make_prefill_map(&tm.k, a.k, a.Hkv, a.Nk, a.kv_sh)) return cudaErrorInvalidValue;
  if (!make_prefill_map(&tm.v, a.v, a.Hkv, a.Nk, a.kv_sh)) return cudaErrorInvalidValue;
  static const cudaError_t attr = cudaFuncSetAttribute(prefill_attn_kernel<MODE>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, pf::kSmemBytes);
  if (attr != cudaSuccess) return attr;
  const int tiles = (a.N + pf::kTileM - 1) / pf::kTileM;
  dim3 grid(tiles, a.Hq / a.slots);
  if (MODE != PMODE_SPARSE) {
    prefill_attn_kernel<MODE><<<grid, pf::kThreads, pf::kSmemBytes, st>>>(tm, a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(pf::kThreads);
  cfg.dynamicSmemBytes = pf::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, prefill_attn_kernel<MODE>, tm, a);
}

#ifdef KSCD_PF_TRACE
extern "C" int kscd_debug_pf_trace(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_pf_trace, sizeof(g_pf_trace));
}
extern "C" int kscd_debug_pf_trace_reset() {
  static long long zeros[256][8];
  return (int)cudaMemcpyToSymbol(g_pf_trace, zeros, sizeof(zeros));
}
#endif

cudaError_t launch_prefill_attn(int mode, const PrefillArgs& a, cudaStream_t st) {
  // (a CTA-pair variant on 2-SM UMMA was measured slower and removed)
  switch (mode) {
    case PMODE_DENSE: return launch_prefill_mode<PMODE_DENSE>(a, st);
    case PMODE_SPARSE: return launch_prefill_mode<PMODE_SPARSE>(a, st);
    default: return launch_prefill_mode<PMODE_LSE>(a, st);
  }
}

}  // namespace kscd
