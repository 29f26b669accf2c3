// Anchor-layer decode attention on the 5th-gen tensor cores: the dense pass
// (layer 0, and the Top-k = 100 % baseline) and the anchor score pass, with
// TMA-fed K / V blocks and tcgen05 MMAs accumulating in TMEM
// (dense_attention's last row, attention.py:106-144; north_star (1)).
//
// One query token per sequence, so the query heads of a kv group (G <= 16)
// are the SMALL side of every product.  Keys go on the UMMA M dimension:
//
//   S^T[key][h] = K_blk . Q^T      M = 128 keys, N = 16 (heads, padded), K = d
//   O^T[d][h]  += V_blk^T . P^T     M = 128 (d),  N = 16,                 K = 128 keys
//
// so the MMA shapes are M128 x N16 (legal kind::f16 shapes) instead of a
// 4-row M tile, S^T (2 buffers) and O^T (2 buffers) live in TMEM (64
// columns), and a softmax thread owns one key (TMEM lane) -- and, for O^T,
// one dimension.
// V^T is the V block as TMA stored it ([key][d], SW128), read as an MN-major
// A operand; P^T (bf16, [head][key], SW128) is written by the softmax threads
// into shared memory as the K-major B operand.  The kernel is HBM-bound:
// 3 K + 3 V slots (dense) or 6 K slots (scores) of 32 KB TMA tile loads keep
// up to 192 KB in flight per SM; a K slot frees when S^T retires, a V slot
// when PV does.
//
// Roles (224 threads): warp 0 lane 0 issues the Q and K loads, warp 6 lane 0
// the V loads, warp 1 lane 0 the MMAs (warp 1 owns the TMEM allocation),
// warps 2-5 are the softmax / epilogue threads (TMEM lane quarters 2, 3, 0,
// 1).  Per key block j:
//
//   MMA:      S^T_j -> TMEM buffer j&1 ; then PV_{j-1} (after P_{j-1})
//   softmax:  load S^T_j; one OR vote whether any key exceeds the running
//             reference by > 2^8 -- only then the CTA-wide block max (warp
//             shuffles + 4-warp smem) and a rescale of O^T in TMEM;
//             p = exp2(s - m), P^T_j (bf16) -> smem buffer j&1
//   score pass (no V): every thread keeps its own lazy reference (no
//             barrier), merged per head in the epilogue
//
// Work split ("stream-K"): a layer's (sequence, kv head, 128-key block)
// space is cut into equal contiguous ranges, waves of CTAs per layer.  A
// CTA streams its range without draining at pair boundaries (Q of each pair
// by TMA into a segment-parity buffer, O^T double-buffered in TMEM); each
// pair it touches is a segment whose partial (m, l, O / l_bf16) goes to the
// executor's split-K workspace, and the last segment of a pair to finish
// merges them in slot order (deterministic; a layer's ranges do not depend
// on how many layers share the launch).  O is normalised by the sum of the
// bf16-rounded weights the MMA multiplied, the LSE by the fp32 sum.
#include "sm100.cuh"
#include "kscd_internal.h"

namespace kscd {
using namespace sm100;

namespace dtc {
constexpr int kBlk = 128;                 // keys per block = UMMA M
constexpr int kN = 16;                    // UMMA N: the group's heads, padded
constexpr int kThreads = 224;             // 7 warps: K/Q TMA, MMA, 4 softmax, V TMA
constexpr int kTile = kBlk * 256;         // one K or V block, 32 KB
constexpr int kHalf = kBlk * 128;         // one 64-column half of a block
constexpr int kQBytes = 2 * kN * 128;     // Q of a group: [2 halves][16 rows][128 B]
constexpr int kMaxSplits = 64;
// CTAs per layer: waves of one CTA per SM (the block scheduler balances SMs
// of unequal speed, and more, shorter CTAs let a launch's tail overlap the
// next launch's start).  The score pass and single-layer dense launches
// (anchor 0) use 16 waves per layer; the multi-layer dense launches (the
// Top-k = 100 % baseline) 4 waves per layer.  A score pass's ranges (so its
// LSE rounding) therefore never depend on how many layers share its launch;
// a dense layer's do (split-K rounding only).  Measured in the 128K b8 decode step (same box, A/B): 4 / 6 / 8 /
// 12 / 16 / 24 waves for the single-layer launches 573.9 / 568.4 / 565.6 /
// 565.2 / 564.2 / 565.5 us/token (a (sequence, kv head) spans at most its
// partial-slot count of ranges -- 20 for 64 pairs -- so 8 and more requested
// waves all land near 8.2 there), while the all-layer dense baseline launches
// lose 2 % above 4 waves per layer; 1 wave and a persistent grid fed by an
// atomic chunk queue were +4 % (round-2 history).
constexpr int kWavesSingle = 16;
constexpr int kWavesMultiDense = 4;
constexpr uint32_t kIdescS = idesc_bf16(128, kN, false, false);   // A = K (K-major), B = Q (K-major)
constexpr uint32_t kIdescO = idesc_bf16(128, kN, true, false);    // A = V^T (MN-major), B = P^T (K-major)
constexpr float kRescale = 8.0f;          // log2 units

template <bool HAS_V>
struct Cfg {
  // K slots free when S^T retires, V slots only when PV does (a 2 / 4
  // split measured the same as 3 / 3)
  static constexpr int kSK = HAS_V ? 3 : 6;
  static constexpr int kSV = HAS_V ? 3 : 0;
  static constexpr int kStages = kSK > kSV ? kSK : kSV;    // barrier slots
  static constexpr int kOffV = kSK * kTile;
  static constexpr int kOffQ = (kSK + kSV) * kTile;        // 2 segment buffers of kQBytes
  static constexpr int kOffP = kOffQ + 2 * kQBytes;        // 2 block buffers of P^T [2 halves][16][128 B]
  static constexpr int kOffRed = kOffP + 8192;             // float [2][4 warps][16] block max
  static constexpr int kOffSum = kOffRed + 2 * 4 * 16 * 4; // float [4][16] l, [4][16] l (bf16 p), [16] m
  static constexpr int kOffW = kOffSum + 144 * 4;          // float [4 warps][64] merge weights
  static constexpr int kOffBar = kOffW + 4 * kMaxSplits * 4;
  static constexpr int kNumBars = 4 * kStages + 16;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;
};

// A layer's work is a flat space of 128-key blocks f = (b * Hkv + g) * nblk
// + j (see the header); blocks past a ragged sequence's length are skipped.
struct Walk {
  int nblk, P, Hkv, n;
  const int* lens;
  KSCD_DEV int blocks_of(int pair) const {
    if (!lens) return (n + kBlk - 1) / kBlk;
    const int b = (pair % P) / Hkv;
    const int cnt = max(0, min(__ldg(lens + b), n));
    return (cnt + kBlk - 1) / kBlk;
  }
};
}  // namespace dtc

// 32 lanes x 16 consecutive 32-bit columns
KSCD_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
KSCD_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
KSCD_DEV void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// named barrier with an OR vote over the participating threads
KSCD_DEV bool bar_any(uint32_t id, uint32_t nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 q, %1, 0;\n barrier.cta.red.or.pred p, %2, %3, q;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}

// Byte offset of element (row, col) in a [2 halves of 64 cols][rows][128 B]
// SWIZZLE_128B tile (16-byte chunks XOR-permuted by row % 8): the canonical
// K-major layout UMMA reads for P^T (rows = heads, cols = keys).
KSCD_DEV uint32_t sw128_off(int row, int col, int rows) {
  const int half = col >> 6, c = col & 63;
  return half * rows * 128 + row * 128 + ((((c >> 3) ^ (row & 7)) & 7) << 4) + (c & 7) * 2;
}

// bars: full[S] / empty[S] (K slots), then pairs s_full, s_free, p_full,
//       pv_done (by block parity), q_full, q_free, o_done, o_free (by segment
//       parity), then vfull[S] / vempty[S] (V slots: a block's K slot frees
//       when S^T retires, its V slot when PV retires)
//
// GM: the query heads per group rounded up to a power of two (<= 16); the
// softmax threads only touch those S^T / O^T columns and P^T rows.
template <int MODE, int GM>
__global__ void __launch_bounds__(dtc::kThreads, 1)
    decode_tc_kernel(const __grid_constant__ DecodeTmaps tm, const DecodeArgs a, const int per) {
  using namespace dtc;
  constexpr bool HAS_V = MODE == MODE_DENSE;
  using C = Cfg<HAS_V>;
  constexpr int S = C::kSK, SV = C::kSV > 0 ? C::kSV : 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* s_full = bars + 2 * S;
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_full + 4;
  uint64_t* pv_done = s_full + 6;
  uint64_t* q_full = s_full + 8;
  uint64_t* q_free = s_full + 10;
  uint64_t* o_done = s_full + 12;
  uint64_t* o_free = s_full + 14;
  uint64_t* vfull = s_full + 16;
  uint64_t* vempty = vfull + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);
  int* flag = reinterpret_cast<int*>(smem + C::kOffTmem + 8);
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  float* lred = reinterpret_cast<float*>(smem + C::kOffSum);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int P = a.B * a.Hkv;
  const Walk w{(a.n + kBlk - 1) / kBlk, P, a.Hkv, a.n, a.lens};
  const int nblk = w.nblk;
  // Within a launch every layer's block space is cut identically into
  // ranges of `per` blocks (see kWavesSingle for when the cut depends on the
  // launch): CTA (layer, c) streams range c of that layer -- waves of one
  // CTA per SM, so the block scheduler balances SMs of unequal speed.  Its
  // pairs (segments) are the layer-local pairs [pl0, pl0 + nv), each over
  // blocks [jb, je).
  const int cpl = (P * nblk + per - 1) / per;
  const int lyr_c = blockIdx.x / cpl, cta = blockIdx.x - lyr_c * cpl;
  const int T1 = P * nblk;
  const int g0 = cta * per, g1 = min(T1, g0 + per);
  const int pl0 = g0 / nblk, nv = (g1 + nblk - 1) / nblk - pl0;
  auto pair_of = [&](int v) { return lyr_c * P + pl0 + v; };
  auto seg_range = [&](int pair, int& jb, int& je) {
    const int pl = pair % P;
    jb = max(g0 - pl * nblk, 0);
    je = min(g1 - pl * nblk, w.blocks_of(pair));
  };

  // PDL: our inputs (q, caches) are complete when we start (as decode.cu);
  // only the workspace / output writes wait for the previous grid
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kNumBars; ++s) {
      const uint64_t* bp = &bars[s];
      const bool by_threads = (bp >= s_free && bp < s_free + 2) || (bp >= p_full && bp < p_full + 2) ||
                              (bp >= o_free && bp < o_free + 2);
      mbar_init(&bars[s], by_threads ? 128 : 1);   // softmax-thread arrivals vs one arrive / commit
    }
    fence_barrier_init();
  }
  if (HAS_V && GM < kN) {
    // P^T rows >= GM are never written: zero them once
    for (int i = threadIdx.x; i < 2 * 4096 / 16; i += kThreads) {
      const int row = (i >> 3) & 15;
      if (row >= GM) reinterpret_cast<uint4*>(smem + C::kOffP)[i] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;          // cols [0,16) S0 | [16,32) S1 | [32,48) O^T 0 | [48,64) O^T 1

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm.q);
      int i = 0, s = 0;
      for (int v = 0; v < nv; ++v) {
        const int pair = pair_of(v);
        int jb, je;
        seg_range(pair, jb, je);
        if (jb >= je) continue;
        const int lyr = pair / P, rem = pair - lyr * P, b = rem / a.Hkv, g = rem - b * a.Hkv;
        const int gk = g / a.kv_rep;
        const CUtensorMap* kmap = &tm.k[lyr];
        const int qb = s & 1;                 // the segment's group Q rows
        if (s >= 2) mbar_wait(&q_free[qb], ((s - 2) >> 1) & 1);
        mbar_expect_tx(&q_full[qb], kQBytes);
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(smem + C::kOffQ + qb * kQBytes + hf * 2048, &tm.q, &q_full[qb], hf * 64, b * a.Hq + g * G, lyr);
        for (int j = jb; j < je; ++j, ++i) {
          const int st = i % S;
          if (i >= S) mbar_wait(&empty[st], ((i / S) - 1) & 1);
          mbar_expect_tx(&full[st], kTile);
          uint8_t* dst = smem + st * kTile;
          for (int hf = 0; hf < 2; ++hf) tma_load_4d(dst + hf * kHalf, kmap, &full[st], hf * 64, j * kBlk, gk, b);
        }
        ++s;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t qaddr0 = smem_u32(smem + C::kOffQ);
      const uint32_t paddr = smem_u32(smem + C::kOffP);
      // O^T_seg += V_ii^T P_ii^T
      auto issue_pv = [&](int ii, int seg, bool first, bool last) {
        const int pb = ii & 1, ob = seg & 1, st = ii % SV;
        if (first && seg >= 2) mbar_wait(&o_free[ob], ((seg - 2) >> 1) & 1);
        mbar_wait(&vfull[st], (ii / SV) & 1);
        mbar_wait(&p_full[pb], (ii >> 1) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(smem + C::kOffV + st * kTile);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + 32 + ob * 16, sw128_desc(vaddr + ks * 2048, kHalf, 1024),
                 sw128_desc(paddr + pb * 4096 + (ks >> 2) * 2048 + (ks & 3) * 32, 16, 1024), kIdescO,
                 (!first || ks > 0) ? 1u : 0u);
        mma_commit(&pv_done[pb]);
        mma_commit(&vempty[st]);
        if (last) mma_commit(&o_done[ob]);
      };
      int i = 0, s = 0, pseg = 0;
      bool pfirst = false, plast = false;
      for (int v = 0; v < nv; ++v) {
        const int pair = pair_of(v);
        int jb, je;
        seg_range(pair, jb, je);
        if (jb >= je) continue;
        mbar_wait(&q_full[s & 1], (s >> 1) & 1);
        const uint32_t qaddr = qaddr0 + (s & 1) * kQBytes;
        for (int j = jb; j < je; ++j, ++i) {
          const int st = i % S, sb = i & 1;
          mbar_wait(&full[st], (i / S) & 1);
          if (i >= 2) mbar_wait(&s_free[sb], ((i - 2) >> 1) & 1);
          tc_fence_after();
          const uint32_t kaddr = smem_u32(smem + st * kTile);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t off = (ks >> 2) * kHalf + (ks & 3) * 32;
            mma_ss(tmem + sb * 16, sw128_desc(kaddr + off, 16, 1024),
                   sw128_desc(qaddr + (ks >> 2) * 2048 + (ks & 3) * 32, 16, 1024), kIdescS, ks > 0);
          }
          mma_commit(&s_full[sb]);
          if (j == je - 1) mma_commit(&q_free[s & 1]);
          mma_commit(&empty[st]);                 // K consumed once S^T retires
          if (HAS_V && i > 0) issue_pv(i - 1, pseg, pfirst, plast);
          pseg = s;
          pfirst = j == jb;
          plast = j == je - 1;
        }
        ++s;
      }
      if (HAS_V && i > 0) issue_pv(i - 1, pseg, pfirst, plast);
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------- V TMA producer
    if (HAS_V && lane == 0) {
      int i = 0;
      for (int v = 0; v < nv; ++v) {
        const int pair = pair_of(v);
        int jb, je;
        seg_range(pair, jb, je);
        if (jb >= je) continue;
        const int lyr = pair / P, rem = pair - lyr * P, b = rem / a.Hkv, g = rem - b * a.Hkv;
        const int gk = g / a.kv_rep;
        const CUtensorMap* vmap = &tm.v[lyr];
        for (int j = jb; j < je; ++j, ++i) {
          const int st = i % SV;
          if (i >= SV) mbar_wait(&vempty[st], ((i / SV) - 1) & 1);
          mbar_expect_tx(&vfull[st], kTile);
          uint8_t* dst = smem + C::kOffV + st * kTile;
          for (int hf = 0; hf < 2; ++hf) tma_load_4d(dst + hf * kHalf, vmap, &vfull[st], hf * 64, j * kBlk, gk, b);
        }
      }
    }
  } else {
    // ------------------------------------------------------ softmax / epilogue
    const int qw = warp & 3;                          // TMEM lane quarter
    const int wi = warp - 2;                          // softmax warp 0..3
    const int kin = qw * 32 + lane;                   // key within the block / dim of O^T
    const uint32_t lane_base = tmem + ((uint32_t)(qw * 32) << 16);
    float* wsp = reinterpret_cast<float*>(smem + C::kOffW) + wi * kMaxSplits;
    bool waited = false;
    int i = 0, s = 0;
    for (int v = 0; v < nv; ++v) {
      const int pair = pair_of(v);
      int jb, je;
      seg_range(pair, jb, je);
      const int lyr = pair / P, rem = pair - lyr * P, b = rem / a.Hkv, g = rem - b * a.Hkv;
      const int64_t bh0 = (int64_t)b * a.Hq + (int64_t)g * G;
      float* out_l = a.out ? a.out + (int64_t)lyr * a.out_ls : nullptr;
      float* lse_l = a.lse ? a.lse + (int64_t)lyr * a.lse_ls : nullptr;
      if (jb >= je) {
        // a pair with no keys at all (ragged length 0) whose first block
        // lies in this CTA's range: zero output, lse = -inf
        if (w.blocks_of(pair) == 0 && (pair % P) * nblk >= g0) {
          if (!waited) {
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            waited = true;
          }
          for (int h = 0; h < G; ++h) {
            if (HAS_V && out_l) out_l[(bh0 + h) * 128 + kin] = 0.f;
            if (kin == 0 && lse_l) lse_l[bh0 + h] = -INFINITY;
          }
        }
        continue;
      }
      const int count = a.lens ? min(__ldg(a.lens + b), a.n) : a.n;
      float* sc_base = a.scores ? a.scores + (int64_t)lyr * a.scores_ls + bh0 * a.score_stride : nullptr;
      float m_used[GM], lsum[GM], lbf[GM];
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        m_used[h] = -INFINITY;
        lsum[h] = 0.f;
        lbf[h] = 0.f;
      }
      for (int j = jb; j < je; ++j, ++i) {
        const int sb = i & 1;
        mbar_wait(&s_full[sb], (i >> 1) & 1);
        tc_fence_after();
        uint32_t r[16];
        tmem_ld16(lane_base + sb * 16, r);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[sb]);
        const int key = j * kBlk + kin;
        const bool valid = key < count;
        float sv[GM];
#pragma unroll
        for (int h = 0; h < GM; ++h) sv[h] = (valid && h < G) ? __uint_as_float(r[h]) * a.scale_log2 : -INFINITY;
        if (sc_base && valid) {
#pragma unroll
          for (int h = 0; h < GM; ++h)
            if (h < G) sc_base[h * a.score_stride + key] = sv[h];
        }
        if (!HAS_V) {
          // score pass: no shared O accumulator, so each thread keeps its own
          // lazy reference per head (merged in the epilogue) -- no barrier
#pragma unroll
          for (int h = 0; h < GM; ++h) {
            if (sv[h] > m_used[h] + kRescale) {
              lsum[h] *= m_used[h] == -INFINITY ? 1.f : fast_exp2(m_used[h] - sv[h]);
              m_used[h] = sv[h];
            }
            lsum[h] += valid && h < G ? fast_exp2(sv[h] - m_used[h]) : 0.f;
          }
          continue;
        }
        // lazy max: the CTA-wide block max is only formed when some key
        // exceeds the running reference by more than 2^8 (one OR vote)
        bool need = false;
#pragma unroll
        for (int h = 0; h < GM; ++h) need |= sv[h] > m_used[h] + kRescale;
        float alpha[GM];
#pragma unroll
        for (int h = 0; h < GM; ++h) alpha[h] = 1.f;
        bool rescaled = false;
        if (bar_any(1, 128, need)) {
          float* rb = red + sb * 64;
#pragma unroll
          for (int h = 0; h < GM; ++h) {
            const float mx = warp_max(sv[h]);
            if (lane == 0) rb[wi * 16 + h] = mx;
          }
          named_bar_sync(1, 128);
#pragma unroll
          for (int h = 0; h < GM; ++h) {
            const float mb = fmaxf(fmaxf(rb[h], rb[16 + h]), fmaxf(rb[32 + h], rb[48 + h]));
            if (mb > m_used[h] + kRescale) {          // uniform across the CTA
              alpha[h] = m_used[h] == -INFINITY ? 1.f : fast_exp2(m_used[h] - mb);
              m_used[h] = mb;
              rescaled = true;
            }
          }
        }
        float p[GM];
#pragma unroll
        for (int h = 0; h < GM; ++h) {
          p[h] = valid && h < G ? fast_exp2(sv[h] - m_used[h]) : 0.f;
          lsum[h] = lsum[h] * alpha[h] + p[h];
        }
        if (HAS_V) {
          if (!valid) {
            // a key past this sequence's length (ragged batch): its V row may
            // hold anything (NaN * 0 would poison O); zero it before PV reads it
            mbar_wait(&vfull[i % SV], (i / SV) & 1);
            uint8_t* vrow = smem + C::kOffV + (i % SV) * kTile + kin * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(vrow)[c] = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(vrow + kHalf)[c] = make_uint4(0, 0, 0, 0);
          }
          if (rescaled && j > jb) {
            // O^T holds this segment's blocks < j: wait for PV_{i-1}, scale each head's column
            mbar_wait(&pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
            tc_fence_after();
            uint32_t o[16];
            tmem_ld16(lane_base + 32 + (s & 1) * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < GM; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * alpha[h]);
            tmem_st16(lane_base + 32 + (s & 1) * 16, o);
            tmem_st_wait();
          }
          if (i >= 2) mbar_wait(&pv_done[sb], ((i - 2) >> 1) & 1);   // P buffer read by PV_{i-2}
          uint8_t* pbuf = smem + C::kOffP + sb * 4096;
#pragma unroll
          for (int h = 0; h < GM; ++h) {
            const __nv_bfloat16 pb = __float2bfloat16_rn(p[h]);
            // O is normalised by the sum of the bf16 weights the MMA used
            lbf[h] = lbf[h] * alpha[h] + __bfloat162float(pb);
            *reinterpret_cast<__nv_bfloat16*>(pbuf + sw128_off(h, kin, kN)) = pb;
          }
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&p_full[sb]);
        }
      }

      // ---- segment epilogue: l per head (4-warp reduce), partial or output --
      if (!HAS_V) {
        // per-thread (m, l) -> one reference per head: the CTA max of the m's
#pragma unroll
        for (int h = 0; h < GM; ++h) {
          const float mw = warp_max(m_used[h]);
          if (lane == 0) red[wi * 16 + h] = mw;
        }
        named_bar_sync(1, 128);
#pragma unroll
        for (int h = 0; h < GM; ++h) {
          const float M = fmaxf(fmaxf(red[h], red[16 + h]), fmaxf(red[32 + h], red[48 + h]));
          lsum[h] = m_used[h] == -INFINITY ? 0.f : lsum[h] * fast_exp2(m_used[h] - M);
          m_used[h] = M;
        }
      }
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        const float t = warp_sum(lsum[h]);
        const float tb = HAS_V ? warp_sum(lbf[h]) : t;
        if (lane == 0) {
          lred[wi * 16 + h] = t;
          lred[64 + wi * 16 + h] = tb;
        }
      }
      if (wi == 0 && lane < GM) {
#pragma unroll
        for (int h = 0; h < GM; ++h)
          if (lane == h) lred[128 + h] = m_used[h];
      }
      named_bar_sync(1, 128);
      float o[GM];
      if (HAS_V) {
        mbar_wait(&o_done[s & 1], (s >> 1) & 1);
        tc_fence_after();
        uint32_t ro[16];
        tmem_ld16(lane_base + 32 + (s & 1) * 16, ro);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&o_free[s & 1]);
#pragma unroll
        for (int h = 0; h < GM; ++h) o[h] = __uint_as_float(ro[h]);
      } else {
#pragma unroll
        for (int h = 0; h < GM; ++h) o[h] = 0.f;
      }
      ++s;
      if (!waited) {
        // the previous grid (PDL) may still use the workspace / outputs
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        waited = true;
      }
      const int pl = pair - lyr * P;                    // pair within the layer
      const int c_first = (pl * nblk) / per;
      const int nseg = (pl * nblk + w.blocks_of(pair) - 1) / per - c_first + 1;
      const int seg = cta - c_first;
      float* part_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part) + (int64_t)lyr * a.ws_ls);
      float* part_ml_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part_ml) + (int64_t)lyr * a.ws_ls);
      const int d = kin;                                // O^T lane = dimension
#pragma unroll
      for (int h = 0; h < GM; ++h) {
        if (h >= G) continue;
        const float L = lred[h] + lred[16 + h] + lred[32 + h] + lred[48 + h];
        const float Lb = lred[64 + h] + lred[80 + h] + lred[96 + h] + lred[112 + h];
        const float M = lred[128 + h];
        const float on = Lb > 0.f ? o[h] / Lb : 0.f;
        if (nseg == 1) {
          if (HAS_V && out_l) out_l[(bh0 + h) * 128 + d] = on;
          if (d == 0 && lse_l) lse_l[bh0 + h] = (M + __log2f(L)) * kLn2;
        } else {
          const int64_t pi = (bh0 + h) * a.splits + seg;
          if (HAS_V) part_l[pi * 128 + d] = on;
          if (d == 0) *reinterpret_cast<float2*>(part_ml_l + pi * 2) = make_float2(M, L);
        }
      }
      if (nseg == 1) continue;
      // the last segment of this (sequence, kv head) to finish merges
      __threadfence();
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) {
        int* ctr = reinterpret_cast<int*>(reinterpret_cast<char*>(a.counters) + (int64_t)lyr * a.ws_ls) +
                   (int64_t)b * a.Hkv + g;
        const int prev_n = atomicAdd(ctr, 1);
        *flag = prev_n == nseg - 1;
        if (*flag) *ctr = 0;                          // re-arm for the next launch / graph replay
      }
      named_bar_sync(1, 128);
      if (!*flag) continue;
      __threadfence();
      for (int h = wi; h < G; h += 4) {
        const int64_t p0 = (bh0 + h) * a.splits;
        float2 ml[kMaxSplits / 32];
#pragma unroll
        for (int u = 0; u < kMaxSplits / 32; ++u) {
          const int sp = lane + 32 * u;
          ml[u] = sp < nseg ? __ldcg(reinterpret_cast<const float2*>(part_ml_l + (p0 + sp) * 2))
                            : make_float2(-INFINITY, 0.f);
        }
        float M = -INFINITY;
#pragma unroll
        for (int u = 0; u < kMaxSplits / 32; ++u) M = fmaxf(M, ml[u].x);
        M = warp_max(M);
        const float Mu = M == -INFINITY ? 0.f : M;
        float L = 0.f;
#pragma unroll
        for (int u = 0; u < kMaxSplits / 32; ++u) {
          const float wgt = ml[u].x == -INFINITY ? 0.f : fast_exp2(ml[u].x - Mu) * ml[u].y;
          L += wgt;
          wsp[lane + 32 * u] = wgt;
        }
        L = warp_sum(L);
        __syncwarp();
        if (HAS_V) {
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          constexpr int kB = 8;
          for (int sp0 = 0; sp0 < nseg; sp0 += kB) {
            float4 v[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u)
              v[u] = sp0 + u < nseg ? __ldcg(reinterpret_cast<const float4*>(part_l + (p0 + sp0 + u) * 128 + lane * 4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < kB; ++u) {
              const float sc = sp0 + u < nseg ? wsp[sp0 + u] : 0.f;
              acc.x += sc * v[u].x; acc.y += sc * v[u].y; acc.z += sc * v[u].z; acc.w += sc * v[u].w;
            }
          }
          const float inv = L > 0.f ? 1.f / L : 0.f;
          if (out_l)
            *reinterpret_cast<float4*>(out_l + (bh0 + h) * 128 + lane * 4) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        }
        if (lane == 0 && lse_l) lse_l[bh0 + h] = (M + __log2f(L)) * kLn2;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

template <int MODE, int GM>
static cudaError_t launch_tc(const cudaLaunchConfig_t& cfg, const DecodeTmaps& tm, const DecodeArgs& c, int per) {
  static const cudaError_t at = cudaFuncSetAttribute(decode_tc_kernel<MODE, GM>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)cfg.dynamicSmemBytes);
  if (at != cudaSuccess) return at;
  return cudaLaunchKernelEx(&cfg, decode_tc_kernel<MODE, GM>, tm, c, per);
}

template <int MODE>
static cudaError_t launch_tc_g(const cudaLaunchConfig_t& cfg, const DecodeTmaps& tm, const DecodeArgs& c, int per) {
  if (c.G <= 1) return launch_tc<MODE, 1>(cfg, tm, c, per);
  if (c.G <= 2) return launch_tc<MODE, 2>(cfg, tm, c, per);
  if (c.G <= 4) return launch_tc<MODE, 4>(cfg, tm, c, per);
  if (c.G <= 8) return launch_tc<MODE, 8>(cfg, tm, c, per);
  return launch_tc<MODE, 16>(cfg, tm, c, per);
}

// ------------------------------------------------------------------- host
typedef CUresult (*EncodeTiled4Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled4Fn encode4_fn() {
  static EncodeTiled4Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled4Fn>(p);
  }
  return fn;
}

// Cache [B][Hkv][>= rows][128] bf16 with element strides (stride_b,
// stride_h), box {64, 128 rows, 1, 1}, 128B swizzle; rows >= `rows` (the
// step's seq_len) read as zeros.
static bool make_cache_map(CUtensorMap* m, const void* base, int B, int Hkv, int rows, int64_t stride_b,
                           int64_t stride_h) {
  EncodeTiled4Fn fn = encode4_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)rows, (cuuint64_t)Hkv, (cuuint64_t)B};
  cuuint64_t strides[3] = {256, (cuuint64_t)stride_h * 2, (cuuint64_t)stride_b * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)dtc::kBlk, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Q of the launch's layers [layers][B*Hq][128] bf16 (layer stride q_ls
// elements), box {64, 16 rows, 1}: a group's (padded) 16 query rows per
// half; rows past B*Hq read as zeros.
static bool make_q_map(CUtensorMap* m, const void* base, int rows, int layers, int64_t layer_stride) {
  EncodeTiled4Fn fn = encode4_fn();
  if (!fn) return false;
  const int64_t ls = layers > 1 ? layer_stride : (int64_t)rows * 128;
  if (ls <= 0 || (ls & 7)) return false;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)layers};
  cuuint64_t strides[2] = {256, (cuuint64_t)ls * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)dtc::kN, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int decode_tc_block_keys() { return dtc::kBlk; }

cudaError_t launch_decode_tc(int mode, const DecodeArgs& a_in, const void* const* k_ptrs, const void* const* v_ptrs,
                             cudaStream_t st) {
  DecodeArgs a = a_in;
  const int nl = a.nl > 0 ? a.nl : 1;
  // layers per launch are bounded by the tensor maps a launch can carry
  for (int l0 = 0; l0 < nl; l0 += kMaxMapLayers) {
    const int m = std::min(kMaxMapLayers, nl - l0);
    DecodeTmaps tm;
    for (int l = 0; l < m; ++l) {
      const void* kp = k_ptrs[l0 + l];
      const void* vp = v_ptrs ? v_ptrs[l0 + l] : kp;
      const int hkv = a.Hkv / a.kv_rep;
      if (!make_cache_map(&tm.k[l], kp, a.B, hkv, a.n, a.kv_sb, a.kv_sh)) return cudaErrorInvalidValue;
      if (!make_cache_map(&tm.v[l], vp, a.B, hkv, a.n, a.kv_sb, a.kv_sh)) return cudaErrorInvalidValue;
    }
    DecodeArgs c = a;
    c.nl = m;
    c.q = a.q + (int64_t)l0 * a.q_ls;
    if (!make_q_map(&tm.q, c.q, a.B * a.Hq, m, a.q_ls)) return cudaErrorInvalidValue;
    if (a.out) c.out = a.out + (int64_t)l0 * a.out_ls;
    if (a.scores) c.scores = a.scores + (int64_t)l0 * a.scores_ls;
    if (a.lse) c.lse = a.lse + (int64_t)l0 * a.lse_ls;
    c.part = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part) + (int64_t)l0 * a.ws_ls);
    c.part_ml = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part_ml) + (int64_t)l0 * a.ws_ls);
    c.counters = reinterpret_cast<int*>(reinterpret_cast<char*>(a.counters) + (int64_t)l0 * a.ws_ls);
    const bool has_v = mode == MODE_DENSE;
    const int smem = has_v ? dtc::Cfg<true>::kSmem : dtc::Cfg<false>::kSmem;
    // stream-K: equal contiguous ranges of the flat block space, one per SM;
    // a (sequence, kv head) spans at most a.splits ranges (its partial slots)
    const int64_t nblk = (a.n + dtc::kBlk - 1) / dtc::kBlk;
    const int64_t T1 = (int64_t)a.B * a.Hkv * nblk;
    if (T1 * m >= ((int64_t)1 << 31) || a.splits < 2) return cudaErrorInvalidValue;
    const int64_t ctas_per_layer = (int64_t)(has_v && nl > 1 ? dtc::kWavesMultiDense : dtc::kWavesSingle) * 148;
    int64_t per = (T1 + ctas_per_layer - 1) / ctas_per_layer;
    per = std::max<int64_t>(per, (nblk - 1 + a.splits - 2) / (a.splits - 1));
    per = std::max<int64_t>(per, 1);
    const int nctas = (int)((T1 + per - 1) / per) * m;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nctas);
    cfg.blockDim = dim3(dtc::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = has_v ? launch_tc_g<MODE_DENSE>(cfg, tm, c, (int)per)
                                : launch_tc_g<MODE_SCORES>(cfg, tm, c, (int)per);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace kscd
