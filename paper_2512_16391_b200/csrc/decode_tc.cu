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
// 4-row M tile, S^T and O^T live in TMEM (48 of 64 allocated columns), and a
// softmax thread owns one key (TMEM lane) -- and, for O^T, one dimension.
// V^T is the V block as TMA stored it ([key][d], SW128), read as an MN-major
// A operand; P^T (bf16, [head][key], SW128) is written by the softmax threads
// into shared memory as the K-major B operand.  The kernel is HBM-bound: a
// 3-stage (dense) or 6-stage (scores, K only) ring of 32 KB TMA tile loads
// keeps ~100-200 KB in flight per SM.
//
// Roles (192 threads): warp 0 lane 0 issues TMA, warp 1 lane 0 issues MMAs
// (warp 1 owns the TMEM allocation), warps 2-5 are the softmax / epilogue
// threads (TMEM lane quarters 2, 3, 0, 1).  Per key block j:
//
//   MMA:      S^T_j -> TMEM buffer j&1 ; then PV_{j-1} (after P_{j-1})
//   softmax:  load S^T_j, block max per head (warp shuffles + 4-warp smem),
//             lazy rescale of O^T (only when the max grows by > 2^8),
//             p = exp2(s - m), per-thread l partials, P^T_j -> smem buffer j&1
//
// Split-K over the keys of a (sequence, kv head) and the last-CTA merge use
// the same workspace layout as decode.cu, so every decode kernel shares the
// executor's workspace.
#include "sm100.cuh"
#include "kscd_internal.h"

namespace kscd {
using namespace sm100;

namespace dtc {
constexpr int kBlk = 128;                 // keys per block = UMMA M
constexpr int kN = 16;                    // UMMA N: the group's heads, padded
constexpr int kThreads = 192;
constexpr int kTile = kBlk * 256;         // one K or V block, 32 KB
constexpr int kHalf = kBlk * 128;         // one 64-column half of a block
constexpr int kMaxSplits = 64;
constexpr uint32_t kIdescS = idesc_bf16(128, kN, false, false);   // A = K (K-major), B = Q (K-major)
constexpr uint32_t kIdescO = idesc_bf16(128, kN, true, false);    // A = V^T (MN-major), B = P^T (K-major)
constexpr float kRescale = 8.0f;          // log2 units

template <bool HAS_V>
struct Cfg {
  static constexpr int kStages = HAS_V ? 3 : 6;
  static constexpr int kStageBytes = HAS_V ? 2 * kTile : kTile;
  static constexpr int kOffQ = kStages * kStageBytes;      // [2 halves][16 rows][128 B]
  static constexpr int kOffP = kOffQ + 4096;               // 2 x [2 halves][16 rows][128 B]
  static constexpr int kOffRed = kOffP + 8192;             // float [2][4 warps][16] block max
  static constexpr int kOffSum = kOffRed + 2 * 4 * 16 * 4; // float [4][16] l partials, [16] m
  static constexpr int kOffBar = kOffSum + 4 * 16 * 4 + 16 * 4;
  static constexpr int kOffTmem = kOffBar + 32 * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;
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

// Byte offset of element (row, col) in a [2 halves of 64 cols][rows][128 B]
// SWIZZLE_128B tile (16-byte chunks XOR-permuted by row % 8): the canonical
// K-major layout UMMA reads for Q (rows = heads, cols = d) and P^T (rows =
// heads, cols = keys).
KSCD_DEV uint32_t sw128_off(int row, int col, int rows) {
  const int half = col >> 6, c = col & 63;
  return half * rows * 128 + row * 128 + ((((c >> 3) ^ (row & 7)) & 7) << 4) + (c & 7) * 2;
}

// bars: 0..S-1 full[st] | S..2S-1 empty[st] | 2S+{0,1} s_full | +{2,3} s_free |
//       +{4,5} p_full | +{6,7} pv_done | +8 o_done
template <int MODE>
__global__ void __launch_bounds__(dtc::kThreads, 1)
    decode_tc_kernel(const __grid_constant__ DecodeTmaps tm, const DecodeArgs a) {
  using namespace dtc;
  constexpr bool HAS_V = MODE == MODE_DENSE;
  using C = Cfg<HAS_V>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* s_full = bars + 2 * S;
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_full + 4;
  uint64_t* pv_done = s_full + 6;
  uint64_t* o_done = s_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  float* lred = reinterpret_cast<float*>(smem + C::kOffSum);

  const int split = blockIdx.x, g = blockIdx.y;
  const int lyr = blockIdx.z / a.B, b = blockIdx.z - lyr * a.B;
  const int gk = g / a.kv_rep;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const __nv_bfloat16* q_l = a.q + (int64_t)lyr * a.q_ls;
  float* out_l = a.out ? a.out + (int64_t)lyr * a.out_ls : nullptr;
  float* part_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part) + (int64_t)lyr * a.ws_ls);
  float* part_ml_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part_ml) + (int64_t)lyr * a.ws_ls);
  int* counters_l = reinterpret_cast<int*>(reinterpret_cast<char*>(a.counters) + (int64_t)lyr * a.ws_ls);
  float* scores_l = a.scores ? a.scores + (int64_t)lyr * a.scores_ls : nullptr;
  float* lse_l = a.lse ? a.lse + (int64_t)lyr * a.lse_ls : nullptr;
  const CUtensorMap* kmap = &tm.k[lyr];
  const CUtensorMap* vmap = &tm.v[lyr];

  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int count = a.lens ? min(__ldg(a.lens + b), a.n) : a.n;
  const int nblk_all = (count + kBlk - 1) / kBlk;
  const int bps = (nblk_all + a.splits - 1) / a.splits;
  const int j0 = split * bps;
  const int nb = max(0, min(nblk_all, j0 + bps) - j0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  // Q of the group -> [2 halves][16 rows][128 B] SW128 (rows >= G zero)
  for (int i = threadIdx.x; i < kN * 16; i += kThreads) {
    const int row = i >> 4, ch = i & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < G) v = *reinterpret_cast<const uint4*>(q_l + ((int64_t)b * a.Hq + g * G + row) * 128 + ch * 8);
    *reinterpret_cast<uint4*>(smem + C::kOffQ + sw128_off(row, ch * 8, kN)) = v;
  }
  fence_proxy_async_smem();
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;          // cols [0,16) S0 | [16,32) S1 | [32,48) O^T

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nb > 0) {
      tma_prefetch(kmap);
      if (HAS_V) tma_prefetch(vmap);
      for (int j = 0; j < nb; ++j) {
        const int st = j % S;
        if (j >= S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
        mbar_expect_tx(&full[st], C::kStageBytes);
        const int key0 = (j0 + j) * kBlk;
        uint8_t* dst = smem + st * C::kStageBytes;
        for (int hf = 0; hf < 2; ++hf) tma_load_4d(dst + hf * kHalf, kmap, &full[st], hf * 64, key0, gk, b);
        if (HAS_V)
          for (int hf = 0; hf < 2; ++hf) tma_load_4d(dst + kTile + hf * kHalf, vmap, &full[st], hf * 64, key0, gk, b);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0 && nb > 0) {
      const uint32_t qaddr = smem_u32(smem + C::kOffQ);
      const uint32_t paddr = smem_u32(smem + C::kOffP);
      auto issue_pv = [&](int jj) {            // O^T += V_jj^T P_jj^T
        const int st = jj % S, pb = jj & 1;
        mbar_wait(&p_full[pb], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(smem + st * C::kStageBytes + kTile);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + 32, sw128_desc(vaddr + ks * 2048, kHalf, 1024),
                 sw128_desc(paddr + pb * 4096 + (ks >> 2) * 2048 + (ks & 3) * 32, 16, 1024), kIdescO,
                 (jj > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&pv_done[pb]);
        mma_commit(&empty[st]);
      };
      for (int j = 0; j < nb; ++j) {
        const int st = j % S, sb = j & 1;
        mbar_wait(&full[st], (j / S) & 1);
        if (j >= 2) mbar_wait(&s_free[sb], ((j - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t kaddr = smem_u32(smem + st * C::kStageBytes);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = (ks >> 2) * kHalf + (ks & 3) * 32;
          mma_ss(tmem + sb * 16, sw128_desc(kaddr + off, 16, 1024),
                 sw128_desc(qaddr + (ks >> 2) * 2048 + (ks & 3) * 32, 16, 1024), kIdescS, ks > 0);
        }
        mma_commit(&s_full[sb]);
        if (!HAS_V) mma_commit(&empty[st]);     // K consumed once S^T retires
        if (HAS_V && j >= 1) issue_pv(j - 1);
      }
      if (HAS_V) issue_pv(nb - 1);
      mma_commit(o_done);
    }
  } else {
    // ------------------------------------------------------ softmax / epilogue
    const int qw = warp & 3;                          // TMEM lane quarter
    const int wi = warp - 2;                          // softmax warp 0..3
    const int kin = qw * 32 + lane;                   // key within the block / dim of O^T
    const uint32_t lane_base = tmem + ((uint32_t)(qw * 32) << 16);
    float m_used[kN], lsum[kN];
#pragma unroll
    for (int h = 0; h < kN; ++h) {
      m_used[h] = -INFINITY;
      lsum[h] = 0.f;
    }
    for (int j = 0; j < nb; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(lane_base + sb * 16, r);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&s_free[sb]);
      const int key = (j0 + j) * kBlk + kin;
      const bool valid = key < count;
      float s[kN];
#pragma unroll
      for (int h = 0; h < kN; ++h) s[h] = (valid && h < G) ? __uint_as_float(r[h]) * a.scale_log2 : -INFINITY;
      if (scores_l && valid) {
#pragma unroll
        for (int h = 0; h < kN; ++h)
          if (h < G) scores_l[((int64_t)b * a.Hq + g * G + h) * a.score_stride + key] = s[h];
      }
      // block max per head: warp shuffles, then the 4 warps through smem
      float* rb = red + sb * 64;
#pragma unroll
      for (int h = 0; h < kN; ++h) {
        if (h < G) {
          const float mx = warp_max(s[h]);
          if (lane == 0) rb[wi * 16 + h] = mx;
        }
      }
      named_bar_sync(1, 128);
      bool need_any = false;
      float alpha[kN];
#pragma unroll
      for (int h = 0; h < kN; ++h) {
        alpha[h] = 1.f;
        if (h < G) {
          const float mb = fmaxf(fmaxf(rb[h], rb[16 + h]), fmaxf(rb[32 + h], rb[48 + h]));
          if (mb > m_used[h] + kRescale) {          // uniform across the CTA
            alpha[h] = m_used[h] == -INFINITY ? 1.f : exp2f(m_used[h] - mb);
            m_used[h] = mb;
            need_any = true;
          }
        }
      }
      const bool rescale = HAS_V && need_any && j > 0;
      float p[kN];
#pragma unroll
      for (int h = 0; h < kN; ++h) {
        const float mu = m_used[h] == -INFINITY ? 0.f : m_used[h];
        p[h] = (h < G && valid) ? exp2f(s[h] - mu) : 0.f;
        lsum[h] = lsum[h] * alpha[h] + p[h];
      }
      if (HAS_V) {
        if (!valid) {
          // a key past this sequence's length (ragged batch): its V row may
          // hold anything (NaN * 0 would poison O); zero it before PV reads it
          uint8_t* vrow = smem + ((j % S) * C::kStageBytes) + kTile + kin * 128;
          *reinterpret_cast<uint4*>(vrow) = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int c = 1; c < 8; ++c) reinterpret_cast<uint4*>(vrow)[c] = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(vrow + kHalf)[c] = make_uint4(0, 0, 0, 0);
        }
        if (rescale) {
          // O^T holds blocks < j: wait for PV_{j-1}, scale each head's column
          mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
          uint32_t o[16];
          tmem_ld16(lane_base + 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < kN; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * alpha[h]);
          tmem_st16(lane_base + 32, o);
          tmem_st_wait();
        }
        if (j >= 2) mbar_wait(&pv_done[sb], ((j - 2) >> 1) & 1);   // P buffer read by PV_{j-2}
        uint8_t* pbuf = smem + C::kOffP + sb * 4096;
#pragma unroll
        for (int h = 0; h < kN; ++h)
          *reinterpret_cast<__nv_bfloat16*>(pbuf + sw128_off(h, kin, kN)) = __float2bfloat16_rn(p[h]);
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
      }
    }
    // ---- epilogue: l per head (4-warp reduce), this split's partial --------
#pragma unroll
    for (int h = 0; h < kN; ++h) {
      if (h < G) {
        const float t = warp_sum(lsum[h]);
        if (lane == 0) lred[wi * 16 + h] = t;
      }
    }
    if (wi == 0 && lane < kN) lred[64 + lane] = m_used[lane];
    named_bar_sync(1, 128);
    float o[kN];
    if (HAS_V && nb > 0) {
      mbar_wait(o_done, 0);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(lane_base + 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int h = 0; h < kN; ++h) o[h] = __uint_as_float(r[h]);
    } else {
#pragma unroll
      for (int h = 0; h < kN; ++h) o[h] = 0.f;
    }
    // the previous grid (PDL) may still use the shared workspace / outputs
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int64_t bh0 = (int64_t)b * a.Hq + (int64_t)g * G;
    const int d = kin;                                // O^T lane = dimension
#pragma unroll
    for (int h = 0; h < kN; ++h) {
      if (h >= G) continue;
      const float L = lred[h] + lred[16 + h] + lred[32 + h] + lred[48 + h];
      const float M = lred[64 + h];
      if (a.splits == 1) {
        if (HAS_V && out_l) out_l[(bh0 + h) * 128 + d] = L > 0.f ? o[h] / L : 0.f;
        if (d == 0 && lse_l) lse_l[bh0 + h] = (M + __log2f(L)) * kLn2;
      } else {
        const int64_t pi = (bh0 + h) * a.splits + split;
        if (HAS_V) part_l[pi * 128 + d] = o[h];
        if (d == 0) *reinterpret_cast<float2*>(part_ml_l + pi * 2) = make_float2(M, L);
      }
    }
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
  if (a.splits == 1) return;

  // ---- the last CTA of this (b, g) merges the splits (as decode.cu) -------
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* ctr = counters_l + (int64_t)b * a.Hkv + g;
    const int prev = atomicAdd(ctr, 1);
    is_last = prev == a.splits - 1;
    if (is_last) *ctr = 0;                     // re-arm for the next launch / graph replay
  }
  __syncthreads();
  if (!is_last || warp < 2) return;
  __threadfence();
  const int wi = warp - 2;
  float* wsp = reinterpret_cast<float*>(smem) + wi * kMaxSplits;      // reuses the ring
  const int64_t bh0 = (int64_t)b * a.Hq + (int64_t)g * G;
  for (int h = wi; h < G; h += 4) {
    const int64_t p0 = (bh0 + h) * a.splits;
    float2 ml[kMaxSplits / 32];
#pragma unroll
    for (int i = 0; i < kMaxSplits / 32; ++i) {
      const int sp = lane + 32 * i;
      ml[i] = sp < a.splits ? __ldcg(reinterpret_cast<const float2*>(part_ml_l + (p0 + sp) * 2))
                            : make_float2(-INFINITY, 0.f);
    }
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxSplits / 32; ++i) M = fmaxf(M, ml[i].x);
    M = warp_max(M);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxSplits / 32; ++i) {
      const float sc = ml[i].x == -INFINITY ? 0.f : fast_exp2(ml[i].x - Mu);
      L += sc * ml[i].y;
      wsp[lane + 32 * i] = sc;
    }
    L = warp_sum(L);
    __syncwarp();
    if (HAS_V) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      constexpr int kB = 8;
      for (int sp0 = 0; sp0 < a.splits; sp0 += kB) {
        float4 v[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
          v[u] = sp0 + u < a.splits ? __ldcg(reinterpret_cast<const float4*>(part_l + (p0 + sp0 + u) * 128 + lane * 4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const float sc = sp0 + u < a.splits ? wsp[sp0 + u] : 0.f;
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
    if (a.out) c.out = a.out + (int64_t)l0 * a.out_ls;
    if (a.scores) c.scores = a.scores + (int64_t)l0 * a.scores_ls;
    if (a.lse) c.lse = a.lse + (int64_t)l0 * a.lse_ls;
    c.part = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part) + (int64_t)l0 * a.ws_ls);
    c.part_ml = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part_ml) + (int64_t)l0 * a.ws_ls);
    c.counters = reinterpret_cast<int*>(reinterpret_cast<char*>(a.counters) + (int64_t)l0 * a.ws_ls);
    const bool has_v = mode == MODE_DENSE;
    const int smem = has_v ? dtc::Cfg<true>::kSmem : dtc::Cfg<false>::kSmem;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.splits, c.Hkv, c.B * m);
    cfg.blockDim = dim3(dtc::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (has_v) {
      static const cudaError_t at = cudaFuncSetAttribute(decode_tc_kernel<MODE_DENSE>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (at != cudaSuccess) return at;
      e = cudaLaunchKernelEx(&cfg, decode_tc_kernel<MODE_DENSE>, tm, c);
    } else {
      static const cudaError_t at = cudaFuncSetAttribute(decode_tc_kernel<MODE_SCORES>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (at != cudaSuccess) return at;
      e = cudaLaunchKernelEx(&cfg, decode_tc_kernel<MODE_SCORES>, tm, c);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace kscd
