// Split-K sparse decode attention for Kascade (one query token per
// sequence): keys idx[b][map[g]][0..cnt) -- reuse layers through the head
// remap table, and anchors over their own fresh sets (topk_attention on a
// decode tile, attention.py:185-253; runner.py:210-225).  The dense and
// anchor score passes stream contiguous keys and run on the tcgen05 / TMA
// kernel (decode_tc.cu); a gather of 256-B rows at random positions has no
// TMA tile shape, so this one stays on cp.async + mma.sync.
//
// Grid = (splits, Hkv, B x layers); 4 warps per CTA.  Gathered K/V rows
// (256 B each) stream through a cp.async (LDGSTS) ring of 64-key tiles,
// XOR-swizzled so the ldmatrix reads are bank-conflict free.  Each warp owns 16 keys of a tile
// and keeps its own online-softmax state for the G query heads of the group
// (G <= 16 rows of one m16n8k16 tile), so there is no CTA barrier per tile
// beyond the ring's.  Partial (m, l, O) of the 4 warps are merged in shared
// memory; the last CTA of a (b, g) to finish merges the splits (warp-shuffle
// LSE merge) and resets its arrival counter, so no extra launch is needed.
#include <stdlib.h>

#include "common.cuh"
#include "kscd_internal.h"

namespace kscd {

constexpr int kTileKeys = 64;
constexpr int kMaxSplitsDev = 64;   // = capi.cu kMaxSplits (the workspace and merge bound)
constexpr int kThreads = 128;
constexpr int kTileBytes = kTileKeys * kRowBytes;  // 16 KB

struct DecodeCfg {
  static constexpr bool kHasV = true;
  static constexpr int kStages = 3;
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kPipeBytes = kStages * kStageBytes;
  // merge scratch reuses the ring: 4 warps x 16 rows x (128 + 2) floats
  static constexpr int kMergeBytes = 4 * 16 * (kHeadDim + 2) * 4;
  static constexpr int kSmemBytes = kPipeBytes > kMergeBytes ? kPipeBytes : kMergeBytes;
  static constexpr int kMinBlocks = 2;
};

template <bool G16>
__global__ void __launch_bounds__(kThreads, DecodeCfg::kMinBlocks)
    decode_attn_kernel(const DecodeArgs a) {
  using Cfg = DecodeCfg;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int split = blockIdx.x, g = blockIdx.y;                     // g: (virtual) head group
  const int lyr = blockIdx.z / a.B, b = blockIdx.z - lyr * a.B;        // layer of a multi-layer launch
  const int gk = g / a.kv_rep;                                        // its kv head
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int G = a.G;
  // this layer's tensors (a multi-layer launch runs consecutive independent
  // layers -- e.g. all reuse layers between two anchors -- as one grid)
  const __nv_bfloat16* q_l = a.q + (int64_t)lyr * a.q_ls;
  const __nv_bfloat16* k_l = a.k_tab ? a.k_tab[lyr] : a.k;
  const __nv_bfloat16* v_l = a.v_tab ? a.v_tab[lyr] : a.v;
  float* out_l = a.out ? a.out + (int64_t)lyr * a.out_ls : nullptr;
  const int* hm_l = a.head_map ? a.head_map + (int64_t)lyr * a.hm_ls : nullptr;
  float* part_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part) + (int64_t)lyr * a.ws_ls);
  float* part_ml_l = reinterpret_cast<float*>(reinterpret_cast<char*>(a.part_ml) + (int64_t)lyr * a.ws_ls);
  int* counters_l = reinterpret_cast<int*>(reinterpret_cast<char*>(a.counters) + (int64_t)lyr * a.ws_ls);
  float* lse_l = a.lse ? a.lse + (int64_t)lyr * a.lse_ls : nullptr;

  const __nv_bfloat16* kbase = k_l + (int64_t)b * a.kv_sb + (int64_t)gk * a.kv_sh;
  const __nv_bfloat16* vbase = v_l + (int64_t)b * a.kv_sb + (int64_t)gk * a.kv_sh;
  const int* sel = nullptr;
  // Programmatic dependent launch (consecutive decode layers): let the next
  // layer's kernel start filling SMs as ours retire.  Our inputs are all
  // complete when we start -- q and the caches are static within a step, the
  // index lists come from a select launch that never triggers early, and no
  // decode launch ever directly follows the pooling kernel that reads the
  // score buffer we may stream into -- so only the merge below (its
  // workspace and counters are shared with the previous layer's kernel, and
  // it writes out / lse) waits for the previous grid.
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  int count = a.lens ? min(__ldg(a.lens + b), a.n) : a.n;
  {
    const int src = hm_l ? __ldg(hm_l + gk) : gk;
    sel = a.idx + (int64_t)lyr * a.idx_ls + (int64_t)b * a.idx_sb + (int64_t)src * a.idx_sh;
    count = min(__ldg(a.cnt + (int64_t)lyr * a.cnt_ls + (int64_t)b * a.cnt_sb + src), a.k_cap);
  }
  const int ntiles = (count + kTileKeys - 1) / kTileKeys;
  const int tps = (ntiles + a.splits - 1) / a.splits;
  const int t0 = split * tps;
  const int t1 = min(ntiles, t0 + tps);
  const int my_tiles = max(0, t1 - t0);

  // ---- Q fragments (A operand: rows = query heads of the group) --------
  uint32_t qa0[8], qa2[8], qa1[8], qa3[8];
  {
    const __nv_bfloat16* qg = q_l + ((int64_t)b * a.Hq + (int64_t)g * G) * kHeadDim;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c = ks * 16 + 2 * tig;
      qa0[ks] = gid < G ? *reinterpret_cast<const uint32_t*>(qg + gid * kHeadDim + c) : 0u;
      qa2[ks] = gid < G ? *reinterpret_cast<const uint32_t*>(qg + gid * kHeadDim + c + 8) : 0u;
      if (G16) {
        const int r = gid + 8;
        qa1[ks] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kHeadDim + c) : 0u;
        qa3[ks] = r < G ? *reinterpret_cast<const uint32_t*>(qg + r * kHeadDim + c + 8) : 0u;
      } else {
        qa1[ks] = 0u;
        qa3[ks] = 0u;
      }
    }
  }

  const uint32_t pipe = smem_u32(smem);
  // Each thread copies chunk column (tid & 15) of rows (tid >> 4) + 8 i.
  const int my_chunk = tid & 15, my_row0 = tid >> 4;

  // Sparse mode: the gather positions of a tile are loaded one iteration
  // before its cp.async is issued, so the dependent index load never sits on
  // the issue path (an L2 round trip per tile otherwise).
  int pos_next[8];
  auto load_positions = [&](int t) {
    const int key0 = (t0 + t) * kTileKeys;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kk = key0 + my_row0 + 8 * i;
      pos_next[i] = (t < my_tiles && kk < count) ? __ldg(sel + kk) : 0;
    }
  };
  auto issue_tile = [&](int t, int stage) {
    const int key0 = (t0 + t) * kTileKeys;
    const uint32_t kdst = pipe + stage * Cfg::kStageBytes;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = my_row0 + 8 * i;
      const int kk = key0 + row;
      const bool valid = kk < count;
      const int pos = valid ? pos_next[i] : 0;
      const uint32_t off = row * kRowBytes + swz(row, my_chunk) * 16;
      const int64_t src = (int64_t)pos * kHeadDim + my_chunk * 8;
      cp_async16_zfill(kdst + off, kbase + src, valid);
      if (Cfg::kHasV) cp_async16_zfill(kdst + kTileBytes + off, vbase + src, valid);
    }
  };

  // ---- online softmax state (rows gid and gid + 8) ---------------------
  float m_r[2] = {-INFINITY, -INFINITY};
  float l_r[2] = {0.f, 0.f};
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  // prologue: the positions of every prologue tile are loaded together (one
  // L2 round trip instead of one per stage before the first gather issues)
  {
    int pos_pro[Cfg::kStages - 1][8];
#pragma unroll
    for (int s = 0; s < Cfg::kStages - 1; ++s) {
      load_positions(s);
#pragma unroll
      for (int i = 0; i < 8; ++i) pos_pro[s][i] = pos_next[i];
    }
#pragma unroll
    for (int s = 0; s < Cfg::kStages - 1; ++s) {
#pragma unroll
      for (int i = 0; i < 8; ++i) pos_next[i] = pos_pro[s][i];
      if (s < my_tiles) issue_tile(s, s);
      cp_async_commit();
    }
  }
  load_positions(Cfg::kStages - 1);

  for (int t = 0; t < my_tiles; ++t) {
    const int stage = t % Cfg::kStages;
    cp_async_wait<Cfg::kStages - 2>();
    __syncthreads();
    {
      const int tn = t + Cfg::kStages - 1;
      if (tn < my_tiles) issue_tile(tn, tn % Cfg::kStages);
      cp_async_commit();
      load_positions(tn + 1);
    }
    const uint32_t ks_base = pipe + stage * Cfg::kStageBytes;
    const int key_w = (t0 + t) * kTileKeys + warp * 16;  // list index of this warp's first key

    // S = Q K^T over the warp's 16 keys (two n8 tiles)
    float s[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
      const int row = warp * 16 + nt * 8 + (lane & 7);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t b0, b1, b2, b3;
        const int chunk = 4 * j + (lane >> 3);
        ldsm_x4(ks_base + row * kRowBytes + swz(row, chunk) * 16, b0, b1, b2, b3);
        mma_bf16_16816(s[nt], qa0[2 * j], qa1[2 * j], qa2[2 * j], qa3[2 * j], b0, b1);
        mma_bf16_16816(s[nt], qa0[2 * j + 1], qa1[2 * j + 1], qa2[2 * j + 1], qa3[2 * j + 1], b2, b3);
      }
    }
    // scale to log2 domain, mask keys past the list
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int kk = key_w + nt * 8 + 2 * tig + (c & 1);
        s[nt][c] = kk < count ? s[nt][c] * a.scale_log2 : -INFINITY;
      }
    }
    // online softmax per head row (quad-reduced max, thread-partial sum)
    float p[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int r = 0; r < (G16 ? 2 : 1); ++r) {
      float mx = fmaxf(fmaxf(s[0][2 * r], s[0][2 * r + 1]), fmaxf(s[1][2 * r], s[1][2 * r + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_r[r], mx);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;
      const float alpha = fast_exp2(m_r[r] - m_use);
      m_r[r] = m_new;
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        p[nt][2 * r] = fast_exp2(s[nt][2 * r] - m_use);
        p[nt][2 * r + 1] = fast_exp2(s[nt][2 * r + 1] - m_use);
        sum += p[nt][2 * r] + p[nt][2 * r + 1];
      }
      l_r[r] = l_r[r] * alpha + sum;
      if (Cfg::kHasV) {
#pragma unroll
        for (int dn = 0; dn < 16; ++dn) {
          o[dn][2 * r] *= alpha;
          o[dn][2 * r + 1] *= alpha;
        }
      }
    }
    if (Cfg::kHasV) {
      // O += P V : A = P (rows = heads, k = the warp's 16 keys), B = V rows
      const uint32_t pa0 = pack_bf16(p[0][0], p[0][1]);
      const uint32_t pa1 = G16 ? pack_bf16(p[0][2], p[0][3]) : 0u;
      const uint32_t pa2 = pack_bf16(p[1][0], p[1][1]);
      const uint32_t pa3 = G16 ? pack_bf16(p[1][2], p[1][3]) : 0u;
      const uint32_t vs_base = ks_base + kTileBytes;
      const int mtx = lane >> 3;
      const int row = warp * 16 + (mtx & 1) * 8 + (lane & 7);
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        uint32_t b0, b1, b2, b3;
        const int chunk = c + (mtx >> 1);
        ldsm_x4_t(vs_base + row * kRowBytes + swz(row, chunk) * 16, b0, b1, b2, b3);
        mma_bf16_16816(o[c], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16_16816(o[c + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  // ---- merge the 4 warps of the CTA in shared memory --------------------
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  float* ms = reinterpret_cast<float*>(smem);                 // [4][16] m
  float* ls = ms + 64;                                         // [4][16] l
  float* os = ls + 64;                                         // [4][16][128] O
  if (tig == 0) {
    ms[warp * 16 + gid] = m_r[0];
    ls[warp * 16 + gid] = l_r[0];
    ms[warp * 16 + gid + 8] = m_r[1];
    ls[warp * 16 + gid + 8] = l_r[1];
  }
  if (Cfg::kHasV) {
#pragma unroll
    for (int dn = 0; dn < 16; ++dn) {
      const int col = dn * 8 + 2 * tig;
      *reinterpret_cast<float2*>(os + (warp * 16 + gid) * kHeadDim + col) = make_float2(o[dn][0], o[dn][1]);
      if (G16)
        *reinterpret_cast<float2*>(os + (warp * 16 + gid + 8) * kHeadDim + col) = make_float2(o[dn][2], o[dn][3]);
    }
  }
  __syncthreads();

  // warp w merges heads w, w+4, ...; lane covers 4 dims
  const int64_t bh0 = (int64_t)b * a.Hq + (int64_t)g * G;
  for (int h = warp; h < G; h += 4) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, ms[w * 16 + h]);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float sc = fast_exp2(ms[w * 16 + h] - Mu);
      L += sc * ls[w * 16 + h];
      if (Cfg::kHasV) {
        const float4 v = *reinterpret_cast<const float4*>(os + (w * 16 + h) * kHeadDim + lane * 4);
        acc.x += sc * v.x; acc.y += sc * v.y; acc.z += sc * v.z; acc.w += sc * v.w;
      }
    }
    if (a.splits == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
      if (Cfg::kHasV)
        *reinterpret_cast<float4*>(out_l + (bh0 + h) * kHeadDim + lane * 4) =
            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      if (lane == 0 && lse_l) lse_l[bh0 + h] = (M + __log2f(L)) * kLn2;
    } else {
      const int64_t pi = (bh0 + h) * a.splits + split;
      if (Cfg::kHasV) *reinterpret_cast<float4*>(part_l + pi * kHeadDim + lane * 4) = acc;
      if (lane == 0) *reinterpret_cast<float2*>(part_ml_l + pi * 2) = make_float2(M, L);
    }
  }
  if (a.splits == 1) return;

  // ---- last CTA of this (b, g) merges the splits -------------------------
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int* ctr = counters_l + (int64_t)b * a.Hkv + g;
    const int prev = atomicAdd(ctr, 1);
    is_last = prev == a.splits - 1;
    if (is_last) *ctr = 0;  // re-arm for the next launch / graph replay
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // The partials are read with every load of a batch in flight: the split
  // weights exp2(m_sp - M) go to shared memory first (lanes over splits), so
  // the O loop has no dependent load per split (a serial load chain over 37
  // splits of the 8-row kv-head-shard case cost ~13 us of L2 latency).
  float* wsp = reinterpret_cast<float*>(smem) + warp * kMaxSplitsDev;   // reuses the ring
  for (int h = warp; h < G; h += 4) {
    const int64_t p0 = (bh0 + h) * a.splits;
    float2 ml[kMaxSplitsDev / 32];
#pragma unroll
    for (int i = 0; i < kMaxSplitsDev / 32; ++i) {
      const int sp = lane + 32 * i;
      ml[i] = sp < a.splits ? __ldcg(reinterpret_cast<const float2*>(part_ml_l + (p0 + sp) * 2))
                            : make_float2(-INFINITY, 0.f);
    }
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxSplitsDev / 32; ++i) M = fmaxf(M, ml[i].x);
    M = warp_max(M);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxSplitsDev / 32; ++i) {
      const float sc = ml[i].x == -INFINITY ? 0.f : fast_exp2(ml[i].x - Mu);
      L += sc * ml[i].y;
      wsp[lane + 32 * i] = sc;
    }
    L = warp_sum(L);
    __syncwarp();
    if (Cfg::kHasV) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      constexpr int kB = 8;
      for (int sp0 = 0; sp0 < a.splits; sp0 += kB) {
        float4 v[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
          v[u] = sp0 + u < a.splits ? __ldcg(reinterpret_cast<const float4*>(part_l + (p0 + sp0 + u) * kHeadDim + lane * 4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const float sc = sp0 + u < a.splits ? wsp[sp0 + u] : 0.f;
          acc.x += sc * v[u].x; acc.y += sc * v[u].y; acc.z += sc * v[u].z; acc.w += sc * v[u].w;
        }
      }
      const float inv = L > 0.f ? 1.f / L : 0.f;
      *reinterpret_cast<float4*>(out_l + (bh0 + h) * kHeadDim + lane * 4) =
          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    }
    if (lane == 0 && lse_l) lse_l[bh0 + h] = (M + __log2f(L)) * kLn2;
    __syncwarp();
  }
}

static cudaError_t launch_sparse(const DecodeArgs& a, cudaStream_t st) {
  using Cfg = DecodeCfg;
  dim3 grid(a.splits, a.Hkv, a.B * (a.nl > 0 ? a.nl : 1));
  const int smem = Cfg::kSmemBytes;
  // one-time opt-in to >48 KB dynamic shared memory per instantiation
  static const cudaError_t attr_hi = cudaFuncSetAttribute(
      decode_attn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static const cudaError_t attr_lo = cudaFuncSetAttribute(
      decode_attn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (attr_hi != cudaSuccess) return attr_hi;
  if (attr_lo != cudaSuccess) return attr_lo;
  // programmatic stream serialization (see the kernel's PDL note)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.G > 8) return cudaLaunchKernelEx(&cfg, decode_attn_kernel<true>, a);
  return cudaLaunchKernelEx(&cfg, decode_attn_kernel<false>, a);
}

cudaError_t launch_decode_attn(int mode, const DecodeArgs& a, cudaStream_t st) {
  // the dense and score passes run on the tcgen05 / TMA kernel (decode_tc.cu)
  if (mode != MODE_SPARSE) return cudaErrorInvalidValue;
  return launch_sparse(a, st);
}

int decode_tile_keys() { return kTileKeys; }

}  // namespace kscd
