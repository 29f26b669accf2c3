// Anchor pass B for prefill: tile-pooled post-softmax weights on tcgen05.
//
// For query tile i (rows [128i, 128i+128)) and kv head g the reference pools
// the post-softmax rows of the G heads of the group over the tile's rows,
// truncated at the causal bound t1 = min(N, 128(i+1)) (_post_pooled,
// runner.py:148-152):
//
//     pooled[g][i][j] = sum_{h in g, r in tile} exp(s[h][r][j] - lse[h][r]),  j < t1
//
// (the reference's mean divides by G*T, a constant that does not change the
// Top-k).  The kernel computes S^T = K Q^T with KEYS on the MMA M dimension:
// TMEM lane = key, TMEM column = (head, row), so each thread owns one key and
// sums exp2(s*scale*log2e - lse2[row]) over its columns in an fp32 register --
// the column sum needs no shuffles and no bf16 rounding of P (which would
// break Top-k parity).  LSE comes from the dense / LSE pass of the same layer.
//
// CTA = (tile i, kv head g, head chunk of <= 4 heads).  Q of the chunk is
// resident in shared memory ([half][rows][128 B], 128B-swizzled, so each
// head's 128 rows are one canonical UMMA operand); K blocks stream through a
// 2-stage TMA ring.  The 512 TMEM columns hold one 128x128 S^T quarter per
// head; warpgroup x owns quarters x and x+2, so the tensor core refills one
// quarter while the warpgroup exponentiates the other (double buffering
// without extra TMEM) and the two warpgroups run decoupled, each writing a
// partial-sum plane that the Top-k reads as plane0 + plane1.
#include "sm100.cuh"
#include "kscd_internal.h"
#include "topk_select.cuh"

#ifndef KSCD_FUSED_NB
#define KSCD_FUSED_NB 2
#endif

namespace kscd {
using namespace sm100;

namespace pp {
constexpr int kThreads = 384;
constexpr int kStages = 2;
constexpr int kBlock = 128;
constexpr int kHalfRows = 512 * 128;        // bytes of one 64-column half for 512 rows
constexpr int kOffQ = 0;                    // [2 halves][512 rows][128 B] = 128 KB
constexpr int kOffK = 2 * kHalfRows;        // stages x 32 KB
constexpr int kOffLse = kOffK + kStages * 32768;   // float[512]
constexpr int kOffRed = kOffLse + 512 * 4;         // float[2][128]
constexpr int kOffBar = kOffRed + 2 * 128 * 4;
constexpr int kOffTmem = kOffBar + 16 * 8;
constexpr int kSmemBytes = kOffTmem + 16 + 1024;
constexpr uint32_t kIdescQ = idesc_bf16(128, 128, false, false);   // S^T quarter: 128 keys x 128 rows
}  // namespace pp

struct PoolTmaps {
  CUtensorMap q, k;
};

#ifdef KSCD_PB_TRACE
// dev instrumentation (variant builds only): clock64 stamps of one pass-B
// CTA (the middle tile, kv head 0) per key block -- scripts/pb_trace.py
__device__ long long g_pb_trace[512][8];
__device__ long long g_pb_tail[4];     // CTA start, column sums done, fused Top-k done
#define PB_TRACE(e, j)                                                                                       \
  do {                                                                                                       \
    if (blockIdx.y == 0 && (int)blockIdx.x == (int)gridDim.x / 2 && (j) < 512) g_pb_trace[(j)][(e)] = clock64(); \
  } while (0)
extern "C" int kscd_debug_pb_trace(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_pb_trace, sizeof(g_pb_trace));
}
extern "C" int kscd_debug_pb_tail(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_pb_tail, sizeof(g_pb_tail));
}
#define PB_TAIL(e)                                                                                 \
  do {                                                                                             \
    if (blockIdx.y == 0 && (int)blockIdx.x == (int)gridDim.x / 2) g_pb_tail[(e)] = clock64();     \
  } while (0)
#else
#define PB_TRACE(e, j) \
  do {                 \
  } while (0)
#define PB_TAIL(e) \
  do {             \
  } while (0)
#endif

// Sum over the 128 (head, row) columns of one S^T quarter held by this
// thread (its key): exp2(s * scale * log2e - lse2[row]), rows after the key
// zeroed on the diagonal block (the causal zeros of _post_pooled).
template <bool DIAG>
KSCD_DEV float2 pool_colsum(const uint32_t (&r)[128], uint32_t l4, float2 sc2, int key, int r0) {
  float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 128; i += 4) {
    const float4 lv = lds_f4(l4 + i * 4);    // broadcast read: same rows for every key
    float2 e0 = __ffma2_rn(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2,
                           make_float2(-lv.x, -lv.y));
    float2 e1 = __ffma2_rn(make_float2(__uint_as_float(r[i + 2]), __uint_as_float(r[i + 3])), sc2,
                           make_float2(-lv.z, -lv.w));
    e0 = exp2_pair_sum<KSCD_PB_POLY>(e0, i >> 1);
    e1 = exp2_pair_sum<KSCD_PB_POLY>(e1, (i >> 1) + 1);
    if (DIAG) {
      if (key > r0 + i) e0.x = 0.f;
      if (key > r0 + i + 1) e0.y = 0.f;
      if (key > r0 + i + 2) e1.x = 0.f;
      if (key > r0 + i + 3) e1.y = 0.f;
    }
    acc2 = __fadd2_rn(acc2, __fadd2_rn(e0, e1));
  }
  return acc2;
}

// Top-k of the pooled row this CTA just wrote into its SM's scratch slot
// (two planes), by threads 128..383.
// The fused anchor selection of one (kv head, tile) row on all 384 threads:
// the exact Top-k with k = k_budget(t1) over plane0 + plane1 of this SM's
// slot, the freed Q shared memory as its workspace.  Out of line, so the
// select's registers never compete with the column-sum loop's.  2 float4
// loads in flight per thread (x2 planes); 4 and 8 spilled and ran slower.
__device__ __noinline__ void fused_select_tail(const PoolPrefillArgs& a, uint8_t* sh_mem, int t1, int64_t r) {
  if (threadIdx.x == 0 && smid_u32() >= (uint32_t)kSmSlots) __trap();   // scratch slot bound
  TopkShared& tsh = *reinterpret_cast<TopkShared*>(sh_mem);
  const float* row0 = a.pooled + (int64_t)smid_u32() * 2 * a.pool_stride;
  const int k = k_budget_dev(a.fraction, a.k_min, t1);
  topk_select<1, 384, 0, KSCD_FUSED_NB>(row0, row0 + a.pool_stride, t1, min(k, t1), a.idx + r * a.k_cap, a.k_cap,
                                        a.counts + r, tsh);
}

// bars: 0 q_full | 1-2 k_full[s] | 3-4 k_empty[s] | 5-6 s_full[x] | 7-8 buf_free[x]
__global__ void __launch_bounds__(pp::kThreads, 1)
    pool_prefill_kernel(const __grid_constant__ PoolTmaps tm, const PoolPrefillArgs a) {
  using namespace pp;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round
  // trip would hide the address space and turn shared loads into generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  float* lse2 = reinterpret_cast<float*>(smem + kOffLse);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = (a.N + 127) / 128;
  const int ti = T - 1 - (int)blockIdx.x;        // long (late) tiles first
  const int g = a.g_fixed >= 0 ? a.g_fixed : (int)blockIdx.y;
  const int r0 = ti * 128;
  const int t1 = min(a.N, r0 + 128);             // causal bound of the tile
  const int nb = (t1 + kBlock - 1) / kBlock;
  const int nh = a.nheads;                       // heads of this chunk (<= 4)
  const int hbase = g * a.G + a.head_begin;

  if (threadIdx.x == 0) {
    PB_TAIL(0);
    mbar_init(&bars[0], 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars[1 + s], 1);
      mbar_init(&bars[3 + s], 1);
    }
    for (int qq = 0; qq < 4; ++qq) {
      mbar_init(&bars[5 + qq], 1);     // s_full[quarter]
      mbar_init(&bars[9 + qq], 128);   // buf_free[quarter]
    }
    fence_barrier_init();
  }
  // per-row log2-domain LSE of the chunk's rows; rows past N never count
  for (int r = threadIdx.x; r < 512; r += kThreads) {
    const int hh = r >> 7, rr = r & 127;
    float v = INFINITY;
    if (hh < nh && r0 + rr < a.N) v = a.lse[(int64_t)(hbase + hh) * a.N + r0 + rr] * kLog2e;
    lse2[r] = v;
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------- TMA producer
      tma_prefetch(&tm.q);
      tma_prefetch(&tm.k);
      mbar_expect_tx(&bars[0], nh * 2 * 16384);
      for (int hh = 0; hh < nh; ++hh)
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(smem + kOffQ + hf * kHalfRows + hh * 16384, &tm.q, &bars[0], hf * 64, r0, hbase + hh);
      for (int j = 0; j < nb; ++j) {
        const int st = j % kStages;
        if (j >= kStages) mbar_wait(&bars[3 + st], ((j / kStages) - 1) & 1);
        mbar_expect_tx(&bars[1 + st], 32768);
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(smem + kOffK + st * 32768 + hf * 16384, &tm.k, &bars[1 + st], hf * 64, j * kBlock, g);
      }
    } else if (warp == 3 && lane == 0) {
      // --------------------------------------------------------- MMA issuer
      const uint32_t qaddr = smem_u32(smem + kOffQ);
      const uint32_t kaddr = smem_u32(smem + kOffK);
      mbar_wait(&bars[0], 0);
      // quarter qq = head qq of the chunk (128 rows) -> TMEM columns
      // [128 qq, 128 qq + 128); issue order alternates the two warpgroups
      for (int j = 0; j < nb; ++j) {
        const int st = j % kStages;
        mbar_wait(&bars[1 + st], (j / kStages) & 1);
        for (int oi = 0; oi < 4; ++oi) {
          const int qq = (oi >> 1) | ((oi & 1) << 1);   // 0, 2, 1, 3
          if (qq >= nh) continue;
          if (j > 0) mbar_wait(&bars[9 + qq], (j - 1) & 1);   // quarter qq of block j-1 consumed
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t koff = (ks >> 2) * 16384 + (ks & 3) * 32;
            const uint32_t qoff = (ks >> 2) * kHalfRows + qq * 128 * 128 + (ks & 3) * 32;
            mma_ss(tmem + 128 * qq, sw128_desc(kaddr + st * 32768 + koff, 16, 1024),
                   sw128_desc(qaddr + qoff, 16, 1024), kIdescQ, ks > 0);
          }
          mma_commit(&bars[5 + qq]);
        }
        mma_commit(&bars[3 + st]);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
    // --------------------------------------------------- column-sum warpgroups
    // WG x owns quarters x and x + 2 (heads of the chunk); while it sums one,
    // the tensor core refills the other's TMEM buffer for the next block.  Each
    // WG writes its own partial plane (read back as plane0 + plane1 by the
    // Top-k), so the warpgroups never wait for each other and the result is
    // deterministic.
    const int x = (warp - 4) >> 2;
    const int q = warp & 3;
    const int key_in_blk = q * 32 + lane;          // TMEM lane = key
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int64_t plane = (int64_t)(a.g_fixed >= 0 ? 1 : a.Hkv) * T * a.pool_stride;
    // all-heads-pooled mode writes one row per tile (runner.py:180-197);
    // fused: the two planes of this SM's slot (one CTA per SM at a time)
    float* out_row = a.fuse ? a.pooled + ((int64_t)smid_u32() * 2 + x) * a.pool_stride
                            : a.pooled + x * plane + ((int64_t)(a.g_fixed >= 0 ? 0 : g) * T + ti) * a.pool_stride;
    const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
    for (int j = 0; j < nb; ++j) {
      const int key = j * kBlock + key_in_blk;
      const bool diag = (j == nb - 1);             // only the last block crosses the staircase
      float2 acc2 = make_float2(0.f, 0.f);
      for (int qq = x; qq < nh; qq += 2) {
        if (lane == 0 && q == 0) PB_TRACE(qq, j);           // quarter qq of block j: waiting starts
        mbar_wait(&bars[5 + qq], j & 1);
        if (lane == 0 && q == 0) PB_TRACE(4 + qq, j);       // ... S^T ready
        tc_fence_after();
        uint32_t r[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tmem_ld32(lane_base + 128 * qq + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars[9 + qq]);                // buffer free: the MMA may refill it
        const uint32_t l4 = smem_u32(lse2 + 128 * qq);
        // separate instantiations: the staircase mask costs 2 ALU ops per
        // element, and only the last block needs it
        acc2 = __fadd2_rn(acc2, diag ? pool_colsum<true>(r, l4, sc2, key, r0) : pool_colsum<false>(r, l4, sc2, key, r0));
      }
      if (key < t1) {
        float v = acc2.x + acc2.y;
        if (a.accumulate) v += out_row[key];
        out_row[key] = v;
      }
    }
  }
  if (a.fuse) {
    // ---- fused selection (runner.py:199-206) right after the row was
    // written, on every thread of the CTA: the producer / MMA warps raise
    // their register budget to 168 as the column-sum warpgroups lower theirs
    // (256 -> 384 threads: the tail went from 10.5 % to 7.1 % of a 128K CTA,
    // pass B 83.9 -> 81.9 ms).  The row's global writes are visible to the
    // CTA after the barrier, and Q shared memory is free (every MMA retired
    // before the last column sums were read).
    // the column-sum warps release their registers BEFORE any producer warp
    // asks for more: an early producer-side inc (warps 1-2 idle through the
    // loop) could otherwise take registers the column-sum warps' own entry
    // inc still waits for -- a deadlock that compute-sanitizer's timing hit
    if (warp >= 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 168;\n");
    __syncthreads();
    if (warp < 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n");
    __syncthreads();
    if (threadIdx.x == 128) PB_TAIL(1);
    fused_select_tail(a, smem + kOffQ, t1, (int64_t)g * T + ti);
#ifdef KSCD_PB_TRACE
    __syncthreads();
    if (threadIdx.x == 128) PB_TAIL(2);
#endif
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------- host
int sm_slots() { return kSmSlots; }
bool make_prefill_map(CUtensorMap* m, const void* base, int heads, int rows, int64_t head_stride);

cudaError_t launch_pool_prefill(const PoolPrefillArgs& a, cudaStream_t st) {
  PoolTmaps tm;
  if (!make_prefill_map(&tm.q, a.q, a.Hq, a.N, a.q_sh)) return cudaErrorInvalidValue;
  if (!make_prefill_map(&tm.k, a.k, a.Hkv, a.N, a.kv_sh)) return cudaErrorInvalidValue;
  static const cudaError_t attr =
      cudaFuncSetAttribute(pool_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pp::kSmemBytes);
  if (attr != cudaSuccess) return attr;
  const int T = (a.N + 127) / 128;
  dim3 grid(T, a.g_fixed >= 0 ? 1 : a.Hkv);
  pool_prefill_kernel<<<grid, pp::kThreads, pp::kSmemBytes, st>>>(tm, a);
  return cudaGetLastError();
}

}  // namespace kscd
