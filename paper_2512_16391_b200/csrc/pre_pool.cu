// Pre-softmax pooled selection at engine scale (_pre_pooled, runner.py:
// 155-161): per (kv head, tile)
//
//     q_bar  = fp64 mean of the tile's G x T query rows
//     s[j]   = K[j] . q_bar * scale,           j < t1 (the tile's causal bound)
//     p[j]   = softmax(s)[j]                   (softmax_row, attention.py:77-90)
//
// and the Top-k of p (topk.cu).  The reference computes s and the softmax in
// fp64 and rounds p to fp32; here q_bar is fp64-accumulated and stored fp32,
// s is an fp32 dot product and p = exp(s - lse) in fp32, so p agrees to a few
// fp32 ulps (index sets differ only at documented near-ties).
//
// Decode rows are (b, g) with the step's token as the tile (T = 1, t1 = n);
// the scores stream K once (HBM-bound GEMV, like the anchor score pass but
// without Q heads).  Prefill rows are (g, t): the scores are a causal
// [T x 128] x [128 x N] product per kv head, run here as an fp32 SIMT GEMM
// (bf16 tensor cores would round q_bar to 8 bits -- far outside the Top-k
// tie tolerance -- and the whole GEMM is ~1 % of an anchor pass B).
#include "common.cuh"
#include "kscd_internal.h"

namespace kscd {

namespace pre {
constexpr int kGemmTiles = 32;    // tiles per GEMM CTA
constexpr int kGemmKeys = 128;    // keys per GEMM CTA (= one partial chunk)
constexpr int kGemmSmem = (128 * kGemmKeys + 128 * kGemmTiles) * 4;
constexpr int kDecThreads = 256;
constexpr int kNormKeys = 4096;   // keys per normalize CTA
}  // namespace pre

// Online (max, sum exp(s - max)) merge.
KSCD_DEV float2 ms_merge(float2 a, float2 b) {
  if (a.x == -INFINITY) return b;
  if (b.x == -INFINITY) return a;
  const float m = fmaxf(a.x, b.x);
  return make_float2(m, a.y * __expf(a.x - m) + b.y * __expf(b.x - m));
}

KSCD_DEV float2 warp_ms(float2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float2 w;
    w.x = __shfl_xor_sync(0xffffffffu, v.x, o);
    w.y = __shfl_xor_sync(0xffffffffu, v.y, o);
    v = ms_merge(v, w);
  }
  return v;
}

KSCD_DEV int row_len(const PrePoolArgs& a, int row) {
  if (a.prefill) return min(a.n, 128 * (row % a.T + 1));
  const int b = row / a.Hkv;
  return a.lens ? max(0, min(a.n, __ldg(a.lens + b))) : a.n;
}

// q_bar of one row: 128 threads, one per dimension, fp64 accumulation.
__global__ void __launch_bounds__(128) pre_qbar_kernel(const PrePoolArgs a) {
  const int row = blockIdx.x, d = threadIdx.x;
  double acc = 0.0;
  double cnt;
  if (a.prefill) {
    const int g = row / a.T, t = row % a.T;
    const int r0 = 128 * t, r1 = min(a.n, r0 + 128);
    for (int h = 0; h < a.G; ++h) {
      const __nv_bfloat16* qh = a.q + (int64_t)(g * a.G + h) * a.q_sh;
      for (int r = r0; r < r1; ++r) acc += (double)__bfloat162float(qh[(int64_t)r * 128 + d]);
    }
    cnt = (double)a.G * (double)(r1 - r0);
  } else {
    const int b = row / a.Hkv, g = row % a.Hkv;
    for (int h = 0; h < a.G; ++h) acc += (double)__bfloat162float(a.q[((int64_t)b * a.Hq + g * a.G + h) * 128 + d]);
    cnt = (double)a.G;
  }
  a.qbar[(int64_t)row * 128 + d] = (float)(acc / cnt);
}

// Decode scores: one CTA per (chunk of keys, row).  A half-warp owns one key
// row (16 lanes x 16 B = 256 B, coalesced); 4 keys per half-warp in flight.
__global__ void __launch_bounds__(pre::kDecThreads) pre_scores_decode_kernel(const PrePoolArgs a) {
  __shared__ float2 red[pre::kDecThreads / 32];
  const int row = blockIdx.y;
  const int b = row / a.Hkv, g = row % a.Hkv;
  const int len = row_len(a, row);
  const int j0 = blockIdx.x * a.chunk_keys, j1 = min(len, j0 + a.chunk_keys);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15;
  float qv[8];
  {
    const float4* qp = reinterpret_cast<const float4*>(a.qbar + (int64_t)row * 128 + hl * 8);
    const float4 x = qp[0], y = qp[1];
    qv[0] = x.x; qv[1] = x.y; qv[2] = x.z; qv[3] = x.w; qv[4] = y.x; qv[5] = y.y; qv[6] = y.z; qv[7] = y.w;
  }
  const __nv_bfloat16* kb = a.k + (int64_t)b * a.kv_sb + (int64_t)g * a.kv_sh;
  float* out = a.pooled + (int64_t)row * a.pool_stride;
  float2 ms = make_float2(-INFINITY, 0.f);
  constexpr int kU = 4;
  const int per_iter = (pre::kDecThreads / 16) * kU;      // keys per CTA iteration
  for (int base = j0; base < j1; base += per_iter) {
    uint4 raw[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = base + (u * (pre::kDecThreads / 16)) + warp * 2 + half;
      raw[u] = j < j1 ? __ldcs(reinterpret_cast<const uint4*>(kb + (int64_t)j * 128 + hl * 8)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = base + (u * (pre::kDecThreads / 16)) + warp * 2 + half;
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[u]);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        s = fmaf(f.x, qv[2 * i], s);
        s = fmaf(f.y, qv[2 * i + 1], s);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      s *= a.scale;
      if (hl == 0 && j < j1) {
        out[j] = s;
        ms = ms_merge(ms, make_float2(s, 1.f));
      }
    }
  }
  ms = warp_ms(ms);
  if (lane == 0) red[warp] = ms;
  __syncthreads();
  if (threadIdx.x == 0) {
    float2 t = red[0];
    for (int w = 1; w < pre::kDecThreads / 32; ++w) t = ms_merge(t, red[w]);
    a.part[(int64_t)row * a.chunks + blockIdx.x] = t;
  }
}

// Prefill scores: CTA = (key block kb, 32-tile group, kv head); thread (ty,
// tx) owns tiles 4ty..4ty+3 x keys 4tx..4tx+3 of the block.
__global__ void __launch_bounds__(256) pre_scores_prefill_kernel(const PrePoolArgs a) {
  extern __shared__ float sm[];
  float* Kt = sm;                                   // [128 d][128 keys]
  float* Qt = sm + 128 * pre::kGemmKeys;            // [128 d][32 tiles]
  const int kb = blockIdx.x, tg = blockIdx.y, g = blockIdx.z;
  const int t0 = tg * pre::kGemmTiles;
  if (kb > min(a.T - 1, t0 + pre::kGemmTiles - 1)) return;   // above every tile's causal bound
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int key0 = kb * pre::kGemmKeys;
  const __nv_bfloat16* kg = a.k + (int64_t)g * a.kv_sh;
  // K block -> Kt (fp32, transposed); a warp covers 32 consecutive keys
#pragma unroll 2
  for (int it = 0; it < 8; ++it) {
    const int idx = it * 256 + tid;
    const int key = idx & 127, ch = idx >> 7;       // ch: 8-element chunk of d
    const int j = key0 + key;
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (j < a.n) raw = __ldg(reinterpret_cast<const uint4*>(kg + (int64_t)j * 128 + ch * 8));
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h2[i]);
      Kt[(ch * 8 + 2 * i) * pre::kGemmKeys + key] = f.x;
      Kt[(ch * 8 + 2 * i + 1) * pre::kGemmKeys + key] = f.y;
    }
  }
  for (int idx = tid; idx < 128 * pre::kGemmTiles; idx += 256) {
    const int t = idx >> 7, d = idx & 127;
    const int row = g * a.T + t0 + t;
    Qt[d * pre::kGemmTiles + t] = (t0 + t < a.T) ? a.qbar[(int64_t)row * 128 + d] : 0.f;
  }
  __syncthreads();
  float acc[4][4] = {};
#pragma unroll 4
  for (int d = 0; d < 128; ++d) {
    const float4 q4 = *reinterpret_cast<const float4*>(Qt + d * pre::kGemmTiles + 4 * ty);
    const float4 k4 = *reinterpret_cast<const float4*>(Kt + d * pre::kGemmKeys + 4 * lane);
    const float qa[4] = {q4.x, q4.y, q4.z, q4.w};
    const float ka[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fmaf(qa[i], ka[jj], acc[i][jj]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + 4 * ty + i;
    if (t >= a.T || kb > t) continue;                // warp-uniform
    const int row = g * a.T + t;
    float* out = a.pooled + (int64_t)row * a.pool_stride;
    float2 ms = make_float2(-INFINITY, 0.f);
    const int jb = key0 + 4 * lane;
    float s[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      s[jj] = acc[i][jj] * a.scale;
      if (jb + jj < a.n) ms = ms_merge(ms, make_float2(s[jj], 1.f));
    }
    if (jb + 3 < a.n) {
      *reinterpret_cast<float4*>(out + jb) = make_float4(s[0], s[1], s[2], s[3]);
    } else {
      for (int jj = 0; jj < 4; ++jj)
        if (jb + jj < a.n) out[jb + jj] = s[jj];
    }
    ms = warp_ms(ms);
    if (lane == 0) a.part[(int64_t)row * a.chunks + kb] = ms;
  }
}

// p = exp(s - lse) over a 4096-key segment of one row, lse from the row's
// chunk partials.
__global__ void __launch_bounds__(256) pre_normalize_kernel(const PrePoolArgs a) {
  __shared__ float2 red[8];
  const int row = blockIdx.y;
  const int len = row_len(a, row);
  const int j0 = blockIdx.x * pre::kNormKeys;
  if (j0 >= len) return;
  const int nch = (len + a.chunk_keys - 1) / a.chunk_keys;
  float2 ms = make_float2(-INFINITY, 0.f);
  for (int c = threadIdx.x; c < nch; c += 256) ms = ms_merge(ms, a.part[(int64_t)row * a.chunks + c]);
  ms = warp_ms(ms);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ms;
  __syncthreads();
  float2 t = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) t = ms_merge(t, red[w]);
  const float lse = t.x + logf(t.y);
  float* p = a.pooled + (int64_t)row * a.pool_stride;
  const int j1 = min(len, j0 + pre::kNormKeys);
  for (int j = j0 + threadIdx.x; j < j1; j += 256) p[j] = expf(p[j] - lse);
}

// all-heads-pooled: the mean over kv heads of the rows' probabilities
// (np.mean over the kv-head pooled vectors, runner.py:180-197).
__global__ void __launch_bounds__(256) pre_mean_heads_kernel(const PrePoolArgs a) {
  const int r = blockIdx.y;                         // decode: b; prefill: t
  const int len = a.prefill ? min(a.n, 128 * (r + 1)) : row_len(a, r * a.Hkv);
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= len) return;
  float acc = 0.f;
  for (int g = 0; g < a.Hkv; ++g) {
    const int row = a.prefill ? g * a.T + r : r * a.Hkv + g;
    acc += a.pooled[(int64_t)row * a.pool_stride + j];
  }
  a.mean_out[(int64_t)r * a.pool_stride + j] = acc / (float)a.Hkv;
}

cudaError_t launch_pre_pool(const PrePoolArgs& a, cudaStream_t st) {
  const int rows = a.prefill ? a.Hkv * a.T : a.B * a.Hkv;
  pre_qbar_kernel<<<rows, 128, 0, st>>>(a);
  if (a.prefill) {
    static const cudaError_t attr = cudaFuncSetAttribute(pre_scores_prefill_kernel,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, pre::kGemmSmem);
    if (attr != cudaSuccess) return attr;
    dim3 grid((a.n + pre::kGemmKeys - 1) / pre::kGemmKeys, (a.T + pre::kGemmTiles - 1) / pre::kGemmTiles, a.Hkv);
    pre_scores_prefill_kernel<<<grid, 256, pre::kGemmSmem, st>>>(a);
  } else {
    dim3 grid(a.chunks, rows);
    pre_scores_decode_kernel<<<grid, pre::kDecThreads, 0, st>>>(a);
  }
  {
    dim3 grid((a.n + pre::kNormKeys - 1) / pre::kNormKeys, rows);
    pre_normalize_kernel<<<grid, 256, 0, st>>>(a);
  }
  if (a.mean_out) {
    dim3 grid((a.n + 255) / 256, a.prefill ? a.T : a.B);
    pre_mean_heads_kernel<<<grid, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

int pre_pool_chunk_keys(bool prefill) { return prefill ? pre::kGemmKeys : 2048; }

}  // namespace kscd
