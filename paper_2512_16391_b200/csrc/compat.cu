// Small-N kernels behind the reference-signature (trace-level) API:
// materialised post-softmax rows, pooled rows of arbitrary tiles, and
// pre-softmax pooled distributions.  The reference materialises P
// [Hq][N][N] in dense_attention (attention.py:121); these kernels give the
// compat layer the same tensors on the GPU for reference-scale traces
// (N up to a few thousand), for any TileSpec (tiles.py:117-152).  The 128-row
// prefill tiles of the performance path never use them.
#include "common.cuh"
#include "kscd_internal.h"

namespace kscd {

// P[h][r][c] = exp(s - lse_r) for visible c (c <= r when causal), else 0.
__global__ void __launch_bounds__(256) dense_probs_kernel(const ProbsArgs a) {
  __shared__ float qs[32][129];
  __shared__ float ks[32][129];
  const int h = blockIdx.z, g = h / a.G;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  if (a.causal && c0 > r0 + 31) {
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, c = c0 + tx;
      if (r < a.N && c < a.N) a.P[((int64_t)h * a.N + r) * a.N + c] = 0.f;
    }
    return;
  }
  for (int i = threadIdx.x; i < 32 * 128; i += 256) {
    const int rr = i >> 7, dd = i & 127;
    const int r = r0 + rr, c = c0 + rr;
    qs[rr][dd] = r < a.N ? __bfloat162float(a.q[(int64_t)h * a.q_sh + (int64_t)r * 128 + dd]) : 0.f;
    ks[rr][dd] = c < a.N ? __bfloat162float(a.k[(int64_t)g * a.kv_sh + (int64_t)c * 128 + dd]) : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + tx;
    if (r >= a.N || c >= a.N) continue;
    float acc = 0.f;
#pragma unroll 8
    for (int dd = 0; dd < 128; ++dd) acc = fmaf(qs[i][dd], ks[tx][dd], acc);
    const bool vis = !a.causal || c <= r;
    const float lse = a.lse[(int64_t)h * a.N + r];
    a.P[((int64_t)h * a.N + r) * a.N + c] = vis ? expf(acc * a.scale - lse) : 0.f;
  }
}

// pooled[row][j] = sum over the heads of kv head g (all heads when
// all_heads) and the rows [start, end) of P[h][r][j], j < end (zero beyond);
// fp64 accumulation like _post_pooled's mean (runner.py:148-152).
__global__ void __launch_bounds__(256) pool_rows_kernel(const PoolRowsArgs a) {
  const int t = blockIdx.y, g = blockIdx.z;
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= a.N) return;
  const int s = a.starts[t], e = a.ends[t];
  const int h0 = a.all_heads ? 0 : g * a.G;
  const int nh = a.all_heads ? a.Hq : a.G;
  double acc = 0.0;
  if (j < e) {
    for (int hh = 0; hh < nh; ++hh)
      for (int r = s; r < e; ++r) acc += (double)a.P[((int64_t)(h0 + hh) * a.N + r) * a.N + j];
  }
  a.pooled[((int64_t)g * a.T + t) * a.pool_stride + j] = (float)acc;
}

// Pre-softmax pooling (runner.py:155-161): q_bar = mean of the tile's G*T
// query rows (fp64), scores over keys < end, softmax in fp64, fp32 result.
// One CTA per (kv head, tile).
__global__ void __launch_bounds__(256) pre_pool_kernel(const PoolRowsArgs a) {
  __shared__ double qbar[128];
  __shared__ double red[256];
  const int t = blockIdx.x, g = blockIdx.y;
  const int s = a.starts[t], e = a.ends[t];
  const int tid = threadIdx.x;
  const double cnt = (double)a.G * (double)(e - s);
  if (tid < 128) {
    double acc = 0.0;
    for (int hh = 0; hh < a.G; ++hh)
      for (int r = s; r < e; ++r) acc += (double)__bfloat162float(a.q[(int64_t)(g * a.G + hh) * a.q_sh + (int64_t)r * 128 + tid]);
    qbar[tid] = acc / cnt;
  }
  __syncthreads();
  float* out = a.pooled + ((int64_t)g * a.T + t) * a.pool_stride;
  const double inv_sqrt_d = 1.0 / sqrt((double)a.d);
  double mx = -1e300;
  for (int j = tid; j < e; j += 256) {
    double acc = 0.0;
    const __nv_bfloat16* kr = a.k + (int64_t)g * a.kv_sh + (int64_t)j * 128;
    for (int dd = 0; dd < 128; ++dd) acc += (double)__bfloat162float(kr[dd]) * qbar[dd];
    acc *= inv_sqrt_d;
    out[j] = (float)acc;             // raw score parked in the output row
    a.scratch[((int64_t)g * a.T + t) * a.pool_stride + j] = acc;
    mx = fmax(mx, acc);
  }
  red[tid] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  double sum = 0.0;
  for (int j = tid; j < e; j += 256) sum += exp(a.scratch[((int64_t)g * a.T + t) * a.pool_stride + j] - mx);
  red[tid] = sum;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  sum = red[0];
  for (int j = tid; j < a.N; j += 256)
    out[j] = j < e ? (float)(exp(a.scratch[((int64_t)g * a.T + t) * a.pool_stride + j] - mx) / sum) : 0.f;
}

cudaError_t launch_dense_probs(const ProbsArgs& a, cudaStream_t st) {
  dim3 grid((a.N + 31) / 32, (a.N + 31) / 32, a.Hq);
  dense_probs_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pool_rows(const PoolRowsArgs& a, cudaStream_t st) {
  if (a.pre) {
    dim3 grid(a.T, a.Hkv);
    pre_pool_kernel<<<grid, 256, 0, st>>>(a);
  } else {
    dim3 grid((a.N + 255) / 256, a.T, a.all_heads ? 1 : a.Hkv);
    pool_rows_kernel<<<grid, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace kscd
