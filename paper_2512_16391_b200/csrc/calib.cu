// Offline calibration on the GPU: the gather-sum at
// the heart of the reference's head similarity and planning similarity
// matrix.  For index-set head i, distribution head j and row r (a token for
// per-token distributions, a tile for tile-pooled ones):
//
//     mass[i][j][r] = sum_{t < counts[i][r]} dist[j][r][idx[i][r][t]]   (fp64)
//
// heads.py:96-108 (num / den of head_similarity_from_dists: anchor head i's
// per-token Top-k set, or reuse head j's own, applied to reuse head j's
// distribution) and metrics.py:254-260 (pair_score of the planning matrix:
// anchor layer a's tile set of head i applied to layer b's pooled tile
// distribution of head j).  One warp per (i, j, r); the Top-k sets come from
// the exact radix-select kernel (topk.cu), the distributions from
// kscd_pool_tiles (compat.cu) -- so the whole calibration pass stays on the
// device and only the [I][J][rows] masses travel to the host.  L2-bound
// gathers; the sets are read once per (i, r) and reused by the J warps of
// the same CTA.
#include "common.cuh"
#include "kscd_internal.h"

namespace kscd {

constexpr int kMassWarps = 8;

__global__ void __launch_bounds__(kMassWarps * 32) masked_mass_kernel(const MaskedMassArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x;
  const int i = blockIdx.y;
  const int cnt = min(a.counts[(int64_t)i * a.rows + r], a.k_cap);
  const int* idx = a.idx + ((int64_t)i * a.rows + r) * a.k_cap;
  for (int j = blockIdx.z * kMassWarps + warp; j < a.J; j += gridDim.z * kMassWarps) {
    const float* d = a.dist + (int64_t)j * a.dist_head_stride + (int64_t)r * a.dist_row_stride;
    double acc = 0.0;
    for (int t = lane; t < cnt; t += 32) acc += (double)__ldg(d + __ldg(idx + t));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) a.mass[((int64_t)i * a.J + j) * a.rows + r] = acc;
  }
}

cudaError_t launch_masked_mass(const MaskedMassArgs& a, cudaStream_t st) {
  if (a.rows <= 0 || a.I <= 0 || a.J <= 0) return cudaSuccess;
  dim3 grid(a.rows, a.I, (a.J + kMassWarps - 1) / kMassWarps);
  masked_mass_kernel<<<grid, kMassWarps * 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace kscd
