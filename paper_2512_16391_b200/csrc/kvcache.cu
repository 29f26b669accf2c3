// Decode-step KV append: the step's new K/V rows of every layer, staged in
// one contiguous bf16 buffer [L][2][B][Hkv][128], are scattered into the
// per-layer caches at row `position` in ONE launch (instead of 2L strided
// copies), so a host -> device -> decode -> host step is a single CUDA graph.
// 16-byte vector per thread: 16 threads per 256-byte row.
#include <algorithm>

#include "kscd_internal.h"

namespace kscd {

__global__ void append_kv_kernel(AppendKvArgs a) {
  const long long total = (long long)a.L * 2 * a.B * a.Hkv * 16;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int chunk = (int)(t & 15);
    long long row = t >> 4;                     // ((l*2 + kv)*B + b)*Hkv + h
    const int h = (int)(row % a.Hkv);
    row /= a.Hkv;
    const int b = (int)(row % a.B);
    row /= a.B;
    const int kv = (int)(row & 1);
    const int l = (int)(row >> 1);
    const uint4 v = reinterpret_cast<const uint4*>(a.kv_new)[t];
    __nv_bfloat16* base = kv ? a.v_caches[l] : a.k_caches[l];
    const long long pos = a.lens ? (long long)__ldg(a.lens + b) - 1 : (long long)a.pos;
    if (pos < 0 || pos >= a.n_cap) continue;   // a bad ragged length never writes outside its rows
    __nv_bfloat16* dst = base + (long long)b * a.stride_b + (long long)h * a.stride_h + pos * 128;
    reinterpret_cast<uint4*>(dst)[chunk] = v;
  }
}

cudaError_t launch_append_kv(const AppendKvArgs& a, cudaStream_t st) {
  const long long total = (long long)a.L * 2 * a.B * a.Hkv * 16;
  const int threads = 256;
  const int blocks = (int)std::min<long long>((total + threads - 1) / threads, 148 * 8);
  append_kv_kernel<<<blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace kscd
