// Internal launch structs shared by the kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace kscd {

constexpr int kHeadDimC = 128;
constexpr float kLog2eC = 1.4426950408889634f;

enum { MODE_DENSE = 0, MODE_SPARSE = 1, MODE_SCORES = 2 };

struct DecodeArgs {
  int B, Hq, Hkv, G, n;
  const __nv_bfloat16* q;                 // [B][Hq][128]
  const __nv_bfloat16* k;                 // rows of (b, g): k + b*kv_sb + g*kv_sh + j*128
  const __nv_bfloat16* v;
  int64_t kv_sb, kv_sh;                   // elements
  float scale_log2;                       // softmax scale * log2(e)
  float* out;                             // fp32 [B][Hq][128]
  float* lse;                             // fp32 [B][Hq] natural log (nullable)
  // sparse selection: idx + b*idx_sb + src*idx_sh, counts at cnt + b*cnt_sb + src
  const int* idx;
  const int* cnt;
  int k_cap;
  int64_t idx_sb, idx_sh, cnt_sb;
  const int* head_map;                    // [Hkv] (nullable = identity)
  float* scores;                          // log2-domain scores [B][Hq][score_stride] (nullable)
  int64_t score_stride;
  float* part;                            // [B][Hq][splits][128]
  float* part_ml;                         // [B][Hq][splits][2]
  int* counters;                          // [B][Hkv], zero at allocation, self re-arming
  int splits;
};

cudaError_t launch_decode_attn(int mode, const DecodeArgs& a, cudaStream_t st);
int decode_tile_keys();

// Pooled post-softmax weights for decode tiles: pooled[b][g][j] =
// sum over the G heads of exp(s[b][h][j] - lse[b][h]).
struct PoolDecodeArgs {
  int B, Hq, Hkv, G, n;
  const float* scores;                    // log2-domain [B][Hq][score_stride]
  int64_t score_stride;
  const float* lse;                       // natural [B][Hq]
  float* pooled;                          // [B*Hkv][pool_stride]
  int64_t pool_stride;
};
cudaError_t launch_pool_decode(const PoolDecodeArgs& a, cudaStream_t st);

// Exact Top-k per row with the reference tie rule (smaller index wins),
// output ascending, padded with INT32_MAX up to k_cap.
struct TopkArgs {
  int rows;
  const float* vals;                      // row r at vals + r*val_stride (+ row_offset)
  int64_t val_stride;
  const int* lens;                        // per-row length (nullable => len)
  int len;
  const int* ks;                          // per-row k (nullable => k)
  int k;
  int* idx;                               // row r at idx + r*k_cap
  int* counts;                            // [rows]
  int k_cap;
};
cudaError_t launch_topk(const TopkArgs& a, cudaStream_t st);

}  // namespace kscd
