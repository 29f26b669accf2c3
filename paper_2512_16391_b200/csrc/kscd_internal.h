// Internal launch structs shared by the kernels and the C-ABI layer.
#pragma once
#include <cuda.h>
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
  // groups of more than 16 query heads run as kv_rep "virtual" kv heads of
  // G = Hq / (Hkv * kv_rep) query heads each; Hkv and G above are the
  // virtual ones, and virtual head gv reads kv head gv / kv_rep
  int kv_rep;
  const int* lens;                        // [B] per-sequence key counts (nullable => n)
  // several layers in one launch (blockIdx.z = layer * B + b): layer l reads
  // q + l*q_ls, caches k_tab[l] / v_tab[l] (nullable => k / v), head_map +
  // l*hm_ls, writes out + l*out_ls, and uses the workspace at + l*ws_ls bytes
  int nl;
  const __nv_bfloat16* const* k_tab;
  const __nv_bfloat16* const* v_tab;
  int64_t q_ls, out_ls, hm_ls, ws_ls;
  // per-layer index lists / counts / scores / lse (element strides, may be
  // negative; 0 = shared by every layer of the launch)
  int64_t idx_ls, cnt_ls, scores_ls, lse_ls;
};

cudaError_t launch_decode_attn(int mode, const DecodeArgs& a, cudaStream_t st);
int decode_tile_keys();

// tcgen05 / TMA decode (decode_tc.cu) for the dense and score passes: K / V
// blocks reach shared memory through per-layer TMA tensor maps, so a launch
// carries up to kMaxMapLayers layers' maps (more layers: several launches)
constexpr int kMaxMapLayers = 16;
struct DecodeTmaps {
  CUtensorMap k[kMaxMapLayers];
  CUtensorMap v[kMaxMapLayers];
  CUtensorMap q;                          // [layers][B*Hq][128] bf16, 16-row boxes
};
// k_ptrs / v_ptrs: HOST arrays of the layers' cache base pointers (v_ptrs
// nullable for the score pass); rows past a.n read as zeros through TMA
cudaError_t launch_decode_tc(int mode, const DecodeArgs& a, const void* const* k_ptrs, const void* const* v_ptrs,
                             cudaStream_t st);
int decode_tc_block_keys();

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
  const float* vals2;                     // optional second plane, same layout: value = vals + vals2
  int64_t val_stride;
  const int* lens;                        // per-row length (nullable => len)
  int len;
  const int* ks;                          // per-row k (nullable => k)
  int k;
  int* idx;                               // row r at idx + r*k_cap
  int* counts;                            // [rows]
  int k_cap;
  // prefill tiles: when tile > 0, row r is tile (r % T) with length
  // min(len, tile*(i+1)) and k = k_budget(fraction, k_min, length)
  int tile, T;
  double fraction;
  int k_min;
  // ragged decode batch: when seq_div > 0, row r has length
  // min(len, seq_lens[r / seq_div]) and k = k_budget(fraction, k_min, length)
  const int* seq_lens;
  int seq_div;
};
cudaError_t launch_topk(const TopkArgs& a, cudaStream_t st);

// ------------------------------------------------------------------ prefill
enum { PMODE_DENSE = 0, PMODE_SPARSE = 1, PMODE_LSE = 2 };

struct PrefillArgs {
  int Hq, Hkv, G, N, Nk;                  // batch 1 (the paper's prefill setting)
  int slots;                              // query tiles per CTA: 2 heads of a group (G even) or 1
  int causal;
  float scale_log2;
  const __nv_bfloat16* q;                 // [Hq][N][128], head stride q_sh
  const __nv_bfloat16* k;                 // [Hkv][Nk][128], head stride kv_sh
  const __nv_bfloat16* v;
  int64_t q_sh, kv_sh;
  // sparse: list of (kv head src, tile t) at idx + src*idx_sg + t*idx_st, length cnt[src*cnt_sg + t]
  const int* idx;
  const int* cnt;
  int k_cap;
  int64_t idx_sg, idx_st, cnt_sg;
  const int* head_map;                    // [Hkv] (nullable = identity)
  __nv_bfloat16* out;                     // [Hq][N][128]
  float* lse;                             // [Hq][N] natural log (nullable)
};
cudaError_t launch_prefill_attn(int mode, const PrefillArgs& a, cudaStream_t st);

// Anchor pass B (tile-pooled post-softmax weights), one chunk of <= 4 heads
// of every kv group per launch.
struct PoolPrefillArgs {
  int Hq, Hkv, G, N;
  int head_begin, nheads;                 // head chunk inside each group
  int accumulate;                         // add into pooled instead of storing
  int g_fixed;                            // >= 0: only this kv head, rows indexed by tile only
  float scale_log2;
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  int64_t q_sh, kv_sh;
  const float* lse;                       // [Hq][N] natural
  float* pooled;                          // [Hkv or 1][T][pool_stride]; fused: [slots][2][pool_stride]
  int64_t pool_stride;
  // fused anchor selection (one launch covers the whole group, post mode):
  // each CTA writes its pooled row into the slot of its SM and runs the exact
  // Top-k of that row in its tail -- no [Hkv][T][N] scratch held for the layer
  int fuse;
  int* idx;                               // [Hkv][T][k_cap]
  int* counts;                            // [Hkv][T]
  int k_cap;
  double fraction;
  int k_min;
};
cudaError_t launch_pool_prefill(const PoolPrefillArgs& a, cudaStream_t st);
constexpr int kSmSlots = 160;            // >= %smid + 1 on B200 (148 SMs): scratch slots of the fused pass B
int sm_slots();

// ------------------------------------------------------- calibration (calib.cu)
struct MaskedMassArgs {
  int I, J, rows, k_cap;
  const float* dist;                      // [J] heads, row r at + j*dist_head_stride + r*dist_row_stride
  int64_t dist_head_stride, dist_row_stride;
  const int* idx;                         // [I][rows][k_cap]
  const int* counts;                      // [I][rows]
  double* mass;                           // [I][J][rows]
};
cudaError_t launch_masked_mass(const MaskedMassArgs& a, cudaStream_t st);

// ------------------------------------------------------------ compat (small N)
struct ProbsArgs {
  int Hq, Hkv, G, N, causal;
  float scale;                            // natural-log softmax scale
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  int64_t q_sh, kv_sh;
  const float* lse;                       // [Hq][N] natural
  float* P;                               // [Hq][N][N]
};
cudaError_t launch_dense_probs(const ProbsArgs& a, cudaStream_t st);

struct PoolRowsArgs {
  int Hq, Hkv, G, N, T;
  const int* starts;                      // [T] tile row ranges
  const int* ends;
  int pre, all_heads;
  const float* P;                         // post: [Hq][N][N]
  const __nv_bfloat16* q;                 // pre
  const __nv_bfloat16* k;
  int64_t q_sh, kv_sh;
  float* pooled;                          // [Hkv or 1][T][pool_stride]
  int64_t pool_stride;
  double* scratch;                        // pre: [Hkv][T][pool_stride]
  int d;                                  // logical head dim (pre-softmax scale 1/sqrt(d))
};
cudaError_t launch_pool_rows(const PoolRowsArgs& a, cudaStream_t st);

struct AppendKvArgs {
  int L, B, Hkv, pos;
  const __nv_bfloat16* kv_new;            // [L][2][B][Hkv][128]
  __nv_bfloat16* const* k_caches;         // device [L] pointers, rows b*stride_b + h*stride_h + j*128
  __nv_bfloat16* const* v_caches;
  int64_t stride_b, stride_h;             // elements
  const int* lens;                        // [B] ragged: row at lens[b] - 1 (nullable => pos)
  int n_cap;                              // rows per cache; rows outside [0, n_cap) are skipped
};
cudaError_t launch_append_kv(const AppendKvArgs& a, cudaStream_t st);

// Pre-softmax pooled selection (pre_pool.cu).  Rows are (b, g) in decode
// (T = 1) and (g, t) in prefill; a row's visible keys are [0, len(row)).
struct PrePoolArgs {
  int B, Hq, Hkv, G, n;                   // n: decode keys / prefill N
  int T;                                  // prefill tiles (decode: 1)
  bool prefill;
  const __nv_bfloat16* q;                 // decode [B][Hq][128]; prefill [Hq][N][128] (q_sh)
  int64_t q_sh;
  const __nv_bfloat16* k;                 // decode rows k + b*kv_sb + g*kv_sh + j*128; prefill k + g*kv_sh + j*128
  int64_t kv_sb, kv_sh;
  float scale;                            // natural-log softmax scale
  float* pooled;                          // [rows][pool_stride]: scores, then probabilities
  int64_t pool_stride;
  float* qbar;                            // [rows][128] fp32
  float2* part;                           // [rows][chunks] (max, sum of exp(s - max))
  int chunks, chunk_keys;                 // per-row partials (prefill: chunk_keys = 128)
  const int* lens;                        // decode ragged [B] (nullable)
  float* mean_out;                        // all-heads: [B or T][pool_stride] mean over kv heads (nullable)
};
cudaError_t launch_pre_pool(const PrePoolArgs& a, cudaStream_t st);

}  // namespace kscd
