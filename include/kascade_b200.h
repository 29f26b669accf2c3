/*
 * kascade_b200.h -- C ABI of the B200-native Kascade anchor/reuse attention
 * engine (libkascade_b200.so, sm_100a).
 *
 * Every entry point replaces one step of the reference package's hot path
 * (kascade 0.1.0, /root/reference/pkg/src/kascade; cited file:line below).
 * The reference is a pure-Python/numpy library with no FFI, so the boundary
 * it would bind is this library through ctypes; the
 * package `paper_2512_16391_b200` is that binding.
 *
 * Conventions
 *   - Plain C: POD parameter structs, raw device pointers, sizes in elements
 *     unless the name says bytes.  No allocation and no device
 *     synchronisation happen inside a call: all work is enqueued on `stream`
 *     (a cudaStream_t passed as void*, NULL = legacy default stream), so the
 *     calls are CUDA-graph capturable.
 *   - Dtypes: Q/K/V bf16 rows of 128 elements (256 bytes); outputs, scores
 *     and LSE fp32; index lists int32.  head_dim is the logical head size,
 *     1..128: for head_dim < 128 the caller zero-pads Q and K past head_dim
 *     (Q.K^T is then exact), the default softmax scale is 1/sqrt(head_dim),
 *     and output columns >= head_dim are padding.  The performance path is
 *     head_dim 128 (the reference's small-d test traces use the padding).
 *   - Index-list wire format (anchor -> reuse): int32 idx[rows][k_cap] sorted
 *     ascending and padded with INT32_MAX, plus int32 counts[rows] -- the
 *     reference's TopKIndexSet.indices (attention.py:40-67) per (kv head,
 *     tile), with rows = batch * kv_heads for decode.
 *   - Return value: KSCD_OK or an error code; kscd_last_error() returns a
 *     thread-local message for the last failing call on this thread.  The
 *     Python binding maps the codes to the reference's exception types
 *     (errors.py:8-58): 1 InvalidArgumentError, 2 UnsupportedOperationError,
 *     3 KascadeError (CUDA launch/runtime failure).
 *   - Workspace: callers allocate `kscd_decode_workspace_size()` bytes and
 *     zero-fill them ONCE at allocation; kernels leave the workspace re-armed.
 */
#ifndef KASCADE_B200_H_
#define KASCADE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KSCD_OK 0
#define KSCD_INVALID_ARGUMENT 1
#define KSCD_UNSUPPORTED 2
#define KSCD_CUDA_ERROR 3

#define KSCD_ABI_VERSION 2

/* One decode step of one layer for a batch of sequences (the reference's
 * decode tile [t, t+1) with causal bound n = t + 1, tiles.py:145-150). */
typedef struct kscd_decode_params {
  int32_t batch;          /* B */
  int32_t num_q_heads;    /* Hq; query head h reads kv head h / (Hq/Hkv), trace.py:38-43; any group size */
  int32_t num_kv_heads;   /* Hkv */
  int32_t head_dim;       /* 1..128, see Conventions */
  int32_t seq_len;        /* n: keys 0..n-1 are visible (the step's own token included) */
  const void* q;          /* bf16 [B][Hq][128], contiguous */
  const void* k_cache;    /* bf16; row j of (b, g) at k_cache + b*kv_stride_batch + g*kv_stride_head + j*128 */
  const void* v_cache;    /* bf16, same layout as k_cache */
  int64_t kv_stride_batch, kv_stride_head;   /* elements; rows are contiguous (stride 128) */
  float softmax_scale;    /* <= 0 selects 1/sqrt(head_dim) (attention.py:120) */
  float* out;             /* fp32 [B][Hq][128] */
  float* lse;             /* fp32 [B][Hq] natural-log normaliser; may be NULL */
  /* sparse selection (kscd_sparse_decode): the list of kv head g in
   * sequence b is indices + (b*num_src_heads + src)*k_cap with
   * src = head_map[g] (runner.py:210-225), length counts[b*num_src_heads + src]. */
  const int32_t* indices;
  const int32_t* counts;
  int32_t k_cap;
  int32_t num_src_heads;  /* kv heads of the anchor's list (usually Hkv) */
  const int32_t* head_map;/* device int32 [Hkv]; NULL = identity */
  /* log2-domain scores s*log2(e) of every (b, h, key) (anchor layers);
   * kscd_dense_decode writes them when non-NULL. */
  float* scores;          /* fp32 [B][Hq][score_stride], score_stride even and >= n */
  int64_t score_stride;
  void* workspace;
  size_t workspace_bytes;
  int32_t num_splits;     /* split-K factor; 0 = automatic */
  /* ragged batch (serving; the reference decodes one trace at a time):
   * device int32 [B], sequence b sees keys 0..seq_lens[b]-1 (each
   * <= seq_len, which then only bounds the split planning); NULL = seq_len
   * for every sequence.  Sparse calls take their lengths from the lists. */
  const int32_t* seq_lens;
} kscd_decode_params;

/* Several independent decode layers in ONE launch (e.g. every reuse layer
 * between two anchors: they share the anchor's index lists and differ in
 * queries, caches and head maps).  `p` describes layer 0 (shapes, strides,
 * lists, q/out of layer 0); layer l reads q + l*q_stride_layer and caches
 * k_caches[l] / v_caches[l] (same shape and strides as layer 0), routes
 * through head_maps[l*Hkv ...] and writes out + l*out_stride_layer.  The
 * workspace holds kscd_decode_layers_workspace_size bytes.  A launch of L
 * layers has L x the CTAs of one, so small layers (few (sequence, kv head)
 * rows, short lists) stop paying a grid ramp each. */
typedef struct kscd_decode_layers {
  int32_t num_layers;
  const void* const* k_caches;  /* device array of L pointers, bf16 [B][Hkv][n_cap][128] */
  const void* const* v_caches;
  int64_t q_stride_layer;       /* elements between consecutive layers' q */
  int64_t out_stride_layer;     /* elements between consecutive layers' out */
  const int32_t* head_maps;     /* device int32 [L][Hkv], or NULL = identity */
  /* per-layer lists (p->indices / counts of layer 0, e.g. a group of
   * consecutive anchors each attending its own fresh sets) and per-layer score
   * / lse outputs (the anchors' pass 1); element strides, may be negative;
   * 0 = one list shared by every layer (reuse runs) */
  int64_t index_stride_layer, count_stride_layer;
  int64_t scores_stride_layer, lse_stride_layer;
  /* HOST arrays of the same L cache pointers: the dense and score passes
   * stream K / V through TMA tensor maps encoded on the host per layer
   * (required by kscd_dense_decode_layers / kscd_anchor_scores_decode_layers) */
  const void* const* k_caches_host;
  const void* const* v_caches_host;
} kscd_decode_layers;

/* Selection of one decode step: pooled post-softmax weights of the G heads
 * of each kv head (runner.py:148-152), k = k_budget(n) (tiles.py:81-89) and
 * the exact Top-k (attention.py:147-174). */
typedef struct kscd_select_decode_params {
  int32_t batch, num_q_heads, num_kv_heads, seq_len;
  const float* scores;    /* from kscd_dense_decode / kscd_anchor_scores_decode */
  int64_t score_stride;
  const float* lse;       /* natural-log LSE of the same call */
  float* pooled;          /* scratch fp32 [B*Hkv][pooled_stride], pooled_stride % 4 == 0, >= n */
  int64_t pooled_stride;
  double topk_fraction;   /* KBudgetPolicy.fraction in (0, 1] */
  int32_t k_min;          /* KBudgetPolicy.k_min >= 1 */
  int32_t* indices;       /* int32 [B*Hkv][k_cap] */
  int32_t* counts;        /* int32 [B*Hkv] */
  int32_t k_cap;          /* >= k_budget(n) */
  const int32_t* seq_lens;/* device int32 [B] or NULL: per-sequence n, k = k_budget(seq_lens[b]) */
} kscd_select_decode_params;

/* Generic exact Top-k over rows of fp32 values (oracle_topk_indices). */
typedef struct kscd_topk_params {
  int32_t rows;
  const float* values;    /* row r at values + r*value_stride */
  int64_t value_stride;
  const int32_t* lengths; /* device [rows] or NULL (=> length) */
  int32_t length;
  const int32_t* ks;      /* device [rows] or NULL (=> k) */
  int32_t k;
  int32_t* indices;       /* [rows][k_cap] */
  int32_t* counts;        /* [rows] = min(k, length) */
  int32_t k_cap;
} kscd_topk_params;

/* Prefill of one layer (batch 1, the paper's prefill setting).  Query tiles
 * are the reference's prefill tiles of 128 rows (tiles.py:137-144). */
typedef struct kscd_prefill_params {
  int32_t num_q_heads, num_kv_heads, head_dim, seq_len;   /* head_dim 1..128 */
  int32_t causal;          /* 1: row r sees keys <= r (attention.py:123-127) */
  const void* q;           /* bf16 [Hq][N][128], rows contiguous, head stride q_stride_head */
  const void* k;           /* bf16 [Hkv][N][128], head stride kv_stride_head */
  const void* v;
  int64_t q_stride_head, kv_stride_head;   /* elements, multiples of 8 */
  float softmax_scale;     /* <= 0 selects 1/sqrt(head_dim) */
  void* out;               /* bf16 [Hq][N][128] contiguous */
  float* lse;              /* fp32 [Hq][N] natural-log normaliser (nullable for attention) */
  /* sparse: the list of (source kv head s, tile t) is indices + (s*T + t)*k_cap,
   * sorted ascending, length counts[s*T + t]; kv head g reads s = head_map[g]. */
  const int32_t* indices;
  const int32_t* counts;
  int32_t k_cap;
  int32_t num_src_heads;
  const int32_t* head_map; /* device int32 [Hkv]; NULL = identity */
  int32_t tile_size;       /* must be 128 */
} kscd_prefill_params;

/* Pooled post-softmax weights of every prefill tile (anchor pass B) + the
 * exact Top-k of each (kv head, tile) with k = k_budget(causal bound). */
typedef struct kscd_select_prefill_params {
  int32_t num_q_heads, num_kv_heads, head_dim, seq_len;
  const void* q;
  const void* k;
  int64_t q_stride_head, kv_stride_head;
  float softmax_scale;
  const float* lse;        /* fp32 [Hq][N] from kscd_dense_prefill / kscd_anchor_lse_prefill */
  float* pooled;           /* fp32 scratch, kscd_select_prefill_scratch_size bytes: when one pass covers
                              the kv group (G <= 4, not all-heads) two row planes per SM slot, each CTA
                              selecting in its own tail (the fused anchor selection); otherwise
                              [2][Hkv or 1][T][pooled_stride] partial-sum planes for a separate Top-k */
  int64_t pooled_stride;   /* >= N, multiple of 4 */
  size_t pooled_bytes;     /* size of pooled (checked) */
  double topk_fraction;
  int32_t k_min;
  int32_t all_heads;       /* 1: all-heads-pooled mode, one shared set per tile (runner.py:180-197) */
  int32_t* indices;        /* int32 [Hkv or 1][T][k_cap] */
  int32_t* counts;         /* int32 [Hkv or 1][T] */
  int32_t k_cap;           /* >= k_budget(N) */
  int32_t tile_size;       /* must be 128 */
} kscd_select_prefill_params;

/* Pre-softmax pooled selection at engine scale (runner.py:155-161, the
 * comparison mode SPEC.md:370): per (kv head, tile) q_bar = the fp64 mean of
 * the tile's G x T query rows, scores = K[:t1] q_bar * scale, pooled =
 * softmax(scores) (fp32 result, as softmax_row, attention.py:77-90), then the
 * exact Top-k with k = k_budget(t1).  Decode: the tile is the step's token
 * (T = 1 row per sequence, t1 = n); prefill: 128-row tiles.  all_heads: the
 * kv heads' pooled vectors are averaged into one shared set (runner.py:180-197).
 * No attention pass is needed (anchor layers skip pass A / the score pass). */
typedef struct kscd_select_pre_params {
  int32_t batch;           /* decode: B; prefill: must be 1 */
  int32_t num_q_heads, num_kv_heads, head_dim;
  int32_t seq_len;         /* decode: n (keys 0..n-1 visible); prefill: N */
  int32_t tile_size;       /* 0: decode (one query token per sequence); 128: prefill tiles */
  const void* q;           /* decode bf16 [B][Hq][128] contiguous; prefill bf16 [Hq][N][128] */
  int64_t q_stride_head;   /* prefill: elements between heads (decode: ignored) */
  const void* k;           /* decode: cache bf16 [B][Hkv][n_cap][128]; prefill bf16 [Hkv][N][128] */
  int64_t kv_stride_batch, kv_stride_head;   /* elements (kv_stride_batch: decode only) */
  float softmax_scale;     /* <= 0 selects 1/sqrt(head_dim) */
  float* pooled;           /* scratch fp32 rows: decode [B*Hkv (+B)][pooled_stride],
                              prefill [Hkv*T (+T)][pooled_stride] (+ rows: all_heads) */
  int64_t pooled_stride;   /* >= seq_len, multiple of 4 */
  void* workspace;         /* kscd_select_pre_workspace_size bytes, any content */
  size_t workspace_bytes;
  double topk_fraction;
  int32_t k_min;
  int32_t all_heads;
  int32_t* indices;        /* int32 [rows][k_cap]; rows = B*Hkv or Hkv*T (B or T with all_heads) */
  int32_t* counts;         /* int32 [rows] */
  int32_t k_cap;           /* >= k_budget(seq_len) */
  const int32_t* seq_lens; /* decode: device int32 [B] or NULL (ragged batch, k = k_budget(seq_lens[b])) */
} kscd_select_pre_params;

/* Reference-scale helpers for the trace-level API (small N only). */
typedef struct kscd_probs_params {
  int32_t num_q_heads, num_kv_heads, head_dim, seq_len, causal;
  const void* q;           /* bf16 [Hq][N][128] */
  const void* k;           /* bf16 [Hkv][N][128] */
  int64_t q_stride_head, kv_stride_head;
  float softmax_scale;     /* <= 0 selects 1/sqrt(head_dim) */
  const float* lse;        /* fp32 [Hq][N] from kscd_dense_prefill */
  float* probs;            /* fp32 [Hq][N][N] */
} kscd_probs_params;

typedef struct kscd_pool_tiles_params {
  int32_t num_q_heads, num_kv_heads, head_dim, seq_len;
  int32_t num_tiles;
  const int32_t* tile_starts;   /* device [T]: rows [start, end) of each tile, end = causal bound */
  const int32_t* tile_ends;
  int32_t pooling;              /* 0 post-softmax (needs probs), 1 pre-softmax (needs q, k) */
  int32_t all_heads;            /* post only: pool every query head into one row per tile */
  const float* probs;           /* fp32 [Hq][N][N] */
  const void* q;
  const void* k;
  int64_t q_stride_head, kv_stride_head;
  float* pooled;                /* fp32 [Hkv or 1][T][pooled_stride] */
  int64_t pooled_stride;
  double* scratch;              /* pre: fp64 [Hkv][T][pooled_stride] */
} kscd_pool_tiles_params;

/* Decode-step KV append (engine plumbing for serving decode; the reference
 * reads whole traces and has no cache): writes the step's new K/V rows of
 * every layer at cache row `position` in one launch. */
typedef struct kscd_append_kv_params {
  int32_t num_layers, batch, num_kv_heads, head_dim;
  int32_t position;             /* cache row written, < cache capacity */
  const void* kv_new;           /* bf16 [L][2][B][Hkv][128], 16-byte aligned */
  void* const* k_caches;        /* device array of L pointers, bf16 [B][Hkv][n_cap][128] */
  void* const* v_caches;
  int64_t kv_stride_batch, kv_stride_head;   /* elements, shared by every layer's cache */
  const int32_t* seq_lens;      /* device int32 [B] or NULL: ragged batch, sequence b's row goes to
                                   seq_lens[b] - 1 (position is then ignored) */
  int32_t cache_capacity;       /* n_cap: rows per (sequence, kv head) of every cache; position must be
                                   < n_cap, and a ragged row outside [0, n_cap) is skipped (never written) */
} kscd_append_kv_params;

int kscd_abi_version(void);
const char* kscd_last_error(void);

/* Bytes of workspace the decode entry points need for these shapes. */
int kscd_decode_workspace_size(const kscd_decode_params* p, size_t* bytes);
/* ... and a multi-layer launch of num_layers layers. */
int kscd_decode_layers_workspace_size(const kscd_decode_params* p, int32_t num_layers, size_t* bytes);
/* Reuse / sparse layers (as kscd_sparse_decode) and dense layers (as
 * kscd_dense_decode without scores or lse), several per launch. */
int kscd_sparse_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* layers, void* stream);
int kscd_dense_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* layers, void* stream);
/* Anchor pass 1 (as kscd_anchor_scores_decode: scores + lse, no V) of
 * several anchor layers in one launch. */
int kscd_anchor_scores_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* layers, void* stream);

/* Dense attention of the step's query over keys 0..n-1: out, lse, and --
 * when p->scores != NULL -- the scores the anchor-0 selection pools.
 * Replaces dense_attention (attention.py:106-144) for the decode row; the
 * dense (Top-k = 100%) baseline mode and layer 0 of run_kascade
 * (runner.py:250-262). */
int kscd_dense_decode(const kscd_decode_params* p, void* stream);

/* Anchor pass 1: scores + lse only, V untouched. */
int kscd_anchor_scores_decode(const kscd_decode_params* p, void* stream);

/* Sparse attention over a selected key list per kv head, gathered through
 * the head-remap table: topk_attention (attention.py:185-253) on the
 * decode tile with _routed_selections (runner.py:210-225). */
int kscd_sparse_decode(const kscd_decode_params* p, void* stream);

/* Pooled post-softmax weights + k_budget + exact Top-k of one decode step
 * (runner.py:164-207 in remapped mode). */
int kscd_select_decode(const kscd_select_decode_params* p, void* stream);

/* oracle_topk_indices (attention.py:147-174) over device rows. */
int kscd_topk(const kscd_topk_params* p, void* stream);

/* Dense causal prefill attention: O and LSE for every row (dense_attention,
 * attention.py:106-144, without materialising P); the Top-k = 100% baseline
 * and the anchor-0 layer. */
int kscd_dense_prefill(const kscd_prefill_params* p, void* stream);

/* Anchor pass A: LSE of every row only (no P V). */
int kscd_anchor_lse_prefill(const kscd_prefill_params* p, void* stream);

/* Sparse prefill over the (kv head, tile) selections routed through the head
 * map, with the causal staircase and the diagonal fallback (topk_attention,
 * attention.py:185-253; runner.py:210-225). */
int kscd_sparse_prefill(const kscd_prefill_params* p, void* stream);

/* Anchor selection for prefill (runner.py:164-207). */
int kscd_select_prefill(const kscd_select_prefill_params* p, void* stream);

/* dense_attention's materialised P (attention.py:121-142) for small N:
 * exp(s - lse) on visible entries, exact zeros elsewhere. */
int kscd_dense_probs(const kscd_probs_params* p, void* stream);

/* Pooled distributions of arbitrary tiles (any TileSpec, tiles.py:117-152):
 * post-softmax _post_pooled (runner.py:148-152, fp64 sums) or pre-softmax
 * _pre_pooled (runner.py:155-161). */
int kscd_pool_tiles(const kscd_pool_tiles_params* p, void* stream);

int kscd_append_kv(const kscd_append_kv_params* p, void* stream);

/* Bytes of `pooled` scratch kscd_select_prefill needs for these shapes. */
int kscd_select_prefill_scratch_size(const kscd_select_prefill_params* p, size_t* bytes);

/* Pre-softmax pooled selection (see kscd_select_pre_params): q_bar, the
 * scores against K, the row softmax and the exact Top-k, stream-ordered. */
int kscd_select_pre(const kscd_select_pre_params* p, void* stream);
int kscd_select_pre_workspace_size(const kscd_select_pre_params* p, size_t* bytes);

/* Offline calibration gather-sum: mass[i][j][r] =
 * fp64 sum over t < counts[i][r] of dist[j][r][indices[i][r][t]] -- the
 * num / den terms of head_similarity_from_dists (heads.py:96-108) and of the
 * planning matrix's pair_score (metrics.py:254-260). */
typedef struct kscd_masked_mass_params {
  int32_t num_sets;             /* I: index-set heads */
  int32_t num_dists;            /* J: distribution heads */
  int32_t rows;                 /* tokens or tiles */
  const float* dist;            /* fp32; row r of head j at dist + j*dist_stride_head + r*dist_stride_row */
  int64_t dist_stride_head, dist_stride_row;
  int32_t dist_len;             /* valid columns of a row (indices must be < dist_len) */
  const int32_t* indices;       /* [I][rows][k_cap], entries < dist_len */
  const int32_t* counts;        /* [I][rows], <= k_cap */
  int32_t k_cap;
  double* mass;                 /* [I][J][rows] */
} kscd_masked_mass_params;

int kscd_masked_mass(const kscd_masked_mass_params* p, void* stream);

/* k_budget (tiles.py:81-89): min(max(floor(fraction*n), k_min), n). */
int32_t kscd_k_budget(double fraction, int32_t k_min, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* KASCADE_B200_H_ */
