// C-ABI layer of libkascade_b200.so: host-side validation (the reference's
// InvalidArgument / Unsupported conditions), split-K planning and launches.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <string.h>

#include <string>

#include "../../include/kascade_b200.h"
#include "kscd_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return KSCD_OK;
  return fail(KSCD_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
}

constexpr int kMaxSplits = 64;

// Every row is stored 128 elements wide.  A logical head_dim d < 128 means
// the caller zero-padded Q and K past d (Q.K^T is then exact) and the
// default softmax scale is 1/sqrt(d); output columns >= d are padding.
bool bad_head_dim(int d) { return d < 1 || d > 128; }
#define KSCD_HEAD_DIM_MSG "head_dim %d unsupported (1..128; rows are 128 wide, zero-padded past head_dim)"
constexpr int kSmCount = 148;
constexpr int kCtasPerSm = 2;

// Largest split-K factor the planner may pick for `pairs` (b, g) pairs; the
// workspace is sized by it, so it depends on the batch and heads only.
int max_splits_for(int pairs) {
  const int slots = kSmCount * kCtasPerSm;
  const int want = std::max(1, (slots + pairs - 1) / pairs);
  return std::min(4 * want, kMaxSplits);
}

// Split-K factor: enough CTAs to cover the SMs in whole waves, each CTA a
// contiguous run of 64-key tiles of one (b, g).
int plan_splits(int pairs, int keys, int requested) {
  const int tiles = (keys + kscd::decode_tile_keys() - 1) / kscd::decode_tile_keys();
  const int cap = max_splits_for(pairs);
  if (requested > 0) return std::max(1, std::min({requested, cap, std::max(tiles, 1)}));
  const int slots = kSmCount * kCtasPerSm;
  const int want = std::max(1, (slots + pairs - 1) / pairs);
  int best = 1;
  double best_eff = -1.0;
  for (int s = want; s <= cap; ++s) {
    if (s > tiles) break;
    const int tps = (tiles + s - 1) / s;
    const int used = (tiles + tps - 1) / tps;            // splits that get work
    const double waves = (double)pairs * s / slots;
    const double eff = (waves / ceil(waves)) * ((double)tiles / (tps * (double)used));
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return std::max(1, std::min(best, std::max(tiles, 1)));
}

// The partial (m, l) block follows the partial O block of `splits` splits.
void set_splits(kscd::DecodeArgs& a, int splits) {
  a.splits = splits;
  a.part_ml = a.part + (size_t)a.B * a.Hq * splits * kscd::kHeadDimC;
}

// The tcgen05 dense / score passes (decode_tc.cu) split the keys stream-K
// style over one CTA per SM; a (sequence, kv head) may span up to the
// workspace's partial slots per head.
int tc_partial_slots(int pairs) { return max_splits_for(pairs); }

// Virtual kv heads per kv head for a query group of G heads: the smallest
// divisor r of G with G / r <= 16 (the decode kernel's m16 tile).
int kv_rep_for(int G) {
  for (int r = 1; r <= G; ++r)
    if (G % r == 0 && G / r <= 16) return r;
  return G;
}

size_t decode_ws_bytes(const kscd_decode_params* p) {
  const int G = p->num_kv_heads > 0 ? p->num_q_heads / p->num_kv_heads : 1;
  const int pairs = p->batch * p->num_kv_heads * kv_rep_for(std::max(G, 1));
  const size_t bh = (size_t)p->batch * p->num_q_heads;
  size_t bytes = bh * max_splits_for(pairs) * (kscd::kHeadDimC + 2) * sizeof(float);
  bytes = (bytes + 255) & ~(size_t)255;
  bytes += (size_t)pairs * sizeof(int);
  return bytes;
}

int check_decode(const kscd_decode_params* p, bool need_v, bool sparse) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->batch < 1 || p->num_q_heads < 1 || p->num_kv_heads < 1)
    return fail(KSCD_INVALID_ARGUMENT, "batch/num_q_heads/num_kv_heads must be >= 1");
  if (p->num_q_heads % p->num_kv_heads)
    return fail(KSCD_INVALID_ARGUMENT, "num_query_heads (%d) must be divisible by num_kv_heads (%d)",
                p->num_q_heads, p->num_kv_heads);
  if (p->seq_len < 1) return fail(KSCD_INVALID_ARGUMENT, "seq_len must be >= 1");
  if (!p->q || !p->k_cache || (need_v && !p->v_cache))
    return fail(KSCD_INVALID_ARGUMENT, "q/k_cache/v_cache must be non-NULL");
  if (need_v && !p->out) return fail(KSCD_INVALID_ARGUMENT, "out must be non-NULL");
  if (((uintptr_t)p->q | (uintptr_t)p->k_cache | (uintptr_t)p->v_cache) & 15)
    return fail(KSCD_INVALID_ARGUMENT, "q/k/v must be 16-byte aligned");
  if ((p->kv_stride_batch | p->kv_stride_head) & 7)
    return fail(KSCD_INVALID_ARGUMENT, "kv strides must be multiples of 8 elements");
  if (sparse) {
    if (!p->indices || !p->counts) return fail(KSCD_INVALID_ARGUMENT, "indices/counts must be non-NULL");
    if (p->k_cap < 1) return fail(KSCD_INVALID_ARGUMENT, "k_cap must be >= 1");
    if (p->num_src_heads < 1) return fail(KSCD_INVALID_ARGUMENT, "num_src_heads must be >= 1");
  }
  if (p->scores) {
    if (p->score_stride < p->seq_len || (p->score_stride & 1))
      return fail(KSCD_INVALID_ARGUMENT, "score_stride must be even and >= seq_len");
  }
  if (!p->workspace || p->workspace_bytes < decode_ws_bytes(p))
    return fail(KSCD_INVALID_ARGUMENT, "workspace too small (%zu < %zu bytes)", p->workspace_bytes,
                decode_ws_bytes(p));
  return KSCD_OK;
}

kscd::DecodeArgs make_args(const kscd_decode_params* p, int keys) {
  kscd::DecodeArgs a{};
  a.B = p->batch;
  a.Hq = p->num_q_heads;
  a.kv_rep = kv_rep_for(p->num_q_heads / p->num_kv_heads);
  a.Hkv = p->num_kv_heads * a.kv_rep;                // virtual heads (kscd_internal.h)
  a.G = p->num_q_heads / a.Hkv;
  a.n = p->seq_len;
  a.q = (const __nv_bfloat16*)p->q;
  a.k = (const __nv_bfloat16*)p->k_cache;
  a.v = (const __nv_bfloat16*)p->v_cache;
  a.kv_sb = p->kv_stride_batch;
  a.kv_sh = p->kv_stride_head;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
  a.scale_log2 = scale * kscd::kLog2eC;
  a.out = p->out;
  a.lse = p->lse;
  a.idx = p->indices;
  a.cnt = p->counts;
  a.k_cap = p->k_cap;
  a.idx_sb = (int64_t)p->num_src_heads * p->k_cap;
  a.idx_sh = p->k_cap;
  a.cnt_sb = p->num_src_heads;
  a.head_map = p->head_map;
  a.scores = p->scores;
  a.score_stride = p->score_stride;
  a.lens = p->seq_lens;
  a.splits = plan_splits(a.B * a.Hkv, keys, p->num_splits);
  const size_t bh = (size_t)a.B * a.Hq;
  a.part = (float*)p->workspace;
  a.part_ml = a.part + bh * a.splits * kscd::kHeadDimC;
  size_t off = bh * max_splits_for(a.B * a.Hkv) * (kscd::kHeadDimC + 2) * sizeof(float);
  off = (off + 255) & ~(size_t)255;
  a.counters = (int*)((char*)p->workspace + off);
  return a;
}

}  // namespace

extern "C" {

int kscd_abi_version(void) { return KSCD_ABI_VERSION; }

const char* kscd_last_error(void) { return g_last_error.c_str(); }

int32_t kscd_k_budget(double fraction, int32_t k_min, int32_t n) {
  if (n < 1) return 0;
  long long k = (long long)floor(fraction * (double)n);
  if (k < k_min) k = k_min;
  if (k > n) k = n;
  return (int32_t)k;
}

int kscd_decode_workspace_size(const kscd_decode_params* p, size_t* bytes) {
  if (!p || !bytes) return fail(KSCD_INVALID_ARGUMENT, "NULL argument");
  *bytes = decode_ws_bytes(p);
  return KSCD_OK;
}

int kscd_dense_decode(const kscd_decode_params* p, void* stream) {
  int rc = check_decode(p, true, false);
  if (rc) return rc;
  kscd::DecodeArgs a = make_args(p, p->seq_len);
  set_splits(a, tc_partial_slots(a.B * a.Hkv));
  return cuda_status(kscd::launch_decode_tc(kscd::MODE_DENSE, a, &p->k_cache, &p->v_cache, (cudaStream_t)stream),
                     "kscd_dense_decode");
}

int kscd_anchor_scores_decode(const kscd_decode_params* p, void* stream) {
  int rc = check_decode(p, false, false);
  if (rc) return rc;
  if (!p->scores || !p->lse) return fail(KSCD_INVALID_ARGUMENT, "scores and lse must be non-NULL");
  kscd::DecodeArgs a = make_args(p, p->seq_len);
  set_splits(a, tc_partial_slots(a.B * a.Hkv));
  return cuda_status(kscd::launch_decode_tc(kscd::MODE_SCORES, a, &p->k_cache, nullptr, (cudaStream_t)stream),
                     "kscd_anchor_scores_decode");
}

int kscd_sparse_decode(const kscd_decode_params* p, void* stream) {
  int rc = check_decode(p, true, true);
  if (rc) return rc;
  kscd::DecodeArgs a = make_args(p, p->k_cap);
  a.scores = nullptr;
  return cuda_status(kscd::launch_decode_attn(kscd::MODE_SPARSE, a, (cudaStream_t)stream), "kscd_sparse_decode");
}

// ---- several independent layers in one launch -------------------------
size_t decode_layer_ws_bytes(const kscd_decode_params* p) { return (decode_ws_bytes(p) + 255) & ~(size_t)255; }

int kscd_decode_layers_workspace_size(const kscd_decode_params* p, int32_t num_layers, size_t* bytes) {
  if (!p || !bytes || num_layers < 1) return fail(KSCD_INVALID_ARGUMENT, "NULL argument or num_layers < 1");
  *bytes = decode_layer_ws_bytes(p) * (size_t)num_layers;
  return KSCD_OK;
}

static int decode_layers(int mode, const kscd_decode_params* p, const kscd_decode_layers* t, void* stream,
                         const char* what) {
  if (!t) return fail(KSCD_INVALID_ARGUMENT, "layers is NULL");
  if (t->num_layers < 1) return fail(KSCD_INVALID_ARGUMENT, "num_layers must be >= 1");
  if (!t->k_caches || (mode != kscd::MODE_SCORES && !t->v_caches))
    return fail(KSCD_INVALID_ARGUMENT, "k_caches/v_caches must be non-NULL");
  if (p && mode == kscd::MODE_SCORES && (!p->scores || !p->lse))
    return fail(KSCD_INVALID_ARGUMENT, "scores and lse must be non-NULL");
  if (p && mode != kscd::MODE_SCORES && p->scores)
    return fail(KSCD_INVALID_ARGUMENT, "only the score pass writes scores");
  if (p && (t->q_stride_layer < (int64_t)p->batch * p->num_q_heads * 128 ||
            t->out_stride_layer < (int64_t)p->batch * p->num_q_heads * 128))
    return fail(KSCD_INVALID_ARGUMENT, "layer strides of q/out overlap");
  int rc = check_decode(p, mode != kscd::MODE_SCORES, mode == kscd::MODE_SPARSE);
  if (rc) return rc;
  const size_t per = decode_layer_ws_bytes(p);
  if (p->workspace_bytes < per * (size_t)t->num_layers)
    return fail(KSCD_INVALID_ARGUMENT, "workspace too small for %d layers (%zu < %zu bytes)", t->num_layers,
                p->workspace_bytes, per * (size_t)t->num_layers);
  kscd::DecodeArgs a = make_args(p, mode == kscd::MODE_SPARSE ? p->k_cap : p->seq_len);
  a.nl = t->num_layers;
  a.k_tab = (const __nv_bfloat16* const*)t->k_caches;
  a.v_tab = (const __nv_bfloat16* const*)(t->v_caches ? t->v_caches : t->k_caches);
  a.idx_ls = t->index_stride_layer;
  a.cnt_ls = t->count_stride_layer;
  a.scores_ls = t->scores_stride_layer;
  a.lse_ls = t->lse_stride_layer;
  a.q_ls = t->q_stride_layer;
  a.out_ls = t->out_stride_layer;
  a.head_map = t->head_maps;
  a.hm_ls = p->num_kv_heads;
  a.ws_ls = (int64_t)per;
  if (mode == kscd::MODE_SPARSE) return cuda_status(kscd::launch_decode_attn(mode, a, (cudaStream_t)stream), what);
  // dense / score passes: tcgen05 + TMA, tensor maps encoded from the host pointers
  if (!t->k_caches_host || (mode == kscd::MODE_DENSE && !t->v_caches_host))
    return fail(KSCD_INVALID_ARGUMENT, "k_caches_host / v_caches_host must be non-NULL for dense / score passes");
  set_splits(a, tc_partial_slots(a.B * a.Hkv));
  return cuda_status(kscd::launch_decode_tc(mode, a, t->k_caches_host,
                                            mode == kscd::MODE_DENSE ? t->v_caches_host : nullptr,
                                            (cudaStream_t)stream), what);
}

int kscd_sparse_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* t, void* stream) {
  return decode_layers(kscd::MODE_SPARSE, p, t, stream, "kscd_sparse_decode_layers");
}

int kscd_dense_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* t, void* stream) {
  return decode_layers(kscd::MODE_DENSE, p, t, stream, "kscd_dense_decode_layers");
}

int kscd_anchor_scores_decode_layers(const kscd_decode_params* p, const kscd_decode_layers* t, void* stream) {
  return decode_layers(kscd::MODE_SCORES, p, t, stream, "kscd_anchor_scores_decode_layers");
}

int kscd_select_decode(const kscd_select_decode_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (p->batch < 1 || p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads)
    return fail(KSCD_INVALID_ARGUMENT, "bad head/batch shape");
  if (p->seq_len < 1) return fail(KSCD_INVALID_ARGUMENT, "seq_len must be >= 1");
  if (!(p->topk_fraction > 0.0 && p->topk_fraction <= 1.0))
    return fail(KSCD_INVALID_ARGUMENT, "fraction must be in (0, 1], got %g", p->topk_fraction);
  if (p->k_min < 1) return fail(KSCD_INVALID_ARGUMENT, "k_min must be >= 1, got %d", p->k_min);
  if (!p->scores || !p->lse || !p->pooled || !p->indices || !p->counts)
    return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  if (p->pooled_stride < p->seq_len || (p->pooled_stride & 3) || (p->score_stride & 3) ||
      (((uintptr_t)p->scores | (uintptr_t)p->pooled) & 15))
    return fail(KSCD_INVALID_ARGUMENT, "pooled/score strides must be multiples of 4 and buffers 16-byte aligned");
  const int k = kscd_k_budget(p->topk_fraction, p->k_min, p->seq_len);
  if (p->k_cap < k) return fail(KSCD_INVALID_ARGUMENT, "k_cap %d < k_budget %d", p->k_cap, k);
  kscd::PoolDecodeArgs pa{};
  pa.B = p->batch;
  pa.Hq = p->num_q_heads;
  pa.Hkv = p->num_kv_heads;
  pa.G = p->num_q_heads / p->num_kv_heads;
  pa.n = p->seq_len;
  pa.scores = p->scores;
  pa.score_stride = p->score_stride;
  pa.lse = p->lse;
  pa.pooled = p->pooled;
  pa.pool_stride = p->pooled_stride;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = cuda_status(kscd::launch_pool_decode(pa, st), "pool_decode");
  if (rc) return rc;
  kscd::TopkArgs ta{};
  ta.rows = p->batch * p->num_kv_heads;
  ta.vals = p->pooled;
  ta.val_stride = p->pooled_stride;
  ta.len = p->seq_len;
  ta.k = k;
  ta.idx = p->indices;
  ta.counts = p->counts;
  ta.k_cap = p->k_cap;
  if (p->seq_lens) {          // ragged batch: per-sequence length and k_budget
    ta.seq_lens = p->seq_lens;
    ta.seq_div = p->num_kv_heads;
    ta.fraction = p->topk_fraction;
    ta.k_min = p->k_min;
  }
  return cuda_status(kscd::launch_topk(ta, st), "topk");
}

int kscd_topk(const kscd_topk_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (p->rows < 0) return fail(KSCD_INVALID_ARGUMENT, "rows must be >= 0");
  if (!p->ks && p->k < 1) return fail(KSCD_INVALID_ARGUMENT, "k must be >= 1, got %d", p->k);
  if (!p->lengths && p->length < 1) return fail(KSCD_INVALID_ARGUMENT, "p must be a non-empty vector");
  if (!p->values || !p->indices || !p->counts) return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  kscd::TopkArgs ta{};
  ta.rows = p->rows;
  ta.vals = p->values;
  ta.val_stride = p->value_stride;
  ta.lens = p->lengths;
  ta.len = p->length;
  ta.ks = p->ks;
  ta.k = p->k;
  ta.idx = p->indices;
  ta.counts = p->counts;
  ta.k_cap = p->k_cap;
  return cuda_status(kscd::launch_topk(ta, (cudaStream_t)stream), "kscd_topk");
}

// ------------------------------------------------------------------ prefill
static int check_prefill(const kscd_prefill_params* p, bool sparse) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->tile_size != 128) return fail(KSCD_UNSUPPORTED, "tile_size %d unsupported (engine tiles are 128)", p->tile_size);
  if (p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads)
    return fail(KSCD_INVALID_ARGUMENT, "num_query_heads (%d) must be divisible by num_kv_heads (%d)",
                p->num_q_heads, p->num_kv_heads);
  if (p->seq_len < 1) return fail(KSCD_INVALID_ARGUMENT, "seq_len must be >= 1");
  if (!p->q || !p->k || !p->v) return fail(KSCD_INVALID_ARGUMENT, "q/k/v must be non-NULL");
  if ((((uintptr_t)p->q | (uintptr_t)p->k | (uintptr_t)p->v) & 15) || ((p->q_stride_head | p->kv_stride_head) & 7))
    return fail(KSCD_INVALID_ARGUMENT, "q/k/v must be 16-byte aligned with head strides multiple of 8");
  if (sparse) {
    if (!p->indices || !p->counts || p->k_cap < 1 || p->num_src_heads < 1)
      return fail(KSCD_INVALID_ARGUMENT, "sparse prefill needs indices/counts/k_cap/num_src_heads");
  }
  return KSCD_OK;
}

static kscd::PrefillArgs make_prefill_args(const kscd_prefill_params* p) {
  kscd::PrefillArgs a{};
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  a.G = a.Hq / a.Hkv;
  a.N = p->seq_len;
  a.Nk = p->seq_len;
  a.slots = (a.G % 2 == 0) ? 2 : 1;
  a.causal = p->causal;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
  a.scale_log2 = scale * kscd::kLog2eC;
  a.q = (const __nv_bfloat16*)p->q;
  a.k = (const __nv_bfloat16*)p->k;
  a.v = (const __nv_bfloat16*)p->v;
  a.q_sh = p->q_stride_head;
  a.kv_sh = p->kv_stride_head;
  const int T = (p->seq_len + 127) / 128;
  a.idx = p->indices;
  a.cnt = p->counts;
  a.k_cap = p->k_cap;
  a.idx_sg = (int64_t)T * p->k_cap;
  a.idx_st = p->k_cap;
  a.cnt_sg = T;
  a.head_map = p->head_map;
  a.out = (__nv_bfloat16*)p->out;
  a.lse = p->lse;
  return a;
}

extern "C" int kscd_dense_prefill(const kscd_prefill_params* p, void* stream) {
  int rc = check_prefill(p, false);
  if (rc) return rc;
  if (!p->out) return fail(KSCD_INVALID_ARGUMENT, "out must be non-NULL");
  return cuda_status(kscd::launch_prefill_attn(kscd::PMODE_DENSE, make_prefill_args(p), (cudaStream_t)stream),
                     "kscd_dense_prefill");
}

extern "C" int kscd_anchor_lse_prefill(const kscd_prefill_params* p, void* stream) {
  int rc = check_prefill(p, false);
  if (rc) return rc;
  if (!p->lse) return fail(KSCD_INVALID_ARGUMENT, "lse must be non-NULL");
  return cuda_status(kscd::launch_prefill_attn(kscd::PMODE_LSE, make_prefill_args(p), (cudaStream_t)stream),
                     "kscd_anchor_lse_prefill");
}

extern "C" int kscd_sparse_prefill(const kscd_prefill_params* p, void* stream) {
  int rc = check_prefill(p, true);
  if (rc) return rc;
  if (!p->out) return fail(KSCD_INVALID_ARGUMENT, "out must be non-NULL");
  if (!p->causal) return fail(KSCD_UNSUPPORTED, "sparse prefill is causal (runner.py:275)");
  return cuda_status(kscd::launch_prefill_attn(kscd::PMODE_SPARSE, make_prefill_args(p), (cudaStream_t)stream),
                     "kscd_sparse_prefill");
}

extern "C" int kscd_dense_probs(const kscd_probs_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads || p->seq_len < 1)
    return fail(KSCD_INVALID_ARGUMENT, "bad shape");
  if (!p->q || !p->k || !p->lse || !p->probs) return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  kscd::ProbsArgs a{};
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  a.G = a.Hq / a.Hkv;
  a.N = p->seq_len;
  a.causal = p->causal;
  a.scale = p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
  a.q = (const __nv_bfloat16*)p->q;
  a.k = (const __nv_bfloat16*)p->k;
  a.q_sh = p->q_stride_head;
  a.kv_sh = p->kv_stride_head;
  a.lse = p->lse;
  a.P = p->probs;
  return cuda_status(kscd::launch_dense_probs(a, (cudaStream_t)stream), "kscd_dense_probs");
}

extern "C" int kscd_pool_tiles(const kscd_pool_tiles_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads || p->seq_len < 1 ||
      p->num_tiles < 1)
    return fail(KSCD_INVALID_ARGUMENT, "bad shape");
  if (!p->tile_starts || !p->tile_ends || !p->pooled) return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  if (p->pooling == 0 && !p->probs) return fail(KSCD_INVALID_ARGUMENT, "post pooling needs probs");
  if (p->pooling == 1 && (!p->q || !p->k || !p->scratch)) return fail(KSCD_INVALID_ARGUMENT, "pre pooling needs q/k/scratch");
  if (p->pooling == 1 && p->all_heads) return fail(KSCD_INVALID_ARGUMENT, "pre pooling is per kv head");
  if (p->pooled_stride < p->seq_len) return fail(KSCD_INVALID_ARGUMENT, "pooled_stride < seq_len");
  kscd::PoolRowsArgs a{};
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  a.G = a.Hq / a.Hkv;
  a.N = p->seq_len;
  a.T = p->num_tiles;
  a.starts = p->tile_starts;
  a.ends = p->tile_ends;
  a.pre = p->pooling == 1;
  a.all_heads = p->all_heads;
  a.P = p->probs;
  a.q = (const __nv_bfloat16*)p->q;
  a.k = (const __nv_bfloat16*)p->k;
  a.q_sh = p->q_stride_head;
  a.kv_sh = p->kv_stride_head;
  a.pooled = p->pooled;
  a.pool_stride = p->pooled_stride;
  a.scratch = p->scratch;
  a.d = p->head_dim;
  return cuda_status(kscd::launch_pool_rows(a, (cudaStream_t)stream), "kscd_pool_tiles");
}

namespace {
// One pass-B launch covers every head of a kv group (G <= 4) in post mode:
// the Top-k then runs in the tail of each pass-B CTA on its SM's scratch slot.
bool select_prefill_fused(const kscd_select_prefill_params* p) {
#ifdef KSCD_NO_FUSED_SELECT      // experiment builds only (A/B of the fused selection)
  return false;
#endif
  return !p->all_heads && p->num_q_heads / p->num_kv_heads <= 4;
}
size_t select_prefill_scratch_bytes(const kscd_select_prefill_params* p) {
  const size_t T = (size_t)(p->seq_len + 127) / 128;
  const size_t rows = select_prefill_fused(p) ? (size_t)kscd::sm_slots() : (p->all_heads ? 1 : p->num_kv_heads) * T;
  return 2 * rows * (size_t)p->pooled_stride * sizeof(float);
}
}  // namespace

extern "C" int kscd_select_prefill_scratch_size(const kscd_select_prefill_params* p, size_t* bytes) {
  if (!p || !bytes) return fail(KSCD_INVALID_ARGUMENT, "NULL argument");
  if (p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads || p->seq_len < 1)
    return fail(KSCD_INVALID_ARGUMENT, "bad shape");
  if (p->pooled_stride < p->seq_len) return fail(KSCD_INVALID_ARGUMENT, "pooled_stride < seq_len");
  *bytes = select_prefill_scratch_bytes(p);
  return KSCD_OK;
}

extern "C" int kscd_select_prefill(const kscd_select_prefill_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->tile_size != 128) return fail(KSCD_UNSUPPORTED, "tile_size %d unsupported", p->tile_size);
  if (p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads)
    return fail(KSCD_INVALID_ARGUMENT, "bad head shape");
  if (p->seq_len < 1) return fail(KSCD_INVALID_ARGUMENT, "seq_len must be >= 1");
  if (!(p->topk_fraction > 0.0 && p->topk_fraction <= 1.0))
    return fail(KSCD_INVALID_ARGUMENT, "fraction must be in (0, 1], got %g", p->topk_fraction);
  if (p->k_min < 1) return fail(KSCD_INVALID_ARGUMENT, "k_min must be >= 1, got %d", p->k_min);
  if (!p->q || !p->k || !p->lse || !p->pooled || !p->indices || !p->counts)
    return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  if (p->pooled_stride < p->seq_len || (p->pooled_stride & 3) || ((uintptr_t)p->pooled & 15))
    return fail(KSCD_INVALID_ARGUMENT, "pooled_stride must be >= seq_len and a multiple of 4, pooled 16-byte aligned");
  if (p->pooled_bytes < select_prefill_scratch_bytes(p))
    return fail(KSCD_INVALID_ARGUMENT, "pooled scratch too small (%zu < %zu bytes, kscd_select_prefill_scratch_size)",
                p->pooled_bytes, select_prefill_scratch_bytes(p));
  const int kmax = kscd_k_budget(p->topk_fraction, p->k_min, p->seq_len);
  if (p->k_cap < kmax) return fail(KSCD_INVALID_ARGUMENT, "k_cap %d < k_budget %d", p->k_cap, kmax);
  const int G = p->num_q_heads / p->num_kv_heads;
  const int T = (p->seq_len + 127) / 128;
  cudaStream_t st = (cudaStream_t)stream;
  kscd::PoolPrefillArgs pa{};
  pa.Hq = p->num_q_heads;
  pa.Hkv = p->num_kv_heads;
  pa.G = G;
  pa.N = p->seq_len;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
  pa.scale_log2 = scale * kscd::kLog2eC;
  pa.q = (const __nv_bfloat16*)p->q;
  pa.k = (const __nv_bfloat16*)p->k;
  pa.q_sh = p->q_stride_head;
  pa.kv_sh = p->kv_stride_head;
  pa.lse = p->lse;
  pa.pooled = p->pooled;
  pa.pool_stride = p->pooled_stride;
  if (select_prefill_fused(p)) {
    pa.head_begin = 0;
    pa.nheads = G;
    pa.g_fixed = -1;
    pa.accumulate = 0;
    pa.fuse = 1;
    pa.idx = p->indices;
    pa.counts = p->counts;
    pa.k_cap = p->k_cap;
    pa.fraction = p->topk_fraction;
    pa.k_min = p->k_min;
    return cuda_status(kscd::launch_pool_prefill(pa, st), "pool_prefill (fused Top-k)");
  }
  const int gcount = p->all_heads ? p->num_kv_heads : 1;
  int launches = 0;
  for (int gi = 0; gi < gcount; ++gi) {
    for (int hb = 0; hb < G; hb += 4) {
      pa.head_begin = hb;
      pa.nheads = std::min(4, G - hb);
      pa.g_fixed = p->all_heads ? gi : -1;
      pa.accumulate = launches > 0;
      int rc = cuda_status(kscd::launch_pool_prefill(pa, st), "pool_prefill");
      if (rc) return rc;
      ++launches;
    }
  }
  kscd::TopkArgs ta{};
  ta.rows = (p->all_heads ? 1 : p->num_kv_heads) * T;
  ta.vals = p->pooled;
  ta.vals2 = p->pooled + (int64_t)ta.rows * p->pooled_stride;   // second warpgroup's partial plane
  ta.val_stride = p->pooled_stride;
  ta.len = p->seq_len;
  ta.k = kmax;
  ta.idx = p->indices;
  ta.counts = p->counts;
  ta.k_cap = p->k_cap;
  ta.tile = 128;
  ta.T = T;
  ta.fraction = p->topk_fraction;
  ta.k_min = p->k_min;
  return cuda_status(kscd::launch_topk(ta, st), "topk");
}

}  // extern "C"

extern "C" int kscd_append_kv(const kscd_append_kv_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->num_layers < 1 || p->batch < 1 || p->num_kv_heads < 1 || p->position < 0)
    return fail(KSCD_INVALID_ARGUMENT, "bad shape");
  if (p->cache_capacity < 1) return fail(KSCD_INVALID_ARGUMENT, "cache_capacity must be >= 1");
  if (!p->seq_lens && p->position >= p->cache_capacity)
    return fail(KSCD_INVALID_ARGUMENT, "position %d outside the cache (capacity %d)", p->position,
                p->cache_capacity);
  if (!p->kv_new || !p->k_caches || !p->v_caches) return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  if (((uintptr_t)p->kv_new & 15) || (p->kv_stride_batch & 7) || (p->kv_stride_head & 7))
    return fail(KSCD_INVALID_ARGUMENT, "kv_new and cache strides must be 16-byte aligned");
  kscd::AppendKvArgs a{};
  a.L = p->num_layers;
  a.B = p->batch;
  a.Hkv = p->num_kv_heads;
  a.pos = p->position;
  a.kv_new = (const __nv_bfloat16*)p->kv_new;
  a.k_caches = (__nv_bfloat16* const*)p->k_caches;
  a.v_caches = (__nv_bfloat16* const*)p->v_caches;
  a.stride_b = p->kv_stride_batch;
  a.stride_h = p->kv_stride_head;
  a.lens = p->seq_lens;
  a.n_cap = p->cache_capacity;
  return cuda_status(kscd::launch_append_kv(a, (cudaStream_t)stream), "kscd_append_kv");
}

int kscd_masked_mass(const kscd_masked_mass_params* p, void* stream) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (p->num_sets < 0 || p->num_dists < 0 || p->rows < 0)
    return fail(KSCD_INVALID_ARGUMENT, "negative size");
  if (p->k_cap < 1) return fail(KSCD_INVALID_ARGUMENT, "k_cap must be >= 1, got %d", p->k_cap);
  if (p->dist_len < 1) return fail(KSCD_INVALID_ARGUMENT, "dist_len must be >= 1");
  if (p->dist_stride_row < p->dist_len) return fail(KSCD_INVALID_ARGUMENT, "dist rows overlap");
  if (!p->dist || !p->indices || !p->counts || !p->mass) return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  kscd::MaskedMassArgs a{};
  a.I = p->num_sets;
  a.J = p->num_dists;
  a.rows = p->rows;
  a.k_cap = p->k_cap;
  a.dist = p->dist;
  a.dist_head_stride = p->dist_stride_head;
  a.dist_row_stride = p->dist_stride_row;
  a.idx = p->indices;
  a.counts = p->counts;
  a.mass = p->mass;
  return cuda_status(kscd::launch_masked_mass(a, (cudaStream_t)stream), "kscd_masked_mass");
}

// ------------------------------------------------ pre-softmax selection
namespace kscd {
int pre_pool_chunk_keys(bool prefill);
}

namespace {

struct PreShape {
  bool prefill;
  int rows, T, chunks, chunk_keys;
};

int check_pre(const kscd_select_pre_params* p, PreShape* sh) {
  if (!p) return fail(KSCD_INVALID_ARGUMENT, "params is NULL");
  if (bad_head_dim(p->head_dim)) return fail(KSCD_UNSUPPORTED, KSCD_HEAD_DIM_MSG, p->head_dim);
  if (p->tile_size != 0 && p->tile_size != 128)
    return fail(KSCD_UNSUPPORTED, "tile_size %d unsupported (0 = decode, 128 = prefill)", p->tile_size);
  if (p->batch < 1 || p->num_q_heads < 1 || p->num_kv_heads < 1 || p->num_q_heads % p->num_kv_heads)
    return fail(KSCD_INVALID_ARGUMENT, "bad head/batch shape");
  if (p->tile_size == 128 && p->batch != 1) return fail(KSCD_INVALID_ARGUMENT, "prefill batch must be 1");
  if (p->seq_len < 1) return fail(KSCD_INVALID_ARGUMENT, "seq_len must be >= 1");
  sh->prefill = p->tile_size == 128;
  sh->T = sh->prefill ? (p->seq_len + 127) / 128 : 1;
  sh->rows = sh->prefill ? p->num_kv_heads * sh->T : p->batch * p->num_kv_heads;
  sh->chunk_keys = kscd::pre_pool_chunk_keys(sh->prefill);
  sh->chunks = (p->seq_len + sh->chunk_keys - 1) / sh->chunk_keys;
  return KSCD_OK;
}

size_t pre_ws_bytes(const PreShape& sh) {
  size_t bytes = (size_t)sh.rows * 128 * sizeof(float);
  bytes = (bytes + 255) & ~(size_t)255;
  return bytes + (size_t)sh.rows * sh.chunks * 2 * sizeof(float);
}

}  // namespace

extern "C" int kscd_select_pre_workspace_size(const kscd_select_pre_params* p, size_t* bytes) {
  PreShape sh;
  int rc = check_pre(p, &sh);
  if (rc) return rc;
  if (!bytes) return fail(KSCD_INVALID_ARGUMENT, "bytes is NULL");
  *bytes = pre_ws_bytes(sh);
  return KSCD_OK;
}

extern "C" int kscd_select_pre(const kscd_select_pre_params* p, void* stream) {
  PreShape sh;
  int rc = check_pre(p, &sh);
  if (rc) return rc;
  if (!(p->topk_fraction > 0.0 && p->topk_fraction <= 1.0))
    return fail(KSCD_INVALID_ARGUMENT, "fraction must be in (0, 1], got %g", p->topk_fraction);
  if (p->k_min < 1) return fail(KSCD_INVALID_ARGUMENT, "k_min must be >= 1, got %d", p->k_min);
  if (!p->q || !p->k || !p->pooled || !p->indices || !p->counts || !p->workspace)
    return fail(KSCD_INVALID_ARGUMENT, "NULL buffer");
  if (p->workspace_bytes < pre_ws_bytes(sh))
    return fail(KSCD_INVALID_ARGUMENT, "workspace too small (%zu < %zu bytes)", p->workspace_bytes, pre_ws_bytes(sh));
  if (p->pooled_stride < p->seq_len || (p->pooled_stride & 3) || ((uintptr_t)p->pooled & 15))
    return fail(KSCD_INVALID_ARGUMENT, "pooled_stride must be >= seq_len and a multiple of 4, pooled 16-byte aligned");
  if ((((uintptr_t)p->q | (uintptr_t)p->k) & 15) || (p->kv_stride_batch & 7) || (p->kv_stride_head & 7) ||
      (p->q_stride_head & 7))
    return fail(KSCD_INVALID_ARGUMENT, "q/k must be 16-byte aligned with strides multiple of 8 elements");
  const int k = kscd_k_budget(p->topk_fraction, p->k_min, p->seq_len);
  if (p->k_cap < k) return fail(KSCD_INVALID_ARGUMENT, "k_cap %d < k_budget %d", p->k_cap, k);
  kscd::PrePoolArgs a{};
  a.B = p->batch;
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  a.G = p->num_q_heads / p->num_kv_heads;
  a.n = p->seq_len;
  a.T = sh.T;
  a.prefill = sh.prefill;
  a.q = (const __nv_bfloat16*)p->q;
  a.q_sh = p->q_stride_head;
  a.k = (const __nv_bfloat16*)p->k;
  a.kv_sb = p->kv_stride_batch;
  a.kv_sh = p->kv_stride_head;
  a.scale = p->softmax_scale > 0.f ? p->softmax_scale : (float)(1.0 / sqrt((double)p->head_dim));
  a.pooled = p->pooled;
  a.pool_stride = p->pooled_stride;
  a.qbar = (float*)p->workspace;
  size_t off = ((size_t)sh.rows * 128 * sizeof(float) + 255) & ~(size_t)255;
  a.part = (float2*)((char*)p->workspace + off);
  a.chunks = sh.chunks;
  a.chunk_keys = sh.chunk_keys;
  a.lens = sh.prefill ? nullptr : p->seq_lens;
  a.mean_out = p->all_heads ? p->pooled + (int64_t)sh.rows * p->pooled_stride : nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  rc = cuda_status(kscd::launch_pre_pool(a, st), "pre_pool");
  if (rc) return rc;
  kscd::TopkArgs ta{};
  ta.rows = p->all_heads ? (sh.prefill ? sh.T : p->batch) : sh.rows;
  ta.vals = p->all_heads ? a.mean_out : p->pooled;
  ta.val_stride = p->pooled_stride;
  ta.len = p->seq_len;
  ta.k = k;
  ta.idx = p->indices;
  ta.counts = p->counts;
  ta.k_cap = p->k_cap;
  ta.fraction = p->topk_fraction;
  ta.k_min = p->k_min;
  if (sh.prefill) {
    ta.tile = 128;
    ta.T = sh.T;
  } else if (p->seq_lens) {
    ta.seq_lens = p->seq_lens;
    ta.seq_div = p->all_heads ? 1 : p->num_kv_heads;
  }
  return cuda_status(kscd::launch_topk(ta, st), "topk");
}
