"""Prefill-path parity (tcgen05 kernels through the C ABI) against the CPU
oracle and the reference's frozen config-1 vectors.  Needs a B200."""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import kascade_oracle as orc
from parity import assert_outputs_close, topk_swaps

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.to(dtype) if dtype is not None else t).cuda()


def _bf(x):
    return _dev(x, torch.bfloat16)


def _rand(seed, Hq, Hkv, N, qscale=1.0):
    rng = np.random.default_rng(seed)
    Q = orc.bf16_round((rng.standard_normal((Hq, N, 128)) * qscale).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((Hkv, N, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((Hkv, N, 128)).astype(np.float32))
    return Q, K, V


def _oracle_lse(Q, K, causal=True):
    Hq, N, _ = Q.shape
    G = Hq // K.shape[0]
    out = np.zeros((Hq, N))
    for h in range(Hq):
        s = (Q[h].astype(np.float64) @ K[h // G].astype(np.float64).T) / math.sqrt(128)
        if causal:
            s = np.where(np.tril(np.ones((N, N), bool)), s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        out[h] = (m + np.log(np.exp(s - m).sum(axis=1, keepdims=True)))[:, 0]
    return out


@pytest.mark.parametrize("Hq,Hkv,N,causal", [(4, 2, 300, True), (2, 1, 128, True), (3, 3, 130, True),
                                             (8, 2, 1000, True), (4, 2, 300, False), (4, 1, 1, True)])
def test_dense_prefill_matches_oracle(cuda_ok, Hq, Hkv, N, causal):
    from paper_2512_16391_b200 import ops
    Q, K, V = _rand(N + Hq, Hq, Hkv, N)
    _, Y = orc.dense_layer(Q, K, V, causal=causal)
    out, lse = ops.dense_prefill(_bf(Q), _bf(K), _bf(V), causal=causal)
    torch.cuda.synchronize()
    assert_outputs_close(out.float().cpu().numpy(), Y)
    np.testing.assert_allclose(lse.cpu().numpy(), _oracle_lse(Q, K, causal), rtol=1e-5, atol=2e-4)


def test_dense_prefill_heavy_tailed_rescale(cuda_ok):
    # large logits force the lazy O rescale path (running max grows > 2^8)
    from paper_2512_16391_b200 import ops
    Q, K, V = _rand(5, 4, 2, 700, qscale=6.0)
    _, Y = orc.dense_layer(Q, K, V)
    out, _ = ops.dense_prefill(_bf(Q), _bf(K), _bf(V))
    # peaked rows make |O| ~ |V| ~ 1-4, where the bf16 OUTPUT rounding alone
    # is 2^-9 relative: bound the error relative to magnitude here
    got = out.float().cpu().numpy()
    err = np.abs(got - Y)
    assert (err <= 2e-2 + 8e-3 * np.abs(Y)).all(), err.max()
    assert np.linalg.norm(got - Y) / np.linalg.norm(Y) < 5e-3


def test_lse_pass_matches_dense_lse(cuda_ok):
    from paper_2512_16391_b200 import ops
    Q, K, V = _rand(2, 8, 2, 900)
    _, lse_d = ops.dense_prefill(_bf(Q), _bf(K), _bf(V))
    lse_a = ops.anchor_lse_prefill(_bf(Q), _bf(K))
    np.testing.assert_allclose(lse_a.cpu().numpy(), lse_d.cpu().numpy(), rtol=1e-6, atol=1e-5)


def _synth_layer(seed, Hq, Hkv, N):
    Q, K, V = orc.synth_qkv(1, Hq, Hkv, 128, N, seed=seed, rho=0.95)
    return [orc.bf16_round(x[0]) for x in (Q, K, V)]


def test_select_prefill_matches_oracle(cuda_ok):
    from paper_2512_16391_b200 import ops
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    Hq, Hkv, N = 8, 2, 1000
    Q, K, V = _synth_layer(3, Hq, Hkv, N)
    pol = KBudgetPolicy(0.1, 32)
    _, lse = ops.dense_prefill(_bf(Q), _bf(K), _bf(V))
    idx, cnt = ops.select_prefill(_bf(Q), _bf(K), lse, pol)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    swaps = 0
    G = Hq // Hkv
    for g in range(Hkv):
        for t in range((N + 127) // 128):
            s, e = t * 128, min(N, t * 128 + 128)
            ref, pooled = orc.prefill_tile_select(Q, K, g, G, s, e, 0.1, 32)
            assert cnt[g, t] == ref.size
            swaps += topk_swaps(idx[g, t, :ref.size], ref, pooled)
    assert swaps <= 3


def test_select_prefill_all_heads_mode(cuda_ok):
    from paper_2512_16391_b200 import ops
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    Hq, Hkv, N = 4, 2, 400
    Q, K, V = _synth_layer(4, Hq, Hkv, N)
    pol = KBudgetPolicy(0.25, 16)
    _, lse = ops.dense_prefill(_bf(Q), _bf(K), _bf(V))
    idx, cnt = ops.select_prefill(_bf(Q), _bf(K), lse, pol, all_heads=True)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for t in range((N + 127) // 128):
        s, e = t * 128, min(N, t * 128 + 128)
        pooled = np.mean([orc.prefill_tile_select(Q, K, g, 2, s, e, 0.25, 16)[1] for g in range(Hkv)], axis=0)
        ref = orc.topk_sorted(pooled, orc.k_budget(0.25, 16, e))
        topk_swaps(idx[0, t, :cnt[0, t]], ref, pooled)


def test_sparse_prefill_remap_staircase_fallback(cuda_ok):
    from paper_2512_16391_b200 import ops
    Hq, Hkv, N = 8, 4, 700
    Q, K, V = _rand(8, Hq, Hkv, N)
    T = (N + 127) // 128
    rng = np.random.default_rng(1)
    k_cap = 300
    idx = np.full((Hkv, T, k_cap), 2**31 - 1, np.int32)
    cnt = np.zeros((Hkv, T), np.int32)
    for s in range(Hkv):
        for t in range(T):
            e = min(N, 128 * t + 128)
            if t == 0 and s == 1:
                sel = np.array([100, 120, 127])                      # early rows fall back to V[r]
            else:
                sel = np.sort(rng.choice(e, int(rng.integers(1, min(k_cap, e) + 1)), replace=False))
            idx[s, t, :sel.size] = sel
            cnt[s, t] = sel.size
    head_map = [1, 3, 0, 2]
    out, _ = ops.sparse_prefill(_bf(Q), _bf(K), _bf(V), _dev(idx), _dev(cnt), _dev(np.array(head_map, np.int32)))
    G = Hq // Hkv
    ref = np.zeros((Hq, N, 128), np.float32)
    fb = 0
    for g in range(Hkv):
        for t in range(T):
            s, e = 128 * t, min(N, 128 * t + 128)
            src = head_map[g]
            sel = idx[src, t, :cnt[src, t]].astype(np.int64)
            y, _, f = orc.sparse_tile(Q, K, V, g, G, s, e, sel)
            ref[g * G:(g + 1) * G, s:e] = y
            fb += len(f)
    assert fb > 0
    assert_outputs_close(out.float().cpu().numpy(), ref)


def test_full_budget_sparse_prefill_equals_dense(cuda_ok):
    # test_attention.py:184-192: selecting every causal key reproduces dense
    from paper_2512_16391_b200 import ops
    Hq, Hkv, N = 4, 2, 500
    Q, K, V = _rand(9, Hq, Hkv, N)
    T = (N + 127) // 128
    idx = np.full((Hkv, T, N), 2**31 - 1, np.int32)
    cnt = np.zeros((Hkv, T), np.int32)
    for g in range(Hkv):
        for t in range(T):
            e = min(N, 128 * t + 128)
            idx[g, t, :e] = np.arange(e)
            cnt[g, t] = e
    sp, _ = ops.sparse_prefill(_bf(Q), _bf(K), _bf(V), _dev(idx), _dev(cnt))
    de, _ = ops.dense_prefill(_bf(Q), _bf(K), _bf(V))
    np.testing.assert_allclose(sp.float().cpu().numpy(), de.float().cpu().numpy(), rtol=0, atol=2e-2)
    assert np.abs(sp.float().cpu().numpy() - de.float().cpu().numpy()).mean() < 1e-4


def test_config1_prefill_vs_reference_golden(cuda_ok):
    """BASELINE configs[0] shapes (4 layers, 8Q/2KV, d=128, N=2048, k=10%,
    anchors {0,2}) through the prefill engine vs the reference's
    run_kascade(phase='prefill'): anchor selections of every tile and the
    last tile's outputs of every layer."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    a = json.load(open(os.path.join(GOLDEN, "golden.json")))["synth_sha256"]["config1"]["args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"])
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    z = golden("config1")
    N = Q.shape[2]
    maps = {l: HeadMap(l, max(x for x in (0, 2) if x <= l), m) for l, m in enumerate(z["head_maps"].tolist())
            if m[0] >= 0}
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps=maps, k_policy=KBudgetPolicy(0.1, 128))
    eng = engine.KascadePrefill(plan, 4, 8, 2, N)
    qs = [_bf(Q[l]) for l in range(4)]
    ks = [_bf(K[l]) for l in range(4)]
    vs = [_bf(V[l]) for l in range(4)]
    # selections of anchor 0 (engine state after running only layer 0's kind)
    from paper_2512_16391_b200 import ops
    for ai, layer in enumerate((0, 2)):
        _, lse = ops.dense_prefill(qs[layer], ks[layer], vs[layer])
        idx, cnt = ops.select_prefill(qs[layer], ks[layer], lse, plan.k_policy)
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        for g in range(2):
            for t in range(N // 128):
                ref = z["pre_idx"][ai, g, t, :cnt[g, t]]
                if np.array_equal(idx[g, t, :cnt[g, t]], ref):
                    continue
                _, pooled = orc.prefill_tile_select(Q[layer], K[layer], g, 4, 128 * t, 128 * t + 128, 0.1, 128)
                topk_swaps(idx[g, t, :cnt[g, t]], ref, pooled)
    out = eng.forward(qs, ks, vs).float().cpu().numpy()
    assert_outputs_close(out[:, :, N - 128:], z["pre_last_tile"])
