"""Decode-path parity: CUDA kernels (through the C ABI) vs the CPU oracle and
the reference's frozen golden vectors.  Needs a B200."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import kascade_oracle as orc
from parity import assert_outputs_close, topk_swaps

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _rand_decode(seed, B, Hq, Hkv, n, n_cap=None, scale_q=1.0):
    rng = np.random.default_rng(seed)
    n_cap = n_cap or n
    q = orc.bf16_round(rng.standard_normal((B, Hq, 128)).astype(np.float32) * scale_q)
    K = orc.bf16_round(rng.standard_normal((B, Hkv, n_cap, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((B, Hkv, n_cap, 128)).astype(np.float32))
    return q, K, V


def _oracle_dense(q, K, V, n):
    B, Hq, _ = q.shape
    G = Hq // K.shape[1]
    Y = np.zeros((B, Hq, 128), np.float32)
    P = np.zeros((B, Hq, n), np.float32)
    lse = np.zeros((B, Hq))
    for b in range(B):
        for h in range(Hq):
            P[b, h], Y[b, h] = orc.dense_row(q[b, h], K[b, h // G, :n], V[b, h // G, :n])
            s = (K[b, h // G, :n].astype(np.float64) @ q[b, h].astype(np.float64)) / math.sqrt(128)
            lse[b, h] = s.max() + np.log(np.exp(s - s.max()).sum())
    return P, Y, lse


@pytest.mark.parametrize("n", [1, 63, 64, 1000, 4133])
def test_dense_decode_matches_oracle(cuda_ok, n):
    from paper_2512_16391_b200 import ops
    B, Hq, Hkv = 3, 8, 2
    q, K, V = _rand_decode(n, B, Hq, Hkv, n, n_cap=n + 5)
    _, Y, lse = _oracle_dense(q, K, V, n)
    sc = ops.score_buffer(B, Hq, n, "cuda")
    out, lse_g = ops.dense_decode(_dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16), n,
                                  scores=sc)
    torch.cuda.synchronize()
    assert_outputs_close(out.cpu().numpy(), Y)
    np.testing.assert_allclose(lse_g.cpu().numpy(), lse, rtol=1e-5, atol=1e-4)
    s_ref = np.einsum("bhnd,bhd->bhn", K[:, :, :n].astype(np.float64).repeat(Hq // Hkv, axis=1),
                      q.astype(np.float64)) / math.sqrt(128) * (1 / math.log(2))
    np.testing.assert_allclose(sc[:, :, :n].cpu().numpy(), s_ref, rtol=1e-5, atol=2e-5)


@pytest.mark.parametrize("splits", [1, 3, 17])
def test_dense_decode_split_invariance(cuda_ok, splits):
    from paper_2512_16391_b200 import ops
    q, K, V = _rand_decode(7, 2, 32, 8, 3000)
    args = [_dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16), 3000]
    ref, _ = ops.dense_decode(*args, num_splits=1)
    got, _ = ops.dense_decode(*args, num_splits=splits)
    # P is rounded to bf16 relative to each split's running max, so splits
    # agree to bf16 rounding of P, not bit-for-bit; repeat runs are exact
    np.testing.assert_allclose(got.cpu().numpy(), ref.cpu().numpy(), rtol=0, atol=1e-3)
    again, _ = ops.dense_decode(*args, num_splits=splits)
    np.testing.assert_array_equal(again.cpu().numpy(), got.cpu().numpy())


def test_dense_decode_group16(cuda_ok):
    # Llama-70B-like grouping (64Q/8KV -> G = 8) and the G > 8 kernel path (G = 16)
    from paper_2512_16391_b200 import ops
    for Hq, Hkv in ((64, 8), (32, 2)):
        q, K, V = _rand_decode(Hq, 2, Hq, Hkv, 700)
        _, Y, _ = _oracle_dense(q, K, V, 700)
        out, _ = ops.dense_decode(_dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16), 700)
        assert_outputs_close(out.cpu().numpy(), Y)


def test_sparse_decode_head_remap_matches_oracle(cuda_ok):
    from paper_2512_16391_b200 import ops
    B, Hq, Hkv, n = 2, 16, 4, 2500
    q, K, V = _rand_decode(3, B, Hq, Hkv, n)
    rng = np.random.default_rng(9)
    head_map = [2, 0, 3, 1]
    k_cap = 300
    idx = np.full((B, Hkv, k_cap), 2**31 - 1, np.int32)
    cnt = np.zeros((B, Hkv), np.int32)
    for b in range(B):
        for s in range(Hkv):
            c = int(rng.integers(1, k_cap + 1))
            sel = np.sort(rng.choice(n, c, replace=False))
            idx[b, s, :c] = sel
            cnt[b, s] = c
    out = ops.sparse_decode(_dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16), n,
                            _dev(idx), _dev(cnt), _dev(np.array(head_map, np.int32)))
    G = Hq // Hkv
    ref = np.zeros((B, Hq, 128), np.float32)
    for b in range(B):
        for g in range(Hkv):
            src = head_map[g]
            sel = idx[b, src, :cnt[b, src]].astype(np.int64)
            ks, vs = K[b, g, sel], V[b, g, sel]
            for j in range(G):
                s = (q[b, g * G + j][None] @ ks.T) * np.float32(1 / math.sqrt(128))
                p = orc.masked_softmax(s, np.ones_like(s, bool))
                ref[b, g * G + j] = (p @ vs)[0]
    assert_outputs_close(out.cpu().numpy(), ref)


def test_full_budget_sparse_equals_dense(cuda_ok):
    # test_attention.py:184-192 on the decode tile: k = n selects every key
    from paper_2512_16391_b200 import ops
    B, Hq, Hkv, n = 2, 8, 2, 1500
    q, K, V = _rand_decode(4, B, Hq, Hkv, n)
    qd, Kd, Vd = _dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16)
    dense, _ = ops.dense_decode(qd, Kd, Vd, n)
    idx = torch.arange(n, dtype=torch.int32, device="cuda").repeat(B, Hkv, 1).contiguous()
    cnt = torch.full((B, Hkv), n, dtype=torch.int32, device="cuda")
    sp = ops.sparse_decode(qd, Kd, Vd, n, idx, cnt)
    # the dense pass runs on the tcgen05 kernel and the sparse pass on the
    # gather kernel: both round P to bf16 once, in different key orders, so
    # they agree to the bf16 weight rounding (2^-9 relative per weight)
    _, Y, _ = _oracle_dense(q, K, V, n)
    for got in (dense, sp):
        rel = assert_outputs_close(got.cpu().numpy(), Y)[2]
        assert rel < 3e-3, rel
    np.testing.assert_allclose(sp.cpu().numpy(), dense.cpu().numpy(), rtol=0, atol=1e-3)


def test_topk_contract_golden(cuda_ok):
    from paper_2512_16391_b200 import ops
    z = golden("topk")
    for i in range(int(z["n"])):
        w = z[f"w{i}"].astype(np.float32)
        k = int(z[f"k{i}"])
        idx, cnt = ops.topk(_dev(w[None]), k)
        c = int(cnt.item())
        got = idx[0, :c].cpu().numpy()
        if np.array_equal(w.astype(np.float64), z[f"w{i}"]):   # exactly representable: bit-exact contract
            np.testing.assert_array_equal(got, z[f"idx{i}"])
        else:
            topk_swaps(got, z[f"idx{i}"], z[f"w{i}"])


def test_topk_ties_and_padding(cuda_ok):
    from paper_2512_16391_b200 import ops
    rng = np.random.default_rng(3)
    w = np.round(rng.random((5, 70000)) * 64).astype(np.float32) / 64  # massive ties
    for k in (1, 100, 6999, 69999, 70000, 80000):
        idx, cnt = ops.topk(_dev(w), k, k_cap=max(k, 8))
        idx = idx.cpu().numpy()
        for r in range(5):
            ref = orc.topk_sorted(w[r], k)
            assert int(cnt[r]) == ref.size
            np.testing.assert_array_equal(idx[r, :ref.size], ref)
            assert (idx[r, ref.size:] == 2**31 - 1).all()


@pytest.mark.parametrize("dist", ["lognormal", "heavy", "tied_block", "aliased"])
def test_topk_long_rows_exact(cuda_ok, dist):
    # long rows take the sample-banded first radix digit; tied blocks and a
    # pattern aliased with the sample stride force its exact fallback
    from paper_2512_16391_b200 import ops
    rng = np.random.default_rng(17)
    n = 150001
    if dist == "lognormal":
        w = np.exp(rng.standard_normal((3, n)) * 2).astype(np.float32)
    elif dist == "heavy":
        w = (rng.pareto(1.5, (3, n)) + 1e-9).astype(np.float32)
    elif dist == "tied_block":
        w = np.exp(rng.standard_normal((3, n))).astype(np.float32)
        w[:, 1000:60000] = np.float32(1.5)          # a huge tie straddling the threshold
    else:
        w = rng.random((3, n)).astype(np.float32)
        w[:, ::16] += np.float32(10.0)              # every sampled key is large: the band misses
    for k in (1, 128, 15000, 149999):
        idx, cnt = ops.topk(_dev(w), k, k_cap=k)
        idx = idx.cpu().numpy()
        for r in range(3):
            np.testing.assert_array_equal(idx[r, :cnt[r]], orc.topk_sorted(w[r], k))


def test_select_decode_matches_oracle(cuda_ok):
    from paper_2512_16391_b200 import ops
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    B, Hq, Hkv, n = 2, 32, 8, 5000
    q, K, V = _rand_decode(5, B, Hq, Hkv, n, scale_q=3.0)
    P, _, _ = _oracle_dense(q, K, V, n)
    sc = ops.score_buffer(B, Hq, n, "cuda")
    _, lse = ops.dense_decode(_dev(q, torch.bfloat16), _dev(K, torch.bfloat16), _dev(V, torch.bfloat16), n,
                              scores=sc)
    pol = KBudgetPolicy(0.1, 128)
    idx, cnt = ops.select_decode(sc, lse, n, pol, Hkv)
    k = orc.k_budget(0.1, 128, n)
    swaps = 0
    G = Hq // Hkv
    for b in range(B):
        for g in range(Hkv):
            pooled = P[b, g * G:(g + 1) * G][:, None, :].mean(axis=(0, 1), dtype=np.float64)
            ref = orc.topk_sorted(pooled, k)
            assert int(cnt[b, g]) == k
            swaps += topk_swaps(idx[b, g, :k].cpu().numpy(), ref, pooled)
    assert swaps <= 2


@pytest.mark.parametrize("B,Hq,Hkv,n,all_heads", [(2, 32, 8, 50000, False), (3, 16, 1, 20000, False),
                                                 (2, 32, 8, 30000, True), (1, 8, 2, 3000, False)])
def test_select_decode_fused_pooling(cuda_ok, B, Hq, Hkv, n, all_heads):
    """The pooling runs inside the Top-k's first pass: the pooled buffer it
    writes is sum_i exp2(s_i - lse_i log2 e) over the row's heads, and the
    lists equal a plain Top-k over that buffer (bit-exact)."""
    from paper_2512_16391_b200 import ops
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    g = torch.Generator(device="cuda").manual_seed(11)
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    K = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    V = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    sc = ops.score_buffer(B, Hq, n, "cuda")
    _, lse = ops.dense_decode(q, K, V, n, scores=sc)
    pol = KBudgetPolicy(0.1, 128)
    Hs = 1 if all_heads else Hkv
    pooled = torch.full((B * Hs, (n + 3) // 4 * 4), float("nan"), device="cuda")
    idx, cnt = ops.select_decode(sc, lse, n, pol, Hkv, pooled=pooled, all_heads=all_heads)
    G = Hq // Hs
    w = torch.exp2(sc[:, :, :n] - (lse * 1.4426950408889634)[:, :, None]).reshape(B * Hs, G, n).sum(1)
    torch.testing.assert_close(pooled[:, :n], w, rtol=2e-6, atol=1e-12)
    k = int(cnt.flatten()[0])
    ridx, rcnt = ops.topk(pooled[:, :n].contiguous(), k)
    assert torch.equal(idx.view(B * Hs, -1)[:, :k], ridx[:, :k])
    assert torch.equal(cnt.flatten(), rcnt)


def _config1():
    import json
    import os
    from conftest import GOLDEN
    a = json.load(open(os.path.join(GOLDEN, "golden.json")))["synth_sha256"]["config1"]["args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"])
    return [orc.bf16_round(x) for x in (Q, K, V)]


def test_decode_step_config1_vs_reference_golden(cuda_ok):
    """BASELINE configs[0]: 4 layers, 8Q/2KV, d=128, ctx 2K, batch 1 decode,
    Top-k 10%, anchors {0,2} -- the engine's decode step against the
    reference's own run_kascade(phase='decode') last row."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    Q, K, V = _config1()
    z = golden("config1")
    N = Q.shape[2]
    maps = {l: HeadMap(l, max(a for a in (0, 2) if a <= l), m) for l, m in enumerate(z["head_maps"].tolist())
            if m[0] >= 0}
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps=maps, k_policy=KBudgetPolicy(0.1, 128))
    dec = engine.KascadeDecoder(plan, 4, 1, 8, 2, N)
    qd = _dev(Q[:, None, :, -1], torch.bfloat16)                       # [L][B=1][Hq][d]
    Kd = [_dev(K[l][None], torch.bfloat16) for l in range(4)]
    Vd = [_dev(V[l][None], torch.bfloat16) for l in range(4)]
    out = dec.step(qd, Kd, Vd, N).cpu().numpy()[:, 0]
    assert_outputs_close(out, z["dec_Y"])
    # selections of the last anchor (layer 2) vs the reference's
    P2 = np.stack([orc.dense_row(Q[2, h, -1], K[2, h // 4], V[2, h // 4])[0] for h in range(8)])
    for g in range(2):
        pooled = P2[g * 4:(g + 1) * 4][:, None, :].mean(axis=(0, 1), dtype=np.float64)
        topk_swaps(dec.indices[0, g, :int(dec.counts[0, g])].cpu().numpy(), z["dec_sel"][2, g], pooled)


def test_decode_engine_llama_shapes_vs_oracle(cuda_ok):
    """Llama-3.1-8B heads (32Q/8KV), 3 layers (anchor0, reuse with a
    non-identity head map, anchor), 32K context, k = 2.5%, batch 2."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, B, Hq, Hkv, n = 3, 2, 32, 8, 32768
    rng = np.random.default_rng(11)
    hm = [3, 1, 0, 2, 7, 5, 6, 4]
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, hm)},
                      k_policy=KBudgetPolicy(0.025, 128))
    # heavy-tailed queries so that the selection is meaningful
    q = orc.bf16_round((rng.standard_normal((L, B, Hq, 128)) * 2.5).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    out = dec.step(_dev(q, torch.bfloat16), [_dev(K[l], torch.bfloat16) for l in range(L)],
                   [_dev(V[l], torch.bfloat16) for l in range(L)], n).cpu().numpy()
    for b in range(B):
        Y, _, _ = orc.decode_step(q[:, b], K[:, b], V[:, b], [0, 2], {1: hm}, 0.025, 128, want_mass=False)
        assert_outputs_close(out[:, b], Y)


def test_decode_engine_all_heads_pooled_vs_oracle(cuda_ok):
    """All-heads-pooled mode (runner.py:180-197) through the engine's step:
    one shared set per sequence from the mean of every kv head's pooled
    vector, used by every head of the anchors and the reuse layers; anchors
    [0, 2, 3] make layers 2-3 a group (its list slots in the side-stream
    schedule) followed by two reuse layers."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, KBudgetPolicy
    L, B, Hq, Hkv, n = 6, 2, 16, 4, 6000
    rng = np.random.default_rng(17)
    plan = AnchorPlan(AnchorPlanCore([0, 2, 3], 3, 0.0), mode="all_heads_pooled", k_policy=KBudgetPolicy(0.05, 64))
    q = orc.bf16_round((rng.standard_normal((L, B, Hq, 128)) * 2.5).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    Ks, Vs = [_dev(K[l], torch.bfloat16) for l in range(L)], [_dev(V[l], torch.bfloat16) for l in range(L)]
    assert dec._can_overlap([(0, L)], Ks, Vs)
    out = dec.step(_dev(q, torch.bfloat16), Ks, Vs, n).cpu().numpy()
    for b in range(B):
        Y, sels, _ = orc.decode_step(q[:, b], K[:, b], V[:, b], [0, 2, 3], {}, 0.05, 64, mode=orc.ALL_HEADS_POOLED,
                                     want_mass=False)
        assert_outputs_close(out[:, b], Y)
        # the last anchor's shared set (every kv head reads it)
        c = int(dec.counts[b, 0])
        got = dec.indices[b, 0, :c].cpu().numpy()
        assert np.array_equal(np.sort(got), np.sort(np.asarray(sels[3][0]))) or len(np.setxor1d(got, sels[3][0])) <= 2


@pytest.mark.parametrize("splits,anchors,L", [((), [0, 2], 3), ((1, 2), [0, 2], 3), ((3,), [0, 2, 3], 5),
                                              ((4,), [0, 2, 3], 5)])
def test_host_step_graph_appends_and_matches_step(cuda_ok, splits, anchors, L):
    """capture_host_step (pinned H2D + one-launch KV append + layer loop +
    D2H as one CUDA graph) equals appending by hand and running step(); the
    appended rows land bit-exactly at position n-1 of every layer.  With
    anchors [0, 2, 3] an output-copy boundary at 3 cuts the anchor group
    (single-stream schedule), one at 4 does not (side-stream schedule)."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    B, Hq, Hkv, n, n_cap = 2, 8, 2, 700, 768
    maps = {l: HeadMap(l, max(a for a in anchors if a <= l), [1, 0]) for l in range(L) if l not in anchors}
    plan = AnchorPlan(AnchorPlanCore(anchors, len(anchors), 0.0), head_maps=maps, k_policy=KBudgetPolicy(0.1, 16))
    g = torch.Generator(device="cuda").manual_seed(5)
    Ks = [torch.randn(B, Hkv, n_cap, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    Vs = [torch.randn(B, Hkv, n_cap, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    q_host = torch.randn(L, B, Hq, 128).to(torch.bfloat16).pin_memory()
    kv_host = torch.randn(L, 2, B, Hkv, 128).to(torch.bfloat16).pin_memory()
    out_host = torch.zeros(L, B, Hq, 128).pin_memory()
    Kr = [x.clone() for x in Ks]
    Vr = [x.clone() for x in Vs]
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n_cap)
    dec.D2H_SPLITS = splits                        # one output copy, or one per layer
    q = torch.empty(L, B, Hq, 128, dtype=torch.bfloat16, device="cuda")
    bounds = sorted({0, 1, L} | {e for e in splits if 0 < e < L})
    assert dec._can_overlap(list(zip(bounds[:-1], bounds[1:])), Ks, Vs) == (splits != (3,))
    graph = dec.capture_host_step(q_host, kv_host, out_host, q, Ks, Vs, n)
    out_host.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(Ks[l][:, :, n - 1].cpu(), kv_host[l, 0]) and torch.equal(Vs[l][:, :, n - 1].cpu(), kv_host[l, 1])
        assert torch.equal(Ks[l][:, :, :n - 1], Kr[l][:, :, :n - 1])
        assert torch.equal(Ks[l][:, :, n:], Kr[l][:, :, n:])
        Kr[l][:, :, n - 1] = kv_host[l, 0].cuda()
        Vr[l][:, :, n - 1] = kv_host[l, 1].cuda()
    ref = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n_cap)
    want = ref.step(q_host.cuda(), Kr, Vr, n).cpu()
    assert torch.equal(out_host, want)


def test_multi_layer_launches_equal_per_layer(cuda_ok):
    """Consecutive reuse layers run as ONE multi-layer launch in step(), a
    group of consecutive anchors as one score launch + one select + one
    sparse launch over per-layer lists, and every dense layer as one launch
    in dense_step(); each layer's result (and the lists the reuse layers
    read) is bit-identical to launching it alone (the dense baseline: within
    split-K merge rounding)."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, B, Hq, Hkv, n = 8, 3, 16, 4, 5000
    maps = {1: HeadMap(1, 0, [3, 2, 1, 0]), 5: HeadMap(5, 4, [1, 0, 3, 2]), 6: HeadMap(6, 4, [0, 0, 1, 1]),
            7: HeadMap(7, 4, [2, 3, 0, 1])}
    plan = AnchorPlan(AnchorPlanCore([0, 2, 3, 4], 4, 0.0), head_maps=maps, k_policy=KBudgetPolicy(0.1, 64))
    _check_multi_layer(plan, L, B, Hq, Hkv, n)
    assert engine.KascadeDecoder(plan, L, B, Hq, Hkv, n).launches_per_step() == 3 + 1 + 4
    # a single anchor whose sparse pass shares a launch with the reuse run behind it
    maps1 = {1: HeadMap(1, 0, [3, 2, 1, 0]), 2: HeadMap(2, 0, [0, 0, 1, 1]), 4: HeadMap(4, 3, [1, 0, 3, 2]),
             5: HeadMap(5, 3, [2, 3, 0, 1]), 6: HeadMap(6, 3, [3, 3, 3, 3])}
    plan1 = AnchorPlan(AnchorPlanCore([0, 3, 7], 3, 0.0), head_maps=maps1, k_policy=KBudgetPolicy(0.1, 64))
    _check_multi_layer(plan1, L, B, Hq, Hkv, n)
    assert engine.KascadeDecoder(plan1, L, B, Hq, Hkv, n).launches_per_step() == 3 + 1 + 4 + 4


def _check_multi_layer(plan, L, B, Hq, Hkv, n):
    from paper_2512_16391_b200 import engine
    g = torch.Generator(device="cuda").manual_seed(3)
    Ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    Vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    q = (torch.randn(L, B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    assert dec._can_overlap([(0, L)], Ks, Vs)       # step() runs the selections on the side stream
    fused = dec.step(q, Ks, Vs, n).clone()
    lists = (dec.indices.clone(), dec.counts.clone())
    # the single-stream schedule of the same launches
    dec._run_range(0, L, q, Ks, Vs, n)
    assert torch.equal(dec.out, fused)
    assert torch.equal(dec.indices, lists[0]) and torch.equal(dec.counts, lists[1])
    for l in range(L):
        dec._layer(l, q, Ks, Vs, n)
    assert torch.equal(dec.out, fused)
    assert torch.equal(dec.indices, lists[0]) and torch.equal(dec.counts, lists[1])
    dfused = dec.dense_step(q, Ks, Vs, n).clone()
    for l in range(L):
        dec._dense_layer(l, q, Ks, Vs, n)
    # the all-layer dense launch cuts each layer into fewer split-K ranges than
    # a single-layer launch (decode_tc.cu kWavesMultiDense): merge rounding only
    torch.testing.assert_close(dec.out, dfused, rtol=1e-5, atol=1e-6)
    # and through a CUDA graph
    graph = dec.capture(q, Ks, Vs, n)
    dec.out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(dec.out, fused)
