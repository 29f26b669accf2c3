"""Pre-softmax pooling at engine scale (_pre_pooled, runner.py:155-161; the
comparison mode of SPEC.md:370): q_bar of each (kv head, tile), softmax of
K q_bar / sqrt(d), exact Top-k -- kscd_select_pre on the device against the
oracle's pooled_pre / prefill_tile_select / decode_step(pooling='pre') on the
same bf16 inputs, from reference-test sizes up to the bench shapes, in both
plan modes, and through both executors.  Needs a B200."""

import numpy as np
import pytest

from oracle import kascade_oracle as orc
from parity import assert_outputs_close, topk_swaps

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)


def _policy(f, kmin):
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    return KBudgetPolicy(f, kmin)


@pytest.mark.parametrize("Hq,Hkv,N,f,kmin", [(8, 2, 1000, 0.1, 16), (4, 4, 128, 0.25, 8), (32, 8, 4096, 0.1, 128),
                                             (8, 1, 300, 0.5, 1)])
def test_select_prefill_pre_matches_oracle(cuda_ok, Hq, Hkv, N, f, kmin):
    from paper_2512_16391_b200 import ops
    rng = np.random.default_rng(N + Hq)
    Q = orc.bf16_round((rng.standard_normal((Hq, N, 128)) * 3).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((Hkv, N, 128)).astype(np.float32))
    idx, cnt = ops.select_prefill_pre(_bf(Q), _bf(K), _policy(f, kmin))
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    G, T = Hq // Hkv, (N + 127) // 128
    swaps = 0
    for g in range(Hkv):
        for t in range(T):
            s, e = 128 * t, min(N, 128 * t + 128)
            sel, pooled = orc.prefill_tile_select(Q, K, g, G, s, e, f, kmin, pooling=orc.PRE)
            assert int(cnt[g, t]) == sel.size
            swaps += topk_swaps(idx[g, t, :sel.size], sel, pooled)
    assert swaps <= max(2, Hkv * T // 50), swaps


def test_select_prefill_pre_all_heads(cuda_ok):
    """all-heads-pooled: the kv heads' pre-softmax vectors averaged, one set
    per tile (runner.py:180-197)."""
    from paper_2512_16391_b200 import ops
    Hq, Hkv, N = 8, 4, 700
    rng = np.random.default_rng(3)
    Q = orc.bf16_round((rng.standard_normal((Hq, N, 128)) * 3).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((Hkv, N, 128)).astype(np.float32))
    idx, cnt = ops.select_prefill_pre(_bf(Q), _bf(K), _policy(0.2, 32), all_heads=True)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    assert idx.shape[0] == 1
    for t in range((N + 127) // 128):
        s, e = 128 * t, min(N, 128 * t + 128)
        pooled = np.mean([orc.pooled_pre(Q, K, g, 2, s, e) for g in range(Hkv)], axis=0)
        ref = orc.topk_sorted(pooled, orc.k_budget(0.2, 32, e))
        topk_swaps(idx[0, t, :cnt[0, t]], ref, pooled)


@pytest.mark.parametrize("B,Hq,Hkv,n", [(3, 8, 2, 5000), (2, 32, 8, 70000), (1, 4, 1, 100)])
def test_select_decode_pre_matches_oracle(cuda_ok, B, Hq, Hkv, n):
    from paper_2512_16391_b200 import ops
    rng = np.random.default_rng(n)
    q = orc.bf16_round((rng.standard_normal((B, Hq, 128)) * 2).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((B, Hkv, n + 3, 128)).astype(np.float32))
    idx, cnt = ops.select_decode_pre(_bf(q), _bf(K), n, _policy(0.1, 64))
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    G = Hq // Hkv
    k = orc.k_budget(0.1, 64, n)
    for b in range(B):
        for g in range(Hkv):
            qbar = q[b, g * G:(g + 1) * G].mean(axis=0, dtype=np.float64)
            pooled = orc.softmax_vec((K[b, g, :n].astype(np.float64) @ qbar) / np.sqrt(128)).astype(np.float64)
            ref = orc.topk_sorted(pooled, k)
            assert int(cnt[b, g]) == k
            topk_swaps(idx[b, g, :k], ref, pooled)


def test_select_decode_pre_ragged(cuda_ok):
    from paper_2512_16391_b200 import ops
    B, Hq, Hkv, n = 3, 8, 2, 3000
    rng = np.random.default_rng(9)
    q = orc.bf16_round((rng.standard_normal((B, Hq, 128)) * 2).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((B, Hkv, n, 128)).astype(np.float32))
    lens = np.array([3000, 1234, 200], np.int32)
    idx, cnt = ops.select_decode_pre(_bf(q), _bf(K), n, _policy(0.1, 64),
                                     seq_lens=torch.from_numpy(lens).cuda())
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(B):
        nb = int(lens[b])
        k = orc.k_budget(0.1, 64, nb)
        for g in range(Hkv):
            qbar = q[b, g * 4:(g + 1) * 4].mean(axis=0, dtype=np.float64)
            pooled = orc.softmax_vec((K[b, g, :nb].astype(np.float64) @ qbar) / np.sqrt(128)).astype(np.float64)
            assert int(cnt[b, g]) == k
            topk_swaps(idx[b, g, :k], orc.topk_sorted(pooled, k), pooled)


def test_decode_engine_pre_pooling_128k_b8(cuda_ok):
    """The Llama plan with pre-softmax pooling through KascadeDecoder at the
    headline shape (128K, batch 8, k = 10 %), every sequence against
    orc.decode_step(pooling='pre')."""
    from test_scale_gpu import _decode_case, _plan
    plan = _plan("llama8b", 0.1)
    plan.pooling = "pre"
    _decode_case(plan, 32, 8, 32, 8, 131072, 41000, check_seqs=range(8))


def test_prefill_engine_pre_pooling_64k(cuda_ok):
    """KascadePrefill with pre-softmax pooling at 64K (Llama heads), sampled
    tiles against prefill_tile_select(pooling='pre') / sparse_tile."""
    from paper_2512_16391_b200 import engine
    from test_scale_gpu import _plan, _sample_tiles
    plan = _plan("llama8b", 0.1, layers=3)
    plan.pooling = "pre"
    N, Hq, Hkv, L = 65536, 32, 8, 3
    G = Hq // Hkv
    gen = torch.Generator(device="cuda")
    qs, ks, vs = [], [], []
    for l in range(L):
        gen.manual_seed(42000 + l)
        qs.append((torch.randn(Hq, N, 128, device="cuda", generator=gen) * 2).to(torch.bfloat16))
        ks.append(torch.randn(Hkv, N, 128, device="cuda", generator=gen, dtype=torch.bfloat16))
        vs.append(torch.randn(Hkv, N, 128, device="cuda", generator=gen, dtype=torch.bfloat16))
    eng = engine.KascadePrefill(plan, L, Hq, Hkv, N)
    eng.forward(qs, ks, vs, stop_after=0)
    sets0 = (eng.indices.cpu().numpy(), eng.counts.cpu().numpy())
    out = eng.forward(qs, ks, vs)
    sets2 = (eng.indices.cpu().numpy(), eng.counts.cpu().numpy())
    host = [(qs[l].float().cpu().numpy(), ks[l].float().cpu().numpy(), vs[l].float().cpu().numpy()) for l in range(L)]
    hm = plan.head_maps[1].map
    swaps = 0
    for t in _sample_tiles(N // 128):
        s, e = 128 * t, 128 * t + 128
        ref = {}
        for layer, (idx, cnt) in ((0, sets0), (2, sets2)):
            for g in range(Hkv):
                sel, pooled = orc.prefill_tile_select(host[layer][0], host[layer][1], g, G, s, e, 0.1, 128,
                                                      pooling=orc.PRE)
                swaps += topk_swaps(idx[g, t, :cnt[g, t]], sel, pooled)
                ref[(layer, g)] = sel
        # outputs on identical index sets (the engine's; a documented near-tie
        # swap of the pre-softmax ranking can move a key that one row weighs heavily)
        for g in range(Hkv):
            e1 = sets0[0][hm[g], t, :sets0[1][hm[g], t]].astype(np.int64)
            e2 = sets2[0][g, t, :sets2[1][g, t]].astype(np.int64)
            y1, _, _ = orc.sparse_tile(*host[1], g, G, s, e, e1)
            y2, _, _ = orc.sparse_tile(*host[2], g, G, s, e, e2)
            assert_outputs_close(out[1, g * G:(g + 1) * G, s:e].float().cpu().numpy(), y1)
            assert_outputs_close(out[2, g * G:(g + 1) * G, s:e].float().cpu().numpy(), y2)
    print(f"pre-softmax prefill 64K: near-tie swaps {swaps}")
    assert swaps <= 8
