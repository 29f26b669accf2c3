"""Parity at the shapes the bench reports (VERDICT r1 "next round" #1).

The CUDA path runs at full size -- 128K context, Llama-3.1-8B heads, batch 8,
Top-k 10 % (k = 13,107), every layer of plans/llama8b.json with its
non-identity head maps; Qwen3-8B heads at batch 32; Llama-3.1-70B heads
(G = 8) and the 70B kv-head shard (1 KV + 8 Q heads); 64K / 128K prefill --
and is checked against the O(n) oracle drivers (oracle/kascade_oracle.py:
decode_step, prefill_tile_select, sparse_tile, restating attention.py:185-253
and runner.py:164-225) on the SAME bf16 inputs:

* every anchor's index lists: set-equal up to documented fp32 near-ties
  (tests/parity.py topk_swaps; the swap count is printed and bounded);
* head-remap routing: the reuse layers read the anchor lists through the
  plan's maps (bit-exact by construction; the outputs would differ otherwise);
* outputs: max-abs <= 2e-2 and mean-abs <= 1e-3 (north_star's bf16
  tolerance), rel-L2 printed.

Decode compares whole sequences (all layers); prefill samples 8 tiles per kv
head, tile 0 and the last tile included.  The K/V caches stay on the device:
the oracle reads them through lazy views (one head's rows, or the gathered
rows of a selection), so the host never holds a whole 137 GB KV set.
Needs a B200 (the 128K batch-8 test allocates ~140 GB)."""

import numpy as np
import pytest

from oracle import kascade_oracle as orc
from parity import assert_outputs_close, topk_swaps

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import os  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class DeviceKV:
    """Lazy fp32 view of one sequence's per-layer device caches for
    orc.decode_step: K[l, g] -> that head's first n rows, K[l, g, sel] -> the
    gathered rows (gathered on the device, so only they cross PCIe)."""

    def __init__(self, caches, b, n):
        self.caches, self.b, self.n = caches, b, n
        self.shape = (len(caches), caches[0].shape[1], n, caches[0].shape[3])
        self._memo = None

    def __getitem__(self, key):
        l, g = key[0], key[1]
        if len(key) == 2:
            if self._memo is None or self._memo[0] != (l, g):
                self._memo = ((l, g), self.caches[l][self.b, g, :self.n].float().cpu().numpy())
            return self._memo[1]
        sel = torch.from_numpy(np.ascontiguousarray(key[2], dtype=np.int64)).to(self.caches[l].device)
        return self.caches[l][self.b, g].index_select(0, sel).float().cpu().numpy()


def _plan(name, fraction, k_min=128, layers=None):
    """A committed plan (reference planner, non-identity maps), optionally
    cut to its first `layers` layers."""
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, KBudgetPolicy, read_plan
    p = read_plan(os.path.join(REPO, "plans", f"{name}.json"))
    if layers is not None:
        anchors = [a for a in p.anchors if a < layers]
        p = AnchorPlan(AnchorPlanCore(anchors, len(anchors), 0.0),
                       head_maps={l: m for l, m in p.head_maps.items() if l < layers})
    p.k_policy = KBudgetPolicy(fraction, k_min)
    return p


def _decode_case(plan, L, B, Hq, Hkv, n, seed, check_seqs, max_swaps_per_list=2):
    """Run the decode engine layer by layer (snapshotting every anchor's
    index lists) and check the listed sequences against orc.decode_step."""
    from paper_2512_16391_b200 import engine
    torch.cuda.empty_cache()
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    Ks, Vs = [], []
    for l in range(L):
        gen.manual_seed(seed + l)
        Ks.append(torch.randn(B, Hkv, n, 128, device=dev, dtype=torch.bfloat16, generator=gen))
        Vs.append(torch.randn(B, Hkv, n, 128, device=dev, dtype=torch.bfloat16, generator=gen))
    gen.manual_seed(seed + 999)
    q = (torch.randn(L, B, Hq, 128, device=dev, generator=gen) * 2.0).to(torch.bfloat16)
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n, device=dev)
    snaps = {}
    for l in range(L):
        dec._layer(l, q, Ks, Vs, n)
        if dec.kinds[l] != "reuse":
            snaps[l] = (dec.indices.cpu().numpy(), dec.counts.cpu().numpy())
    out = dec.out.cpu().numpy()
    # the same step as one CUDA graph replay gives the same outputs
    g = dec.capture(q, Ks, Vs, n)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dec.out.cpu().numpy(), out)
    qn = q.float().cpu().numpy()
    maps = {l: m.map for l, m in plan.head_maps.items()}
    k = orc.k_budget(plan.k_policy.fraction, plan.k_policy.k_min, n)
    worst, swaps = 0.0, 0
    for b in check_seqs:
        pooled = {}
        Y, sels, _ = orc.decode_step(qn[:, b], DeviceKV(Ks, b, n), DeviceKV(Vs, b, n), plan.anchors, maps,
                                     plan.k_policy.fraction, plan.k_policy.k_min, pooling=plan.pooling,
                                     want_mass=False, pooled_out=pooled)
        for l, (idx, cnt) in snaps.items():
            for gg in range(Hkv):
                assert int(cnt[b, gg]) == k, (l, b, gg, int(cnt[b, gg]), k)
                s = topk_swaps(idx[b, gg, :k], sels[l][gg], pooled[l][gg])
                assert s <= max_swaps_per_list, (l, b, gg, s)
                swaps += s
        mx, mean, rel = assert_outputs_close(out[:, b], Y, what=f"sequence {b}")
        worst = max(worst, mx)
        print(f"seq {b}: max-abs {mx:.2e} mean-abs {mean:.2e} rel-L2 {rel:.2e}")
    print(f"decode L={L} B={B} Hq={Hq} Hkv={Hkv} n={n} k={k}: {len(check_seqs)} sequences, "
          f"{len(snaps)} anchor layers, near-tie swaps {swaps}, worst max-abs {worst:.2e}")
    del Ks, Vs, q, dec, g
    torch.cuda.empty_cache()
    return swaps


def test_decode_llama8b_128k_b8_all_layers(cuda_ok):
    """The headline: Llama-3.1-8B heads, 128K, batch 8, k = 10 %, the
    32-layer plan (anchors [0,2,8,13,14], 27 remapped reuse layers), every
    sequence against the oracle."""
    plan = _plan("llama8b", 0.1)
    _decode_case(plan, 32, 8, 32, 8, 131072, 21000, check_seqs=range(8))


def test_decode_llama8b_32k_b8_k2p5_all_layers(cuda_ok):
    """BASELINE configs[1]: 32K, batch 8, Top-k 2.5 % (k = 819)."""
    plan = _plan("llama8b", 0.025)
    _decode_case(plan, 32, 8, 32, 8, 32768, 22000, check_seqs=range(8))


def test_decode_qwen3_128k_b32_subset(cuda_ok):
    """BASELINE configs[3] shapes: Qwen3-8B heads, 128K, batch 32 (the split
    counts and 256-row Top-k of the bench), first 3 layers of the Qwen3 plan
    (anchor0, remapped reuse, anchor); sequences 0, 13, 31 checked."""
    plan = _plan("qwen3_8b", 0.1, layers=3)
    _decode_case(plan, 3, 32, 32, 8, 131072, 23000, check_seqs=(0, 13, 31))


def test_decode_llama70b_heads_128k(cuda_ok):
    """Llama-3.1-70B heads (64 Q / 8 KV, G = 8) at 128K: first 4 layers of
    the 70B plan (anchor0, remapped reuse, anchors 2 and 3), batch 4."""
    plan = _plan("llama70b", 0.1, layers=4)
    _decode_case(plan, 4, 4, 64, 8, 131072, 24000, check_seqs=(0, 3))


def test_decode_llama70b_kv_head_shard_128k_b8(cuda_ok):
    """One rank of the 8-way kv-head-sharded 70B decode (bench configs[4]):
    1 KV + 8 Q heads, batch 8, the low-parallelism 8-row case; 16 layers of
    the 70B plan's anchor pattern with the shard's own head (map [0])."""
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    p70 = _plan("llama70b", 0.1)
    L = 16
    anchors = [a for a in p70.anchors if a < L]
    plan = AnchorPlan(AnchorPlanCore(anchors, len(anchors), 0.0),
                      head_maps={l: HeadMap(l, m.anchor_layer, [0]) for l, m in p70.head_maps.items() if l < L},
                      k_policy=KBudgetPolicy(0.1, 128))
    _decode_case(plan, L, 8, 8, 1, 131072, 25000, check_seqs=range(8))


# ------------------------------------------------------------------ prefill
def _sample_tiles(T, per=8):
    return sorted({0, T - 1} | {int(x) for x in np.linspace(1, T - 2, per - 2)})


def _prefill_case(N, Hq, Hkv, plan_layers, seed, tiles_per_head=8):
    """3 layers (anchor0, remapped reuse, anchor) through KascadePrefill;
    sampled tiles of every kv head against prefill_tile_select / sparse_tile
    / the dense tile rows."""
    from paper_2512_16391_b200 import engine
    torch.cuda.empty_cache()
    plan = plan_layers
    L = 3
    G = Hq // Hkv
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    qs, ks, vs = [], [], []
    for l in range(L):
        gen.manual_seed(seed + l)
        qs.append(torch.randn(Hq, N, 128, device=dev, generator=gen, dtype=torch.bfloat16))
        ks.append(torch.randn(Hkv, N, 128, device=dev, generator=gen, dtype=torch.bfloat16))
        vs.append(torch.randn(Hkv, N, 128, device=dev, generator=gen, dtype=torch.bfloat16))
    eng = engine.KascadePrefill(plan, L, Hq, Hkv, N, device=dev)
    eng.forward(qs, ks, vs, stop_after=0)
    sets = {0: (eng.indices.cpu().numpy(), eng.counts.cpu().numpy())}
    out = eng.forward(qs, ks, vs)
    sets[2] = (eng.indices.cpu().numpy(), eng.counts.cpu().numpy())
    hm = plan.head_maps[1].map
    T = (N + 127) // 128
    host = [(qs[l].float().cpu().numpy(), ks[l].float().cpu().numpy(), vs[l].float().cpu().numpy())
            for l in range(L)]
    pol = plan.k_policy
    swaps, worst = 0, 0.0
    tiles = _sample_tiles(T, tiles_per_head)
    for t in tiles:
        s, e = 128 * t, min(N, 128 * t + 128)
        ref_sets = {}
        for layer in (0, 2):
            Ql, Kl, _ = host[layer]
            idx, cnt = sets[layer]
            for g in range(Hkv):
                sel, pooled = orc.prefill_tile_select(Ql, Kl, g, G, s, e, pol.fraction, pol.k_min)
                assert int(cnt[g, t]) == sel.size, (layer, g, t)
                swaps += topk_swaps(idx[g, t, :sel.size], sel, pooled)
                ref_sets[(layer, g)] = sel
        for g in range(Hkv):
            heads = slice(g * G, (g + 1) * G)
            # layer 0: dense rows of the tile
            Ql, Kl, Vl = host[0]
            Pt = orc.prefill_tile_rows(Ql, Kl, g, G, s, e)
            y0 = np.stack([Pt[j] @ Vl[g] for j in range(G)])
            # layer 1 (reuse): the anchor-0 set of head_map[g]
            y1, _, _ = orc.sparse_tile(*host[1], g, G, s, e, ref_sets[(0, hm[g])])
            # layer 2 (anchor): its own fresh set
            y2, _, _ = orc.sparse_tile(*host[2], g, G, s, e, ref_sets[(2, g)])
            for layer, y in ((0, y0), (1, y1), (2, y2)):
                mx, _, _ = assert_outputs_close(out[layer, heads, s:e].float().cpu().numpy(), y,
                                                what=f"layer {layer} kv head {g} tile {t}")
                worst = max(worst, mx)
    n_sets = 2 * Hkv * len(tiles)
    print(f"prefill N={N} Hq={Hq} Hkv={Hkv}: tiles {tiles} x {Hkv} kv heads, {n_sets} anchor sets, "
          f"near-tie swaps {swaps}, worst max-abs {worst:.2e}")
    assert swaps <= n_sets, swaps
    del qs, ks, vs, eng
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N", [65536, 131072])
def test_prefill_llama8b_sampled_tiles(cuda_ok, N):
    """BASELINE configs[2] (64K) and the 128K headline prefill: Llama-8B heads,
    k = 10 % per tile (k_i up to 13,107 of 128K), the Llama plan's layer-1
    head map."""
    _prefill_case(N, 32, 8, _plan("llama8b", 0.1, layers=3), 31000 + N // 1024)


def test_prefill_llama70b_shard_128k(cuda_ok):
    """One rank of the kv-head-sharded 70B prefill: 1 KV + 8 Q heads (G = 8),
    128K, 3 layers."""
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, [0])},
                      k_policy=KBudgetPolicy(0.1, 128))
    _prefill_case(131072, 8, 1, plan, 32000)
