"""Host-side logic of the decode executor (CPU, no kernels): layer kinds,
anchor groups and reuse runs, launch counts, when the overlapped
(side-stream) schedule applies, the head-map table that lets one launch
address an anchor group's list slots, and which lists each reuse run reads
(runner.py:228-297's layer loop, restructured; engine.py)."""
import pytest
import torch

from paper_2512_16391_b200 import engine
from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy, POOL_PRE


def _plan(anchors, L, Hkv=4, **kw):
    maps = {l: HeadMap(l, max(a for a in anchors if a <= l), [(h + l) % Hkv for h in range(Hkv)])
            for l in range(L) if l not in anchors}
    return AnchorPlan(AnchorPlanCore(anchors, len(anchors), 0.0), head_maps=maps, k_policy=KBudgetPolicy(0.1, 64),
                      **kw)


def _caches(L, B=3, Hkv=4, n=256):
    return [torch.empty(B, Hkv, n, 128, dtype=torch.bfloat16) for _ in range(L)]


@pytest.mark.parametrize("anchors,L,groups,launches", [
    ([0, 2, 3, 4], 8, [(2, 5)], 3 + 1 + 4),          # anchor 0, reuse 1, group 2-4 + reuse 5-7
    ([0, 3, 7], 8, [(3, 4), (7, 8)], 3 + 1 + 4 + 4),  # a lone last anchor keeps its own sparse launch
    ([0, 2, 8, 13, 14], 32, [(2, 3), (8, 9), (13, 15)], 3 + 1 + 4 + 4 + 4),   # the bench's Llama plan
    ([0], 4, [], 3 + 1),
])
def test_groups_and_launch_counts(anchors, L, groups, launches):
    dec = engine.KascadeDecoder(_plan(anchors, L), L, 3, 16, 4, 256, device="cpu")
    assert dec.groups == groups
    assert dec.launches_per_step() == launches
    assert dec.launches_per_step(dense=True) == 1
    for gl, ge in groups:
        b = dec.group_bufs[gl]
        assert b["end"] == ge and b["idx"].shape[0] == ge - gl
    if groups:     # the last group's lists are the executor's public lists
        last = dec.group_bufs[groups[-1][0]]
        assert last["idx"].data_ptr() == dec.indices.data_ptr()
        assert dec.idx0.data_ptr() != dec.indices.data_ptr()


def test_overlap_decision():
    L = 8
    dec = engine.KascadeDecoder(_plan([0, 2, 3, 4], L), L, 3, 16, 4, 256, device="cpu")
    Ks = _caches(L)
    assert dec._can_overlap([(0, L)], Ks, Ks)
    assert dec._can_overlap([(0, 1), (1, 5), (5, 8)], Ks, Ks)        # boundaries around the group
    assert not dec._can_overlap([(0, 1), (1, 3), (3, 8)], Ks, Ks)    # a boundary inside group 2-4
    mixed = Ks[:7] + [torch.empty(3, 4, 512, 128, dtype=torch.bfloat16)]
    assert not dec._can_overlap([(0, L)], mixed, mixed)             # one launch needs one cache layout
    dec.seq_lens = torch.zeros(3, dtype=torch.int32)
    assert not dec._can_overlap([(0, L)], Ks, Ks)                   # ragged batches run per layer
    pre = engine.KascadeDecoder(_plan([0, 2, 3, 4], L, pooling=POOL_PRE), L, 3, 16, 4, 256, device="cpu")
    assert pre.groups == [] and not pre._can_overlap([(0, L)], Ks, Ks)


def test_fused_map_table_addresses_group_slots():
    """Anchor gl + i of an m-anchor group reads list slot m - 1 - i: map
    entry s * B * Hsrc + h; the reuse layers behind it read slot 0 through
    their own maps."""
    L, B, Hkv = 8, 3, 4
    dec = engine.KascadeDecoder(_plan([0, 2, 3, 4], L), L, B, 16, Hkv, 256, device="cpu")
    t = dec._fused_maps(2, 5, 8)
    assert t.shape == (6, Hkv)
    for i in range(3):
        assert t[i].tolist() == [(2 - i) * B * Hkv + h for h in range(Hkv)]
    for r, l in enumerate(range(5, 8)):
        assert t[3 + r].tolist() == dec.plan.head_maps[l].map


def test_reuse_runs_read_the_latest_anchor():
    L = 32
    dec = engine.KascadeDecoder(_plan([0, 2, 8, 13, 14], L), L, 3, 16, 4, 256, device="cpu")
    assert dec._lists_before(1)[0] is dec.idx0
    g2 = dec.group_bufs[2]["idx"][0]
    assert dec._lists_before(5)[0].data_ptr() == g2.data_ptr()
    assert dec._lists_before(20)[0].data_ptr() == dec.indices.data_ptr()   # the last group's slot 0
