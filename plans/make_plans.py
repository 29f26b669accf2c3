"""Build the anchor plans the bench uses, with the REFERENCE's own offline
planner (run in the dev container, where /root/reference is importable; the
JSON outputs are committed and read on the GPU box by host_types.read_plan).

- llama8b / qwen3_8b: published anchor sets with head maps from
  the reference's compute_head_maps (pipeline.py:31-73) on a small synthetic
  trace whose kv heads are permuted per layer, so the remaps are non-identity
  and the cross-head gather is exercised (SURVEY.md 8(d) "Plans").
- llama70b: no published anchor set -- the reference's full build_plan
  (pipeline.py:76-118: planning similarity, importance weighting, DP anchor
  selection, head maps) on an 80-layer synthetic trace, budget 12.

The synthetic traces use head_dim 64 and 512 tokens: the planner's outputs
depend on the layer / kv-head structure, not on the bench's head_dim or
context, and this keeps the O(L^2 Hkv^2) planning loop to about a minute.

    PYTHONPATH=/root/reference/pkg/src python plans/make_plans.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from kascade.pipeline import build_plan, compute_head_maps  # noqa: E402
from kascade.planner import AnchorPlanCore  # noqa: E402
from kascade.runner import AnchorPlan  # noqa: E402
from kascade.tiles import KBudgetPolicy  # noqa: E402
from kascade.traceio import SynthConfig, generate_synthetic, write_plan  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def permuted_trace(L, Hq, Hkv, seed):
    rng = np.random.default_rng(seed)
    perms = [list(range(Hkv))] + [rng.permutation(Hkv).tolist() for _ in range(L - 1)]
    return generate_synthetic(SynthConfig(num_layers=L, num_query_heads=Hq, num_kv_heads=Hkv, head_dim=64,
                                          seq_len=512, seed=seed, layer_correlation=0.9,
                                          head_permutations=perms, include_xy=True,
                                          prompt_id=f"plan-L{L}-seed{seed}"))


def fixed_anchor_plan(name, L, Hq, Hkv, anchors, seed):
    trace = permuted_trace(L, Hq, Hkv, seed)
    maps = compute_head_maps(trace, anchors)
    plan = AnchorPlan(core=AnchorPlanCore(anchors=list(anchors), budget=len(anchors), objective_value=0.0),
                      head_maps=maps, k_policy=KBudgetPolicy(0.1, 128))
    plan.validate(trace)
    write_plan(os.path.join(HERE, f"{name}.json"), plan)
    ident = sum(m.map == list(range(Hkv)) for m in maps.values())
    print(f"{name}: anchors {anchors}, {len(maps)} head maps ({ident} identity)")


def main():
    fixed_anchor_plan("llama8b", 32, 32, 8, [0, 2, 8, 13, 14], seed=8)
    fixed_anchor_plan("qwen3_8b", 36, 32, 8, [0, 2, 7, 14, 23], seed=3)
    trace = permuted_trace(80, 64, 8, seed=70)
    plan = build_plan(trace, budget=12, k_policy=KBudgetPolicy(0.1, 128))
    write_plan(os.path.join(HERE, "llama70b.json"), plan)
    print(f"llama70b: anchors {plan.anchors}, {len(plan.head_maps)} head maps")


if __name__ == "__main__":
    main()
