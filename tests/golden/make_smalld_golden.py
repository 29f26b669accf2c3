"""Freeze golden vectors for head_dim < 128 from the REFERENCE itself.

The reference's own tests run traces with d in {4, 8, 16, 32, 64}; the engine
serves them by zero-padding rows to 128 (include/kascade_b200.h,
Conventions).  Run in the dev container (the only place /root/reference
exists):

    python tests/golden/make_smalld_golden.py

writes ``smalld.npz``: for d = 16 and 64 a dense layer (P, Y), a full
run_kascade prefill with remapped head maps and tile 16, the pre-softmax
pooling variant, and a decode-phase run -- all from the reference's public
functions on seeded bf16-representable inputs.
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import bf16_trace_random, orc, ref, trace_of  # noqa: E402


def main():
    out = {}
    for d in (16, 64):
        Q, K, V = bf16_trace_random(100 + d, 3, 4, 2, d, 48)
        t = trace_of(Q, K, V, pid=f"smalld{d}")
        P, Y = ref.dense_attention(t, 0)
        anchors = [0, 1]
        maps = {2: ref.HeadMap(reuse_layer=2, anchor_layer=1, map=[1, 0])}
        core = ref.AnchorPlanCore(anchors=anchors, budget=2, objective_value=0.0)
        pol = ref.KBudgetPolicy(fraction=0.25, k_min=4)
        plan = ref.AnchorPlan(core=core, head_maps=maps, k_policy=pol, tile_size=16)
        outs, rep = ref.run_kascade(t, plan)
        plan_pre = ref.AnchorPlan(core=core, head_maps=maps, pooling="pre", k_policy=pol, tile_size=16)
        outs_pre, _ = ref.run_kascade(t, plan_pre)
        outs_dec, rep_dec = ref.run_kascade(t, plan, phase="decode")
        out.update({f"Q{d}": orc.bf16_bits(Q), f"K{d}": orc.bf16_bits(K), f"V{d}": orc.bf16_bits(V),
                    f"P{d}": P, f"Y{d}": Y, f"outs{d}": outs, f"outs_pre{d}": outs_pre, f"outs_dec{d}": outs_dec,
                    f"mass{d}": np.array([r.mass_recovered_mean for r in rep.per_layer]),
                    f"mass_dec{d}": np.array([r.mass_recovered_mean for r in rep_dec.per_layer])})
    np.savez_compressed(os.path.join(HERE, "smalld.npz"), **out)
    print("wrote smalld.npz")


if __name__ == "__main__":
    main()
