"""Freeze the reference cost model's outputs (costmodel.py) so the B200
restatement (paper_2512_16391_b200/costmodel.py) is pinned to them.  Runs in
the dev container only (imports /root/reference/pkg/src read-only).

    python tests/golden/make_costmodel_golden.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from kascade import costmodel as cm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rep(r):
    return {"kascade_time": r.kascade_time, "speedup": r.speedup, "baseline_time": r.baseline_time,
            "per_kind": r.per_kind, "valid": r.valid}


def main():
    out = {"rows": [], "fits": {}, "presets": {}, "weighted": [], "predict": []}
    for r in cm.PUBLISHED_BENCH:
        out["rows"].append({"phase": r.phase, "seq_len": r.seq_len, "topk_pct": r.topk_pct, "tl_ms": r.tl_ms,
                            "anchor0_ms": r.anchor0_ms, "anchor_ms": r.anchor_ms, "reuse_ms": r.reuse_ms,
                            "anchor0_ratio": r.anchor0_ratio, "anchor_ratio": r.anchor_ratio,
                            "reuse_ratio": r.reuse_ratio})
        out["presets"][r.preset_name] = rep(cm.report_from_preset(r.preset_name))
    for ph in ("decode", "prefill"):
        f = cm.fit_ratios(ph)
        out["fits"][ph] = {"c_gather": f.c_gather, "c_select": f.c_select, "c_pass1": f.c_pass1,
                           "max_residual": f.max_residual}
    for args in [("decode", 32, 5, 0.1, 131072, 2.0, (1.2, 0.9, 0.12)), ("prefill", 80, 12, 0.2, 8192, 1.0,
                                                                           (1.8, 1.6, 0.3))]:
        ph, L, M, fr, n, base, (a0, a, r) = args
        p = cm.CostParams(phase=ph, num_layers=L, num_anchors=M, topk_fraction=fr, seq_len=n,
                          baseline_layer_time=base)
        out["weighted"].append({"args": [ph, L, M, fr, n, base, [a0, a, r]],
                                "report": rep(cm.weighted_pipeline_time(p, {"anchor0": a0, "anchor": a,
                                                                            "reuse": r}))})
    for args in [("decode", 0.1, 131072, 32, 5, 1.0), ("prefill", 0.25, 8192, 36, 5, 3.0)]:
        out["predict"].append({"args": list(args), "report": rep(cm.predict_report(*args))})
    json.dump(out, open(os.path.join(HERE, "costmodel_ref.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
