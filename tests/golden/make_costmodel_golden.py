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
    # the reference CLI's `cost` output (cli.py:236-320), stdout verbatim
    import contextlib
    import io
    from kascade.cli import main as ref_main
    out["cli"] = []
    for argv in (["cost", "--preset", "table3-decode-131072-k10", "--preset", "table3-prefill-8192-k30"],
                 ["cost", "--preset", "table3-prefill-131072-k20", "--csv"],
                 ["cost", "--predict", "--phase", "prefill", "--csv"],
                 ["cost", "--predict", "--fraction", "0.25", "--seq-len", "8192"],
                 ["cost", "--ratios", "1.2,0.9,0.1", "--baseline-time", "2", "--layers", "40", "--anchors", "6"],
                 ["cost", "--list-presets"],
                 ["cost"]):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = ref_main(list(argv))
        out["cli"].append({"argv": argv, "rc": rc, "stdout": buf.getvalue()})
    json.dump(out, open(os.path.join(HERE, "costmodel_ref.json"), "w"), indent=1)
    # the paper's Table 3 rows (costmodel.py:64-112) as package data, so the
    # reference-named presets resolve to the same numbers
    fields = ["phase", "seq_len", "topk_pct", "fa3_ms", "tl_ms", "anchor0_ms", "anchor0_ratio", "anchor_ms",
              "anchor_ratio", "reuse_ms", "reuse_ratio", "kascade_ms", "speedup_fa3", "speedup_tl"]
    table = {"source": "Kascade paper Table 3 (H100 kernel microbenchmarks), as bundled by the reference "
                       "(costmodel.py:64-112); frozen by tests/golden/make_costmodel_golden.py",
             "fields": fields, "rows": [[getattr(r, f) for f in fields] for r in cm.PUBLISHED_BENCH]}
    with open(os.path.join(HERE, "..", "..", "paper_2512_16391_b200", "published_table3.json"), "w") as f:
        head = json.dumps({k: v for k, v in table.items() if k != "rows"}, indent=1)[:-2]
        rows = ",\n  ".join(json.dumps(r) for r in table["rows"])
        f.write(f'{head},\n "rows": [\n  {rows}\n ]\n}}\n')


if __name__ == "__main__":
    main()
