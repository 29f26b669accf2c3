"""Golden cases from MODEL traces: KSCD files written
by the reference's own exporter (pkg/exporter, kscd_exporter.export:
capture.py:146-198) from its reference transformer (reference.py: GQA
attention with RoPE and RMSNorm, random-init weights, byte tokenizer) on
English prompts, plus the reference planner's plan for them
(pipeline.build_plan, pipeline.py:76-120) and the reference's `run_kascade`
reports (runner.py:228-318) for both phases and both plan modes.

Run in the dev container (the reference tree does not travel to the GPU box):

    python tests/golden/make_exporter_golden.py

Writes tests/golden/exporter/*.kscd, *_plan.json and exporter_cases.json.
tests/test_exporter_traces_gpu.py runs the B200 engine's `run` CLI on the
same files and compares its reports with these."""

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "exporter", "src")]

from kascade import pipeline, runner, tiles, traceio  # noqa: E402
from kscd_exporter import ExportConfig, export  # noqa: E402

PROMPT = (
    "The anchor layers of a long-context model compute exact attention, pick the keys that matter most for every "
    "tile of queries, and hand those positions to the layers that follow, which then attend sparsely. Whether the "
    "shortcut holds depends on how similar the attention of neighbouring layers really is, which is why the plan "
    "is calibrated offline on traces captured from the model itself rather than on random data. Heads may change "
    "roles between layers, so each reuse layer carries a head map that tells it whose selection to borrow. "
    "This paragraph is long enough to give the byte-level tokenizer a few hundred positions to work with."
)

def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


CASES = [
    # name, tiny model spec, max tokens, plan (tile, budget, k, fraction, k_min)
    ("exp_d64", "tiny:layers=4,kv_heads=2,q_heads=8,dim=64,seed=11,max_seq=512", 384, (128, 2, 32, 0.1, 32)),
    ("exp_d128", "tiny:layers=3,kv_heads=2,q_heads=4,dim=128,seed=5,max_seq=512", 384, (32, 2, 16, 0.25, 16)),
]


def main():
    out_dir = os.path.join(HERE, "exporter")
    os.makedirs(out_dir, exist_ok=True)
    cases = {}
    with tempfile.TemporaryDirectory() as tmp:
        pf = os.path.join(tmp, "prompts.txt")
        with open(pf, "w") as f:
            f.write(PROMPT + "\n")
        for name, spec, max_tokens, (tile, budget, k, frac, kmin) in CASES:
            paths = export(ExportConfig(model=spec, prompt_file=pf, output_dir=os.path.join(tmp, name),
                                        max_tokens=max_tokens, capture_xy=False))
            # the engine computes in bf16: both sides get the same
            # bf16-representable inputs (SURVEY.md 8(c) parity definition)
            t = traceio.read_trace(paths[0])
            t.Q, t.K, t.V = bf16_round(t.Q), bf16_round(t.K), bf16_round(t.V)
            trace_file = os.path.join(out_dir, f"{name}.kscd")
            traceio.write_trace(trace_file, t)
            data = open(trace_file, "rb").read()
            trace = traceio.read_trace(trace_file)
            plan = pipeline.build_plan([trace], budget=budget, k=k, tile_size=tile,
                                       k_policy=tiles.KBudgetPolicy(fraction=frac, k_min=kmin))
            plan_file = os.path.join(out_dir, f"{name}_plan.json")
            traceio.write_plan(plan_file, plan)
            runs = {}
            for phase in ("prefill", "decode"):
                for mode in ("remapped", "all_heads_pooled"):
                    p = traceio.read_plan(plan_file)
                    p.mode = mode
                    _, report = runner.run_kascade(trace, p, phase=phase)
                    rf = os.path.join(tmp, "r.json")
                    traceio.write_report(rf, report)
                    runs[f"{phase}_{mode}"] = json.load(open(rf))
            cases[name] = {
                "model": spec, "tokens": trace.seq_len, "layers": trace.num_layers,
                "q_heads": trace.num_query_heads, "kv_heads": trace.num_kv_heads, "head_dim": trace.head_dim,
                "trace": f"exporter/{name}.kscd", "sha256": hashlib.sha256(data).hexdigest(),
                "plan": f"exporter/{name}_plan.json", "anchors": plan.anchors, "runs": runs,
            }
            print(name, trace.seq_len, plan.anchors, {r: v["overall"]["max_output_rel_err_l2"] for r, v in runs.items()})
    with open(os.path.join(HERE, "exporter_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_exporter_golden.py", "prompt": PROMPT, "cases": cases}, f,
                  indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
