"""Per-stream GPU timeline of one overlapped decode step (dev tool): wraps
the ops the executor calls with CUDA events on the calling stream and prints
each launch's start / end relative to the step start (eager step after a
warm-up; the CPU enqueues far ahead of the GPU at these kernel lengths).
python scripts/timeline_step.py [n] [B]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_16391_b200 import engine, ops  # noqa: E402

MARKS = []


def wrap(name):
    fn = getattr(ops, name)

    def w(*a, **k):
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r = fn(*a, **k)
        e1.record(s)
        tag = name
        if name == "decode_layers":
            tag += f"[{len(a[1])}L{' scores' if k.get('scores') is not None else ''}]"
        MARKS.append((tag, s.stream_id, e0, e1))
        return r
    setattr(ops, name, w)


def main(n=131072, B=8, distinct=8):
    L, Hq, Hkv = 32, 32, 8
    plan = bench.make_plan(L, Hkv, bench.LLAMA_ANCHORS, 0.1, 128)
    g = torch.Generator(device="cuda").manual_seed(0)
    Kc = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(distinct)]
    Vc = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(distinct)]
    q = (torch.randn(L, B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    Ks, Vs = [Kc[l % distinct] for l in range(L)], [Vc[l % distinct] for l in range(L)]
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    for _ in range(2):
        dec.step(q, Ks, Vs, n)
    torch.cuda.synchronize()
    for name in ("dense_decode", "select_decode", "decode_layers", "sparse_decode", "anchor_scores_decode"):
        wrap(name)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    dec.step(q, Ks, Vs, n)
    end.record()
    torch.cuda.synchronize()
    main_id = torch.cuda.current_stream().stream_id
    print(f"step {start.elapsed_time(end) * 1e3:.0f} us")
    for tag, sid, e0, e1 in sorted(MARKS, key=lambda m: start.elapsed_time(m[2])):
        t0, t1 = start.elapsed_time(e0) * 1e3, start.elapsed_time(e1) * 1e3
        print(f"{'main' if sid == main_id else 'side':4s} {t0:7.0f} {t1:7.0f} {t1 - t0:6.0f}  {tag}")


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
