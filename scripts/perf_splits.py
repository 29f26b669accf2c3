"""Decode kernels (dense, scores, sparse) vs split-K factor, isolated and
chained launches (dev tool).  HQ=32 HKV=8 python scripts/perf_splits.py B n [splits ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def timed(fn, L):
    for i in range(3):
        fn(i % L)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(30):
        fn(i % L)
    e.record()
    torch.cuda.synchronize()
    chain = s.elapsed_time(e) / 30 * 1e3
    ev = []
    for i in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(i % L)
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return chain, sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3


def main():
    B, n = int(sys.argv[1]), int(sys.argv[2])
    splits = [int(x) for x in sys.argv[3:]] or [0]
    Hq, Hkv = int(os.environ.get("HQ", 32)), int(os.environ.get("HKV", 8))
    L = max(2, min(6, int(50e9 // (2 * B * Hkv * n * 256))))
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    frac = 0.1 if n >= 65536 else 0.025
    _, _, idx, cnt = ops.anchor_decode(q, ks[0], vs[0], n, KBudgetPolicy(frac, 128), layer0=True)
    out = torch.empty(B, Hq, 128, dtype=torch.float32, device="cuda")
    lse = torch.empty(B, Hq, dtype=torch.float32, device="cuda")
    sc = ops.score_buffer(B, Hq, n, "cuda")
    print(f"B={B} n={n} k={int(cnt.flatten()[0])}")
    for sp in splits:
        r = {
            "dense": timed(lambda i: ops.dense_decode(q, ks[i], vs[i], n, out=out, lse=lse, num_splits=sp), L),
            "scores": timed(lambda i: ops.anchor_scores_decode(q, ks[i], n, sc, lse, num_splits=sp), L),
            "sparse": timed(lambda i: ops.sparse_decode(q, ks[i], vs[i], n, idx, cnt, None, out=out, num_splits=sp), L),
        }
        print(f"  splits={sp:2d} " + "  ".join(f"{k}: chain {c:7.1f} iso {s:7.1f}" for k, (c, s) in r.items()))


if __name__ == "__main__":
    main()
