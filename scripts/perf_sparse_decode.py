"""Reuse-layer sparse decode timing vs split-K factor (dev tool).
KSCD_SPARSE_STAGES=2|3 python scripts/perf_sparse_decode.py [splits ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    B, Hq, Hkv, n = 8, 32, 8, 131072
    L = 6
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    pol = KBudgetPolicy(0.1, 128)
    _, _, idx, cnt = ops.anchor_decode(q, ks[0], vs[0], n, pol, layer0=True)
    out = torch.empty(B, Hq, 128, dtype=torch.float32, device="cuda")
    ref = ops.sparse_decode(q, ks[0], vs[0], n, idx, cnt, None).clone()
    k = int(cnt.flatten()[0].item())
    res = []
    for sp in [int(x) for x in sys.argv[1:]] or [0]:
        o = ops.sparse_decode(q, ks[0], vs[0], n, idx, cnt, None, num_splits=sp)
        err = (o - ref).abs().max().item()
        for _ in range(3):
            ops.sparse_decode(q, ks[1], vs[1], n, idx, cnt, None, out=out, num_splits=sp)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        reps = 60
        for i in range(reps):
            ops.sparse_decode(q, ks[i % L], vs[i % L], n, idx, cnt, None, out=out, num_splits=sp)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / reps * 1e3
        iso = []
        for i in range(20):   # isolated launches, events around each (as bench.py's roofline)
            s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s1.record()
            ops.sparse_decode(q, ks[i % L], vs[i % L], n, idx, cnt, None, out=out, num_splits=sp)
            e1.record()
            iso.append((s1, e1))
        torch.cuda.synchronize()
        iso_us = sum(a.elapsed_time(b) for a, b in iso) / len(iso) * 1e3
        res.append(f"splits={sp}:chain {us:.1f}us iso {iso_us:.1f}us (err={err:.1e})")
    print(f"stages={os.environ.get('KSCD_SPARSE_STAGES', '3')}", " ".join(res))


if __name__ == "__main__":
    main()
