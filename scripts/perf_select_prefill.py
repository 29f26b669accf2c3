"""Prefill select (pass B + Top-k) timing on bench-like rows (dev tool).
python scripts/perf_select_prefill.py [N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    Hq, Hkv = 32, 8
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn(Hq, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    lse = ops.anchor_lse_prefill(q, k)
    pol = KBudgetPolicy(0.1, 128)
    idx, cnt = ops.select_prefill(q, k, lse, pol)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ops.select_prefill(q, k, lse, pol, indices=idx, counts=cnt)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"N={N} nocand={int('KSCD_TOPK_NOCAND' in os.environ)} select_prefill ms: " + " ".join(f"{t:.2f}" for t in ts))


if __name__ == "__main__":
    main()
