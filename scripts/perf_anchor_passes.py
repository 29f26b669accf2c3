"""Anchor prefill passes A (LSE) and B (pooled + Top-k) timing (dev tool).
python scripts/perf_anchor_passes.py N [reps]   (KSCD_LIB_PATH selects a library variant)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    Hq, Hkv = 32, 8
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn(Hq, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    lse = ops.anchor_lse_prefill(q, k)
    pol = KBudgetPolicy(0.1, 128)
    idx, cnt = ops.select_prefill(q, k, lse, pol)
    torch.cuda.synchronize()

    def t(fn):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    a = t(lambda: ops.anchor_lse_prefill(q, k, lse=lse))
    b = t(lambda: ops.select_prefill(q, k, lse, pol, indices=idx, counts=cnt))
    lib = os.path.basename(os.environ.get("KSCD_LIB_PATH", "in-tree"))
    print(f"{lib} N={N} passA {a:.2f} ms  passB+topk {b:.2f} ms  sum {a + b:.2f}")


if __name__ == "__main__":
    main()
