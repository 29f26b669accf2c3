"""Run one prefill kernel repeatedly while sampling SM clocks / power (dev tool).
python scripts/clock_probe.py {dense|lse|select|sparse} N reps"""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    which, N, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    Hq, Hkv, d = 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(Hq, N, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, N, d, device="cuda", generator=g).to(torch.bfloat16)
    out, lse = ops.dense_prefill(q, k, v)
    pol = KBudgetPolicy(0.1, 128)
    idx, cnt = ops.select_prefill(q, k, lse, pol)
    hm = torch.arange(Hkv, dtype=torch.int32, device="cuda")
    fn = {"dense": lambda: ops.dense_prefill(q, k, v, out=out, lse=lse),
          "lse": lambda: ops.anchor_lse_prefill(q, k, lse=lse),
          "select": lambda: ops.select_prefill(q, k, lse, pol, indices=idx, counts=cnt),
          "sparse": lambda: ops.sparse_prefill(q, k, v, idx, cnt, hm, out=out)}[which]
    fn()
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    p.terminate()
    lines = p.stdout.read().strip().splitlines()
    print(which, N, f"{s.elapsed_time(e) / reps:.3f} ms/launch", lines[len(lines) // 4: len(lines) // 4 + 6])


if __name__ == "__main__":
    main()
