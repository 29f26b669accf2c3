"""Per-block timeline of one pass-B CTA (dev tool; KSCD_PB_TRACE variant):
for each key block and quarter (head) the column-sum warpgroups' wait start
and S^T-ready stamps (warp quarter 0, lane 0).
    bash scripts/build_variant.sh pbtrace -DKSCD_PB_TRACE
    KSCD_LIB_PATH=_exp/libkascade_pbtrace.so python scripts/pb_trace.py [N]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import _lib, ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    Hq, Hkv = 32, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(Hq, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    lse = ops.anchor_lse_prefill(q, k)
    ops.select_prefill(q, k, lse, KBudgetPolicy(0.1, 128))
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * (512 * 8))()
    _lib.load().kscd_debug_pb_trace(ctypes.cast(buf, ctypes.c_void_p))
    t = np.frombuffer(buf, dtype=np.int64).reshape(512, 8).astype(np.float64)
    nb = int((t[:, 4] > 0).sum())
    t = t[:nb] - t[0, 0]
    mid = slice(nb // 4, 3 * nb // 4)
    # WG 0 owns quarters 0 and 2
    wait0, wait2 = t[:, 4] - t[:, 0], t[:, 6] - t[:, 2]
    per = np.diff(t[:, 0])
    work0 = t[:, 2] - t[:, 4]                 # quarter 0 ready -> quarter 2 wait start (ld + colsum of q0)
    work2 = t[1:, 0] - t[:-1, 6]              # quarter 2 ready -> next block's quarter 0 wait start
    q = lambda a: f"med {np.median(a):6.0f}  p10 {np.percentile(a, 10):6.0f}  p90 {np.percentile(a, 90):6.0f}"
    print(f"N={N} blocks={nb}")
    print("period per block:          ", q(per[mid]))
    print("quarter 0: wait for S^T    ", q(wait0[mid]), "  work", q(work0[mid]))
    print("quarter 2: wait for S^T    ", q(wait2[mid]), "  work", q(work2[mid]))
    tb = (ctypes.c_longlong * 4)()
    _lib.load().kscd_debug_pb_tail(ctypes.cast(tb, ctypes.c_void_p))
    t0, t1, t2 = tb[0], tb[1], tb[2]
    print(f"CTA: column sums {t1 - t0} clocks ({nb} blocks, {(t1 - t0) / nb:.0f} per block incl. prologue), "
          f"fused Top-k tail {t2 - t1} clocks ({(t2 - t1) / max(t2 - t0, 1):.1%} of the CTA)")


if __name__ == "__main__":
    main()
