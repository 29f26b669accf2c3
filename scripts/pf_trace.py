"""Per-block pipeline timeline of one prefill CTA (the middle tile, head pair
0) from a KSCD_PF_TRACE variant build (dev tool):
    bash scripts/build_variant.sh pftrace -DKSCD_PF_TRACE
    KSCD_LIB_PATH=_exp/libkascade_pftrace.so python scripts/pf_trace.py {dense|sparse|lse} [N]
Events per key block j (SM clock64): MMA thread after P0(j) / after issuing
S0(j+1) / after P1(j) / after issuing S1(j+1); softmax tile 0 and tile 1
(warp lane 0 of quarter 0): S(j) ready / P(j) written."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import _lib, ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "dense"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    Hq, Hkv = 32, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(Hq, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    lib = _lib.load()
    if mode == "lse":
        torch.cuda.synchronize()
        lib.kscd_debug_pf_trace_reset()
        lse = ops.anchor_lse_prefill(q, k)
    else:
        out, lse = ops.dense_prefill(q, k, v)
    if mode == "sparse":
        idx, cnt = ops.select_prefill(q, k, lse, KBudgetPolicy(0.1, 128))
        torch.cuda.synchronize()
        lib.kscd_debug_pf_trace_reset()
        ops.sparse_prefill(q, k, v, idx, cnt, None, out=out)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * (256 * 8))()
    rc = lib.kscd_debug_pf_trace(ctypes.cast(buf, ctypes.c_void_p))
    t = np.frombuffer(buf, dtype=np.int64).reshape(256, 8).astype(np.float64)
    nb = int((t[:, 4] > 0).sum())
    t = t[:nb]
    t -= t[0, 4]
    print(f"mode={mode} N={N} rc={rc} blocks traced={nb}")
    per = np.diff(t[:, 4])
    sm0, sm1 = t[:, 5] - t[:, 4], t[:, 7] - t[:, 6]
    wake0 = t[:, 0] - t[:, 5]                  # P0 written -> MMA thread past its wait
    s_next0 = t[1:, 4] - t[:-1, 1]             # S0(j+1) issued -> softmax 0 sees it
    gap01 = t[:, 6] - t[:, 4]                  # tile 1 lag behind tile 0
    q = lambda a: f"med {np.median(a):6.0f}  p10 {np.percentile(a, 10):6.0f}  p90 {np.percentile(a, 90):6.0f}"
    mid = slice(nb // 4, 3 * nb // 4)
    print("period per block (S0 ready -> next S0 ready):", q(per[mid]))
    print("softmax tile 0 (S ready -> P written):        ", q(sm0[mid]))
    print("softmax tile 1:                                ", q(sm1[mid]))
    print("P0 written -> MMA issues PV0:                  ", q(wake0[mid]))
    print("S0(j+1) issued -> softmax 0 sees it:           ", q(s_next0[mid]))
    print("tile 1 S-ready lag behind tile 0:              ", q(gap01[mid]))
    print("MMA: PV0 issue -> S0 issued:", q((t[:, 1] - t[:, 0])[mid]), " P1 wait done - S0 issued:",
          q((t[:, 2] - t[:, 1])[mid]))
    for j in list(range(nb // 2, nb // 2 + 4)):
        print(j, " ".join(f"{x:8.0f}" for x in t[j]))


if __name__ == "__main__":
    main()
