"""Per-kernel prefill timing at Llama-3.1-8B head shapes (dev tool; the
judged numbers come from bench.py).  python scripts/perf_prefill.py [N]"""

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    Hq, Hkv, d = 32, 8, 128
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(Hq, N, d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, N, d, device=dev, generator=g).to(torch.bfloat16)
    pol = KBudgetPolicy(0.1, 128)
    out = torch.empty(Hq, N, d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(Hq, N, dtype=torch.float32, device=dev)
    res = {"N": N}
    flops_dense = 2.0 * d * Hq * N * (N + 1)          # QK^T + PV, causal
    t = timeit(lambda: ops.dense_prefill(q, k, v, out=out, lse=lse))
    res["dense_ms"] = t
    res["dense_tflops"] = flops_dense / t / 1e9
    t = timeit(lambda: ops.anchor_lse_prefill(q, k, lse=lse))
    res["lse_pass_ms"] = t
    res["lse_pass_tflops"] = flops_dense / 2 / t / 1e9
    if len(sys.argv) > 2 and sys.argv[2] == "dense-only":
        res["lib"] = os.environ.get("KSCD_LIB_PATH", "default")
        print(json.dumps({k_: (round(v_, 3) if isinstance(v_, float) else v_) for k_, v_ in res.items()}))
        return
    T = (N + 127) // 128
    pooled = ops.select_prefill_scratch(Hq, Hkv, N, dev)
    idx = torch.empty(Hkv, T, ops.prefill_k_cap(pol, N), dtype=torch.int32, device=dev)
    cnt = torch.empty(Hkv, T, dtype=torch.int32, device=dev)
    t = timeit(lambda: ops.select_prefill(q, k, lse, pol, indices=idx, counts=cnt, pooled=pooled))
    res["select_ms"] = t
    hm = torch.tensor([3, 1, 0, 2, 7, 5, 6, 4], dtype=torch.int32, device=dev)
    t = timeit(lambda: ops.sparse_prefill(q, k, v, idx, cnt, hm, out=out))
    c = cnt.cpu()
    rows_keys = 0
    for ti in range(T):
        rows = min(N, 128 * ti + 128) - 128 * ti
        rows_keys += rows * int(c[:, ti].sum())
    flops_sparse = 4.0 * d * (Hq // Hkv) * rows_keys
    res["sparse_ms"] = t
    res["sparse_tflops"] = flops_sparse / t / 1e9
    print(json.dumps({k_: (round(v_, 3) if isinstance(v_, float) else v_) for k_, v_ in res.items()}))


if __name__ == "__main__":
    main()
