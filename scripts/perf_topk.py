"""Top-k kernel timing at the bench's decode and prefill shapes (dev tool).
python scripts/perf_topk.py            (KSCD_LIB_PATH selects a library variant)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {}
    # decode: realistic pooled rows (dense pass scores -> select_decode), 8
    # sequences x 8 kv heads, n = 128K, k = 10 %
    from paper_2512_16391_b200.host_types import KBudgetPolicy
    B, Hq, Hkv, n = 8, 32, 8, 131072
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    kc = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    sc = ops.score_buffer(B, Hq, n, "cuda")
    _, lse = ops.dense_decode(q, kc, kc, n, scores=sc)
    del kc
    pol = KBudgetPolicy(0.1, 128)
    pooled = torch.empty(B * Hkv, n, dtype=torch.float32, device="cuda")
    idx0, _ = ops.select_decode(sc, lse, n, pol, Hkv, pooled=pooled)
    k = ops.k_budget(pol, n)
    idx, _ = ops.topk(pooled, k)
    assert torch.equal(idx.view(B, Hkv, -1)[:, :, :k], idx0[:, :, :k]), "decode top-k mismatch"
    ref = torch.sort(torch.topk(pooled, k, dim=1).indices, dim=1).values.to(torch.int32)
    assert torch.equal(idx[:, :k], ref), "decode top-k differs from torch.topk"
    res["decode_64x128K"] = timed(lambda: ops.topk(pooled, k))
    p8 = pooled[:8].contiguous()
    res["shard_8x128K"] = timed(lambda: ops.topk(p8, k))
    p32 = pooled[:, :32768].contiguous()
    res["decode_64x32K"] = timed(lambda: ops.topk(p32, 32768 // 40))
    # prefill: 8 kv heads x T tiles, row t has 128 (t + 1) keys, k = 10 % (k_min 128)
    for N in (32768, 131072):
        T = N // 128
        stride = N
        pv = torch.exp(torch.randn(8 * T, stride, device="cuda", generator=g) * 2 - 12)
        lens = (torch.arange(T, device="cuda", dtype=torch.int32) + 1).repeat(8) * 128
        ks = torch.clamp(lens // 10, min=128).to(torch.int32)
        res[f"prefill_{N // 1024}K"] = timed(lambda: ops.topk(pv, ks, lengths=lens, k_cap=int(ks.max())), reps=5)
        del pv
    lib = os.environ.get("KSCD_LIB_PATH", "in-tree")
    print(os.path.basename(lib), " ".join(f"{k}={v:.1f}us" for k, v in res.items()))


if __name__ == "__main__":
    main()
