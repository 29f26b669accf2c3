"""Per-op decode timing at any shape (dev tool).
python scripts/perf_decode_ops.py B Hq Hkv n [fraction]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    B, Hq, Hkv, n = (int(x) for x in sys.argv[1:5])
    frac = float(sys.argv[5]) if len(sys.argv) > 5 else 0.1
    L = max(2, min(8, int(60e9 // (2 * B * Hkv * n * 256))))
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    pol = KBudgetPolicy(frac, 128)
    scores = ops.score_buffer(B, Hq, n, q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device="cuda")
    out, lse, idx, cnt = ops.anchor_decode(q, ks[0], vs[0], n, pol, layer0=True, scores=scores, lse=lse)
    pooled = None

    def t(fn, reps=40):
        fn(0)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(reps):
            fn(i)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps * 1e3

    kv = B * Hkv * n * 256
    k = int(cnt[0, 0].item()) if cnt.dim() == 2 else int(cnt.flatten()[0].item())
    r = {}
    r["dense"] = t(lambda i: ops.dense_decode(q, ks[i % L], vs[i % L], n, out=out, lse=lse))
    r["dense_scores"] = t(lambda i: ops.dense_decode(q, ks[i % L], vs[i % L], n, out=out, lse=lse, scores=scores))
    r["scores_pass1"] = t(lambda i: ops.anchor_scores_decode(q, ks[i % L], n, scores, lse))
    r["select"] = t(lambda i: ops.select_decode(scores, lse, n, pol, Hkv, indices=idx, counts=cnt))
    r["sparse"] = t(lambda i: ops.sparse_decode(q, ks[i % L], vs[i % L], n, idx, cnt, None, out=out))
    gbs = {"dense": 2 * kv, "dense_scores": 2 * kv + B * Hq * n * 4, "scores_pass1": kv + B * Hq * n * 4,
           "sparse": B * Hkv * k * 516}
    print(f"B={B} Hq={Hq} Hkv={Hkv} n={n} k={k}")
    for name, us in r.items():
        extra = f"  {gbs[name] / us / 1e3:7.0f} GB/s" if name in gbs else ""
        print(f"  {name:14s} {us:9.1f} us{extra}")


if __name__ == "__main__":
    main()
