"""Per-CTA fixed cost of the sparse prefill (dev tool): every (kv head, tile)
selects exactly c * 128 keys (random positions before the tile), so every CTA
runs c key blocks; T(c) = waves * (F + c * B) separates the per-CTA fixed
cost F from the per-block cost B.  python scripts/perf_sparse_fixed.py [N]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    Hq, Hkv, d = 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(Hq, N, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, N, d, device="cuda", generator=g).to(torch.bfloat16)
    T = N // 128
    out = torch.empty(Hq, N, d, dtype=torch.bfloat16, device="cuda")
    res = {}
    for c in (4, 16, 48, 96):
        kc = c * 128
        lim = torch.clamp(torch.arange(T, device="cuda") * 128, min=1)            # keys strictly before the tile
        pos = (torch.rand(Hkv, T, kc, device="cuda", generator=g) * lim[None, :, None]).to(torch.int32)
        idx = torch.sort(pos, dim=-1).values.contiguous()
        cnt = torch.full((Hkv, T), kc, dtype=torch.int32, device="cuda")
        ops.sparse_prefill(q, k, v, idx, cnt, None, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            ops.sparse_prefill(q, k, v, idx, cnt, None, out=out)
        e.record()
        torch.cuda.synchronize()
        res[c] = s.elapsed_time(e) / 3
    ctas = T * Hq // 2
    waves = ctas / 148
    cs = sorted(res)
    # least-squares line through (c, T(c) / waves)
    xs = cs
    ys = [res[c] * 1e3 / waves for c in cs]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    B = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    F = my - B * mx
    print(json.dumps({"N": N, "ms": {c: round(res[c], 3) for c in cs}, "waves": round(waves, 1),
                      "per_cta_fixed_us": round(F, 2), "per_block_us": round(B, 3)}))


if __name__ == "__main__":
    main()
