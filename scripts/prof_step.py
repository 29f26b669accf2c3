"""One Kascade decode step of the bench's Llama-8B plan at 128K, batch 8
(8 distinct KV buffers cycled over the 32 layers, each 4.3 GB >> L2), for
ncu captures of the step's own launches -- e.g. its longest reuse run as
the single multi-layer launch it is (dev tool).
    ncu -k 'regex:decode_attn_kernel' -s 3 -c 1 ... python scripts/prof_step.py  (4th sparse launch: layers 13-31)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_16391_b200 import engine  # noqa: E402


def main(n=131072, B=8, distinct=8):
    L, Hq, Hkv = 32, 32, 8
    plan = bench.make_plan(L, Hkv, bench.LLAMA_ANCHORS, 0.1, 128)
    g = torch.Generator(device="cuda").manual_seed(0)
    Kc = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(distinct)]
    Vc = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(distinct)]
    q = (torch.randn(L, B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    dec.step(q, [Kc[l % distinct] for l in range(L)], [Vc[l % distinct] for l in range(L)], n)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
