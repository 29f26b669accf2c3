"""Drive each engine kernel a few times at bench shapes so that ncu can
capture it (dev tool).  python scripts/prof_kernels.py {decode|prefill} [N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def decode(n=131072, B=8, Hq=32, Hkv=8):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    k = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
    pol = KBudgetPolicy(0.1, 128)
    out, lse, idx, cnt = ops.anchor_decode(q, k, v, n, pol, layer0=True)
    hm = torch.arange(Hkv - 1, -1, -1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ops.reuse_decode(q, k, v, n, idx, cnt, hm, out=out)
    for _ in range(2):
        ops.anchor_decode(q, k, v, n, pol)
    torch.cuda.synchronize()


def prefill(N=32768, Hq=32, Hkv=8):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(Hq, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    pol = KBudgetPolicy(0.1, 128)
    hm = torch.tensor([3, 1, 0, 2, 7, 5, 6, 4], dtype=torch.int32, device="cuda")
    for _ in range(2):
        out, lse = ops.dense_prefill(q, k, v)
        ops.anchor_lse_prefill(q, k, lse=lse)
        idx, cnt = ops.select_prefill(q, k, lse, pol)
        ops.sparse_prefill(q, k, v, idx, cnt, hm, out=out)
    torch.cuda.synchronize()


def decode_shard(n=131072, B=8):
    """One rank of the 8-way kv-head-sharded 70B decode: 1 KV + 8 Q heads."""
    decode(n, B, 8, 1)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "decode"
    args = [int(a) for a in sys.argv[2:]]
    {"decode": decode, "prefill": prefill, "decode_shard": decode_shard}[which](*args)
