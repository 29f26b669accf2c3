"""Per-kernel decode timing at the bench shape (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402

B, Hq, Hkv, n = 8, 32, 8, 131072
L = 6
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
pol = KBudgetPolicy(0.1, 128)
out, lse, idx, cnt = ops.anchor_decode(q, ks[0], vs[0], n, pol, layer0=True)
hm = torch.tensor([3, 1, 0, 2, 7, 5, 6, 4], dtype=torch.int32, device="cuda")


def t(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(reps):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


us = t(lambda i=0: ops.sparse_decode(q, ks[i % L], vs[i % L], n, idx, cnt, hm, out=out))
byt = int(cnt.sum()) * 516
print(f"stages={os.environ.get('KSCD_SPARSE_STAGES', '3')} sparse_us={us:.1f} GB/s={byt / us / 1e3:.0f}")
