"""Sparse decode time vs split-K factor for few (sequence, kv head) rows (dev tool)."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2512_16391_b200 import ops
from paper_2512_16391_b200.host_types import KBudgetPolicy
B, Hq, Hkv, n = (int(x) for x in sys.argv[1:5])
L = 6
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
ks = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
vs = [torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
out, lse, idx, cnt = ops.anchor_decode(q, ks[0], vs[0], n, KBudgetPolicy(0.1, 128), layer0=True)
for s_ in (0, 9, 18, 37, 64, 74, 128):
    def f(i):
        ops.sparse_decode(q, ks[i % L], vs[i % L], n, idx, cnt, None, out=out, num_splits=s_)
    f(0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(30): f(i)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 30 * 1e3
    print(f"splits={s_:4d} {us:7.1f} us  {int(cnt.sum()) * 516 / us / 1e3:6.0f} GB/s")
