"""Time the exact Top-k on realistic decode pooled rows (dev tool).
KSCD_TOPK_VARIANT=<cluster><agg> python scripts/perf_topk.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402

B, Hq, Hkv, n = 8, 32, 8, 131072
g = torch.Generator(device="cuda").manual_seed(0)
q = (torch.randn(B, Hq, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
k = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(B, Hkv, n, 128, device="cuda", generator=g).to(torch.bfloat16)
sc = ops.score_buffer(B, Hq, n, "cuda")
_, lse = ops.dense_decode(q, k, v, n, scores=sc)
pol = KBudgetPolicy(0.1, 128)
pooled = torch.empty(B * Hkv, n, dtype=torch.float32, device="cuda")
idx, cnt = ops.select_decode(sc, lse, n, pol, Hkv, pooled=pooled)
ref = idx.clone()
kk = ops.k_budget(pol, n)
for _ in range(3):
    i2, c2 = ops.topk(pooled, kk)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    i2, c2 = ops.topk(pooled, kk)
e.record()
torch.cuda.synchronize()
same = torch.equal(i2.view(B, Hkv, -1)[:, :, :kk], ref[:, :, :kk])
print(f"variant={os.environ.get('KSCD_TOPK_VARIANT', 'default')} topk_us={s.elapsed_time(e) / 20 * 1e3:.1f} same={same}")
