"""Debug: engine vs ops pre-softmax selection at growing sizes (dev tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import kascade_oracle as orc
from paper_2512_16391_b200 import ops, engine
from paper_2512_16391_b200.host_types import KBudgetPolicy, AnchorPlan, AnchorPlanCore, HeadMap

pol = KBudgetPolicy(0.1, 128)
for (B, n) in ((2, 70000), (8, 70000), (2, 131072), (8, 131072)):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = (torch.randn(B, 32, 128, device="cuda", generator=g) * 2).bfloat16()
    K = torch.randn(B, 8, n, 128, device="cuda", generator=g).bfloat16()
    idx, cnt = ops.select_decode_pre(q, K, n, pol)
    qn, Kn = q.float().cpu().numpy(), K.float().cpu().numpy()
    k = orc.k_budget(0.1, 128, n)
    bad = 0
    for b in range(B):
        for gg in range(8):
            qbar = qn[b, gg * 4:(gg + 1) * 4].mean(axis=0, dtype=np.float64)
            pooled = orc.softmax_vec((Kn[b, gg].astype(np.float64) @ qbar) / np.sqrt(128)).astype(np.float64)
            ref = orc.topk_sorted(pooled, k)
            d = np.setxor1d(idx[b, gg, :k].cpu().numpy(), ref).size
            bad += d > 10
    print(B, n, "rows with >10 differences:", bad, flush=True)
