import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2512_16391_b200 import ops
torch.manual_seed(0)
for N in (64, 128, 192, 256, 300, 1000):
    for Hq, Hkv in ((4, 1), (8, 2), (16, 2)):
        q = torch.randn(Hq, N, 128, device="cuda").bfloat16()
        k = torch.randn(Hkv, N, 128, device="cuda").bfloat16()
        v = torch.randn(Hkv, N, 128, device="cuda").bfloat16()
        out, lse = ops.dense_prefill(q, k, v)
        G = Hq // Hkv
        kk = k.float().repeat_interleave(G, 0); vv = v.float().repeat_interleave(G, 0)
        s = q.float() @ kk.transpose(1, 2) / 128 ** 0.5
        mask = torch.triu(torch.ones(N, N, dtype=torch.bool, device="cuda"), 1)
        s = s.masked_fill(mask, float("-inf"))
        ref = torch.softmax(s, -1) @ vv
        rl = torch.logsumexp(s, -1)
        e = (out.float() - ref).abs()
        rows = e.amax(dim=(0, 2))
        bad = (rows > 2e-2).nonzero().flatten().tolist()
        print(N, Hq, Hkv, "out max", e.max().item(), "lse max", (lse - rl).abs().max().item(), "bad rows", bad[:8], len(bad))
