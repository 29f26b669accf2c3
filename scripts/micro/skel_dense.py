import sys, torch, json
sys.path.insert(0, "/root/repo")
from paper_2512_16391_b200 import ops
for N in (32768, 131072):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(32, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(8, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(8, N, 128, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty_like(q); lse = torch.empty(32, N, device="cuda")
    ops.dense_prefill(q, k, v, out=out, lse=lse); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): ops.dense_prefill(q, k, v, out=out, lse=lse)
    e.record(); torch.cuda.synchronize()
    print(N, "dense skeleton ms", s.elapsed_time(e) / 3)
