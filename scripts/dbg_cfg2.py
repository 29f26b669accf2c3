import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2512_16391_b200 import engine, ops
plan = bench.make_plan(32, 8, bench.LLAMA_ANCHORS, 0.1, 128)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
eng = engine.KascadePrefill(plan, 32, 32, 8, N)
g = torch.Generator(device="cuda").manual_seed(0)
qs = [torch.randn(32, N, 128, device="cuda", generator=g).bfloat16() for _ in range(2)]
ks = [torch.randn(8, N, 128, device="cuda", generator=g).bfloat16() for _ in range(2)]
vs = [torch.randn(8, N, 128, device="cuda", generator=g).bfloat16() for _ in range(2)]
for l, kind in enumerate(eng.kinds[:4]):
    print("layer", l, kind, flush=True)
    eng.forward([qs[i % 2] for i in range(32)], [ks[i % 2] for i in range(32)], [vs[i % 2] for i in range(32)], stop_after=l)
    torch.cuda.synchronize()
print("ok")
