"""Time the kv-head-sharded decode step (dev tool): one NCCL rank holding
every kv head of the 70B plan (80 layers, 64Q/8KV, 128K, batch 8; 8 distinct
KV buffers cycled), the whole step captured as one CUDA graph -- the code
path configs[4] runs on every rank at N > 1.  python scripts/perf_sharded_decode.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import sharding  # noqa: E402
from paper_2512_16391_b200.host_types import read_plan  # noqa: E402


def main(N=131072, B=8, L=80, Hq=64, Hkv=8, distinct=8):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    plan = read_plan(os.path.join(repo, "plans", "llama70b.json"))
    g = torch.Generator(device=dev).manual_seed(0)
    Kc = [torch.randn(B, Hkv, N, 128, device=dev, dtype=torch.bfloat16, generator=g) for _ in range(distinct)]
    Vc = [torch.randn(B, Hkv, N, 128, device=dev, dtype=torch.bfloat16, generator=g) for _ in range(distinct)]
    Ks, Vs = [Kc[l % distinct] for l in range(L)], [Vc[l % distinct] for l in range(L)]
    q = (torch.randn(L, B, Hq, 128, device=dev, generator=g) * 2).to(torch.bfloat16)
    dec = sharding.ShardedKascadeDecoder(plan, L, B, Hq, Hkv, N)
    gr = dec.capture(q, Ks, Vs, N)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        gr.replay()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"sharded decode step (1 rank, all heads): {ms:.3f} ms = {ms * 1e3 / B:.1f} us/token")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
