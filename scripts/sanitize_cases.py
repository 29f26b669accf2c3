"""Small launches of every product kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck --error-exitcode 1 python scripts/sanitize_cases.py

Shapes are tiny but take every code path that matters for the checks:
split-K decode with several splits and the last-CTA merge + counter re-arm
(run twice on one workspace), the cluster Top-k (rows >= 8192 keys, DSMEM
histogram reduction) and the single-CTA one, the decode select, the tcgen05
prefill kernels (dense, LSE pass, pass B + Top-k, sparse gather with a head
map and fallback rows), the KV append (fixed and ragged positions)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16391_b200 import ops  # noqa: E402
from paper_2512_16391_b200.host_types import KBudgetPolicy  # noqa: E402


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    pol = KBudgetPolicy(0.1, 16)
    # ---------------- decode: B=2, 8Q/2KV, n=9000 (several splits, cluster Top-k)
    B, Hq, Hkv, n = 2, 8, 2, 9000
    q = (torch.randn(B, Hq, 128, device=dev) * 2).bfloat16()
    k = torch.randn(B, Hkv, n + 8, 128, device=dev).bfloat16()
    v = torch.randn(B, Hkv, n + 8, 128, device=dev).bfloat16()
    ws = ops.new_decode_workspace(dev, B, Hq, Hkv)
    sc = ops.score_buffer(B, Hq, n, dev)
    for rep in range(2):                        # second run reuses the re-armed counters
        out, lse = ops.dense_decode(q, k, v, n, scores=sc, num_splits=5, workspace=ws)
        idx, cnt = ops.select_decode(sc, lse, n, pol, Hkv)
        ops.anchor_scores_decode(q, k, n, sc, lse, num_splits=3, workspace=ws)
        hm = torch.tensor([1, 0], dtype=torch.int32, device=dev)
        ops.sparse_decode(q, k, v, n, idx, cnt, hm, num_splits=4, workspace=ws)
    lens = torch.tensor([n, n // 2], dtype=torch.int32, device=dev)
    out, lse = ops.dense_decode(q, k, v, n, scores=sc, seq_lens=lens, workspace=ws)
    ops.select_decode(sc, lse, n, pol, Hkv, seq_lens=lens)
    # single-CTA Top-k (short rows) and ties
    vals = torch.randint(0, 50, (6, 3000), device=dev).float()
    ops.topk(vals, 100)
    # KV append: one layer table, fixed position and ragged lengths
    kv_new = torch.randn(1, 2, B, Hkv, 128, device=dev).bfloat16()
    tables = ops.cache_pointer_tables([k], [v], dev)
    ops.append_kv(kv_new, n, tables)
    ops.append_kv(kv_new, n, tables, torch.tensor([5, n + 8], dtype=torch.int32, device=dev))
    # ---------------- prefill: 4Q/2KV, N=640 (5 tiles, last one ragged)
    Hq, Hkv, N = 4, 2, 600
    qp = torch.randn(Hq, N, 128, device=dev).bfloat16()
    kp = torch.randn(Hkv, N, 128, device=dev).bfloat16()
    vp = torch.randn(Hkv, N, 128, device=dev).bfloat16()
    o, lse = ops.dense_prefill(qp, kp, vp)
    lse2 = ops.anchor_lse_prefill(qp, kp)
    idx, cnt = ops.select_prefill(qp, kp, lse2, KBudgetPolicy(0.1, 64))
    ops.sparse_prefill(qp, kp, vp, idx, cnt, torch.tensor([1, 0], dtype=torch.int32, device=dev))
    # hand-made selection with rows that see no key (V[r] fallback)
    T = (N + 127) // 128
    sel = torch.full((Hkv, T, 8), 2**31 - 1, dtype=torch.int32, device=dev)
    sel[:, :, :3] = torch.tensor([100, 120, 127], dtype=torch.int32, device=dev)
    c3 = torch.full((Hkv, T), 3, dtype=torch.int32, device=dev)
    ops.sparse_prefill(qp, kp, vp, sel, c3)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
