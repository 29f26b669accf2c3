"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host path:
batch / kv-head partitioning, the anchor index-list all-gather that the
head remap needs, and head-sharded output reassembly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kascade_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_exchange(rank, world, port, errq):
    try:
        _init(rank, world, port)
        from paper_2512_16391_b200 import sharding
        B, Hq, Hkv, n = 2, 8, 4, 300
        G = Hq // Hkv
        rng = np.random.default_rng(0)   # same inputs on every rank
        q = orc.bf16_round(rng.standard_normal((B, Hq, 128)).astype(np.float32) * 2)
        K = orc.bf16_round(rng.standard_normal((B, Hkv, n, 128)).astype(np.float32))
        V = orc.bf16_round(rng.standard_normal((B, Hkv, n, 128)).astype(np.float32))
        k = orc.k_budget(0.1, 16, n)
        # unsharded reference selection (decode tile of the last token)
        full = np.zeros((B, Hkv, k), np.int32)
        for b in range(B):
            for g in range(Hkv):
                P = np.stack([orc.dense_row(q[b, g * G + j], K[b, g], V[b, g])[0] for j in range(G)])
                full[b, g] = orc.topk_sorted(P[:, None, :].mean(axis=(0, 1), dtype=np.float64), k)
        g0, g1 = sharding.kv_head_shard(Hkv)
        assert (g0, g1) == (rank * 2, rank * 2 + 2)
        local_idx = torch.from_numpy(full[:, g0:g1].copy())
        local_cnt = torch.full((B, g1 - g0), k, dtype=torch.int32)
        idx, cnt = sharding.gather_index_lists(local_idx, local_cnt)
        assert torch.equal(idx, torch.from_numpy(full)), "gathered lists differ from the unsharded selection"
        assert torch.equal(cnt, torch.full((B, Hkv), k, dtype=torch.int32))
        # the overlapped form the sharded executors use gives the same lists
        # (prefill layout too: heads on dim 0)
        pidx, pcnt = sharding.PendingIndexGather(local_idx, local_cnt, head_dim=1).wait()
        assert torch.equal(pidx, idx) and torch.equal(pcnt, cnt)
        tidx, tcnt = sharding.PendingIndexGather(local_idx.permute(1, 0, 2).contiguous(), local_cnt.t().contiguous(),
                                                 head_dim=0).wait()
        assert torch.equal(tidx, idx.permute(1, 0, 2)) and torch.equal(tcnt, cnt.t())
        # head-remap routing of this rank's reuse heads through the GLOBAL map
        head_map = [3, 0, 2, 1]
        lm = sharding.local_head_map(head_map, g0, g1)
        sels = {(g, 0): full[0, g] for g in range(Hkv)}
        routed = orc.route(sels, head_map, Hkv)
        for gl, src in enumerate(lm.tolist()):
            np.testing.assert_array_equal(idx[0, src].numpy(), routed[(g0 + gl, 0)])
        # prefill layout: [Hloc][T][k] gathered along dim 0
        T = 3
        pidx = torch.arange(2 * T * 5, dtype=torch.int32).reshape(2, T, 5) + 1000 * rank
        pcnt = torch.full((2, T), 5, dtype=torch.int32)
        gi, gc = sharding.gather_index_lists(pidx, pcnt, head_dim=0)
        assert gi.shape == (4, T, 5) and int(gi[2, 0, 0]) == 1000 and int(gi[0, 0, 0]) == 0
        # head-sharded outputs reassemble in head order
        out = torch.full((B, (g1 - g0) * G, 4), float(rank))
        allo = sharding.gather_head_outputs(out, head_dim=1)
        assert allo.shape == (B, Hq, 4)
        assert float(allo[0, 0, 0]) == 0.0 and float(allo[0, Hq - 1, 0]) == 1.0
        # batch sharding is a partition
        b0, b1 = sharding.batch_shard(5)
        spans = [None, None]
        dist.all_gather_object(spans, (b0, b1))
        assert spans == [(0, 3), (3, 5)]
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_two_rank_index_exchange_and_routing():
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_exchange, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    msgs = []
    while not errq.empty():
        msgs.append(errq.get())
    assert not msgs, msgs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_even_split_partitions():
    from paper_2512_16391_b200.sharding import even_split
    for n in (0, 1, 7, 8, 64):
        for world in (1, 2, 3, 8):
            spans = [even_split(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_kv_head_shard_rejects_uneven_split():
    from paper_2512_16391_b200 import sharding
    from paper_2512_16391_b200.exceptions import InvalidArgumentError
    with pytest.raises(InvalidArgumentError):
        sharding.even_split(4, 2, 5)
    assert sharding.kv_head_shard(8) == (0, 8)   # no process group: one rank owns all
