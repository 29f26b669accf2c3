"""KV-head-sharded decode and prefill executors with a real 2-process group
(gloo, both ranks on cuda:0): the anchor index lists cross ranks through the
all-gather, reuse heads gather through the global head map, and the
reassembled outputs match the unsharded engine.  Needs a B200."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errq, backend="gloo"):
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dev = 0 if backend == "gloo" else rank          # NCCL: one GPU per rank
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import kascade_oracle as orc
        from paper_2512_16391_b200 import engine, sharding
        from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
        L, B, Hq, Hkv, n = 7, 2, 8, 4, 1200
        G = Hq // Hkv
        # anchors 2-3 run as one group (one all-gather of layer 3's lists);
        # reuse layers 4-6 run as one multi-layer launch over the gathered lists
        plan = AnchorPlan(AnchorPlanCore([0, 2, 3], 3, 0.0),
                          head_maps={1: HeadMap(1, 0, [2, 0, 3, 1]), 4: HeadMap(4, 3, [3, 2, 1, 0]),
                                     5: HeadMap(5, 3, [1, 1, 2, 2]), 6: HeadMap(6, 3, [0, 3, 0, 3])},
                          k_policy=KBudgetPolicy(0.1, 64))
        rng = np.random.default_rng(5)
        q = orc.bf16_round((rng.standard_normal((L, B, Hq, 128)) * 2).astype(np.float32))
        K = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
        V = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)  # noqa: E731
        g0, g1 = sharding.kv_head_shard(Hkv)
        dec = sharding.ShardedKascadeDecoder(plan, L, B, Hq, Hkv, n)
        qs_, Ks_, Vs_ = t(q[:, :, g0 * G:g1 * G]), [t(K[l][:, g0:g1]) for l in range(L)], \
            [t(V[l][:, g0:g1]) for l in range(L)]
        if backend == "nccl":
            # the whole sharded step, NCCL all-gathers included, as one CUDA graph
            dec.capture(qs_, Ks_, Vs_, n).replay()
        else:
            dec.step(qs_, Ks_, Vs_, n)
        full = dec.gather_outputs().cpu().numpy()
        if rank == 0:
            ref = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
            want = ref.step(t(q), [t(K[l]) for l in range(L)], [t(V[l]) for l in range(L)], n).cpu().numpy()
            # the split-K factor follows the local (sequence, kv head) count,
            # so outputs agree to the bf16 rounding of P per split
            err = np.abs(full - want).max()
            assert err < 2e-3, f"sharded decode differs from unsharded by {err}"
            # the gathered lists of the last anchor ARE the unsharded lists
            assert torch.equal(dec.full_cnt, ref.counts)
            for b in range(B):
                for g in range(Hkv):
                    c = int(ref.counts[b, g])
                    assert torch.equal(dec.full_idx[b, g, :c], ref.indices[b, g, :c]), (b, g)
        # prefill: [L][H][N][d]
        N = 600
        Qp = orc.bf16_round(rng.standard_normal((L, Hq, N, 128)).astype(np.float32))
        Kp = orc.bf16_round(rng.standard_normal((L, Hkv, N, 128)).astype(np.float32))
        Vp = orc.bf16_round(rng.standard_normal((L, Hkv, N, 128)).astype(np.float32))
        pf = sharding.ShardedKascadePrefill(plan, L, Hq, Hkv, N)
        loc = pf.forward([t(Qp[l, g0 * G:g1 * G]) for l in range(L)], [t(Kp[l, g0:g1]) for l in range(L)],
                         [t(Vp[l, g0:g1]) for l in range(L)])
        allp = pf.gather_outputs().float().cpu().numpy()
        if rank == 0:
            ref = engine.KascadePrefill(plan, L, Hq, Hkv, N)
            want = ref.forward([t(Qp[l]) for l in range(L)], [t(Kp[l]) for l in range(L)],
                               [t(Vp[l]) for l in range(L)]).float().cpu().numpy()
            # every (head, tile) runs the same CTA program on the same inputs
            # with or without sharding: outputs and lists are bit-exact
            assert np.array_equal(allp, want), f"sharded prefill differs by {np.abs(allp - want).max()}"
            assert torch.equal(pf.full_cnt, ref.counts)
            assert torch.equal(pf.full_idx, ref.indices)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_kv_head_sharded_executors_match_unsharded(cuda_ok):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    msgs = []
    while not errq.empty():
        msgs.append(errq.get())
    assert not msgs, msgs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="NCCL across ranks needs >= 2 GPUs (NCCL rejects two ranks on one device)")
def test_kv_head_sharded_executors_nccl_two_gpus(cuda_ok):
    """The same check over NCCL on two GPUs, with the sharded decode step
    captured as one CUDA graph (kernels + index-list all-gathers)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq, "nccl")) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    msgs = []
    while not errq.empty():
        msgs.append(errq.get())
    assert not msgs, msgs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def _bench_worker(rank, world, port, errq):
    """bench.py's multi-GPU configs[4] path (sharded_70b) at toy sizes, two
    gloo ranks sharing cuda:0: it must run end to end and time on every rank."""
    import sys
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, repo)
        import bench
        from paper_2512_16391_b200.host_types import KBudgetPolicy, read_plan
        plan = read_plan(os.path.join(repo, "plans", "llama70b.json"))
        plan.k_policy = KBudgetPolicy(0.1, 64)
        out = bench.sharded_70b(torch.device("cuda", 0), world, dist, plan, 1024, 2, 2, 1, 7 + 97 * rank,
                                n_distinct_max=2)
        assert out["config"] == 4 and out["prefill_speedup_vs_dense"] > 0 and out["decode_speedup_vs_dense"] > 0, out
        assert "x2" in out["sharding"]
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_bench_sharded_70b_path_runs(cuda_ok):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
