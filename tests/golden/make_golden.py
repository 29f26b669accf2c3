"""Freeze golden vectors from the REFERENCE implementation itself.

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src,
runs its own public functions (and its private runner seams
``_anchor_selections`` / ``_routed_selections`` where a single tile is
needed) on seeded, bf16-representable inputs, and writes small fixtures next
to this script.  ``tests/test_oracle_golden.py`` pins the CPU oracle to them
and the GPU parity tests compare the CUDA path against them.  Nothing here
runs on the GPU box.
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import kascade as ref  # noqa: E402  (the reference package)
from kascade import runner as ref_runner  # noqa: E402
from kascade.tiles import Tile, TileSpec  # noqa: E402

from oracle import kascade_oracle as orc  # noqa: E402


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def trace_of(Q, K, V, pid="golden"):
    L, Hq, N, d = Q.shape
    return ref.AttentionTrace(num_layers=L, num_query_heads=Hq, num_kv_heads=K.shape[1],
                              head_dim=d, seq_len=N, Q=Q, K=K, V=V, prompt_id=pid)


def bf16_trace_random(seed, L, Hq, Hkv, d, N):
    Q, K, V = orc.random_qkv(seed, L, Hq, Hkv, d, N)
    return [orc.bf16_round(x) for x in (Q, K, V)]


def sels_to_arrays(sels, Hkv, tids):
    """dict (g, tid) -> TopKIndexSet  ==>  int32 [Hkv][T][kmax] padded with -1 + counts."""
    kmax = max(len(sels[(g, t)].indices) for g in range(Hkv) for t in tids)
    idx = np.full((Hkv, len(tids), kmax), -1, np.int32)
    cnt = np.zeros((Hkv, len(tids)), np.int32)
    for g in range(Hkv):
        for i, t in enumerate(tids):
            s = sels[(g, t)].indices
            idx[g, i, :len(s)] = s
            cnt[g, i] = len(s)
    return idx, cnt


def main():
    meta = {"reference": "kascade " + ref.__version__, "numpy": np.__version__}

    # 1. generator pins (traceio.py:218-296 vs oracle.synth_qkv)
    gens = {
        "conformance": dict(L=2, Hq=2, Hkv=1, d=4, N=3, seed=42, rho=0.5),
        "config1": dict(L=4, Hq=8, Hkv=2, d=128, N=2048, seed=0, rho=0.95),
        "permuted": dict(L=3, Hq=8, Hkv=4, d=16, N=64, seed=26, rho=1.0,
                         perms=[[0, 1, 2, 3], [2, 0, 3, 1], [2, 0, 3, 1]]),
    }
    meta["synth_sha256"] = {}
    for name, c in gens.items():
        cfg = ref.SynthConfig(num_layers=c["L"], num_query_heads=c["Hq"], num_kv_heads=c["Hkv"],
                              head_dim=c["d"], seq_len=c["N"], seed=c["seed"],
                              layer_correlation=c["rho"], head_permutations=c.get("perms"))
        t = ref.generate_synthetic(cfg)
        meta["synth_sha256"][name] = {"args": c, "sha256": sha(t.Q, t.K, t.V)}

    # 2. Top-k contract (attention.py:147-174)
    rng = np.random.default_rng(5)
    vecs = [rng.random(64), np.full(16, 0.25), np.array([0.2, 0.8]),
            np.round(rng.random(300) * 8) / 8, np.zeros(40), rng.random(5000).astype(np.float32)]
    ks = [8, 2, 5, 37, 7, 499]
    topk = {}
    for i, (v, k) in enumerate(zip(vecs, ks)):
        topk[f"w{i}"] = np.asarray(v, np.float64)
        topk[f"k{i}"] = np.array(k)
        topk[f"idx{i}"] = ref.oracle_topk_indices(v, k).indices
    np.savez_compressed(os.path.join(HERE, "topk.npz"), n=len(vecs), **topk)

    # 3. dense attention (attention.py:106-144), causal and not
    Q, K, V = bf16_trace_random(3, 1, 4, 2, 128, 96)
    t = trace_of(Q, K, V)
    P, Y = ref.dense_attention(t, 0)
    Pn, Yn = ref.dense_attention(t, 0, causal=False)
    np.savez_compressed(os.path.join(HERE, "dense_small.npz"), Q=orc.bf16_bits(Q), K=orc.bf16_bits(K),
                        V=orc.bf16_bits(V), P=P, Y=Y, Pn=Pn, Yn=Yn)

    # 4. sparse attention with fallback rows (attention.py:185-253)
    Q, K, V = bf16_trace_random(11, 1, 4, 2, 128, 72)
    t = trace_of(Q, K, V)
    tiles = ref.make_tiles(72, "prefill", 4, 2, tile_size=16)
    P, _ = ref.dense_attention(t, 0)
    core = ref.AnchorPlanCore(anchors=[0], budget=1, objective_value=0.0)
    plan = ref.AnchorPlan(core=core, k_policy=ref.KBudgetPolicy(fraction=0.25, k_min=4), tile_size=16)
    sels = ref_runner._anchor_selections(t, 0, P, tiles, plan)
    res = ref.topk_attention(t, 0, sels, tiles, dense_P=P)
    tids = sorted({tl.tile_id for tl in tiles.tiles})
    idx, cnt = sels_to_arrays(sels, 2, tids)
    fb = np.array(sorted(res.fallback_rows), np.int32).reshape(-1, 2)
    # hand-made sets whose first keys sit late in the tile: early rows of
    # tile 0 see nothing and take the diagonal fallback (attention.py:248-252)
    hand = {}
    for tl in tiles.tiles:
        s, e = tl.start, tl.end
        keys = [e - 3, e - 2, e - 1] if tl.tile_id == 0 else sorted({5 + tl.kv_head, s + 2, e - 1})
        hand[(tl.kv_head, tl.tile_id)] = ref.TopKIndexSet(tl.kv_head, tl.tile_id, np.array(keys), len(keys))
    res2 = ref.topk_attention(t, 0, hand, tiles, dense_P=P)
    idx2, cnt2 = sels_to_arrays(hand, 2, tids)
    fb2 = np.array(sorted(res2.fallback_rows), np.int32).reshape(-1, 2)
    np.savez_compressed(os.path.join(HERE, "sparse_small.npz"), Q=orc.bf16_bits(Q), K=orc.bf16_bits(K),
                        V=orc.bf16_bits(V), idx=idx, cnt=cnt, Y=res.Y, mass=res.mass_recovered,
                        fallback=fb, tile=np.array(16), fraction=np.array(0.25), k_min=np.array(4),
                        idx2=idx2, cnt2=cnt2, Y2=res2.Y, mass2=res2.mass_recovered, fallback2=fb2)

    # 5. full run_kascade prefill on a head-permuted heavy-tailed trace
    #    (remapped head maps are non-identity, so the gather crosses heads)
    cfg = ref.SynthConfig(num_layers=4, num_query_heads=4, num_kv_heads=2, head_dim=128, seq_len=256,
                          seed=7, layer_correlation=0.95, head_permutations=[[0, 1], [1, 0], [1, 0], [0, 1]])
    g = ref.generate_synthetic(cfg)
    Q, K, V = (orc.bf16_round(x) for x in (g.Q, g.K, g.V))
    t = trace_of(Q, K, V)
    anchors = [0, 2]
    maps = ref.compute_head_maps(t, anchors, k=16)
    core = ref.AnchorPlanCore(anchors=anchors, budget=2, objective_value=0.0)
    plan = ref.AnchorPlan(core=core, head_maps=maps, k_policy=ref.KBudgetPolicy(fraction=0.1, k_min=16),
                          tile_size=64)
    outs, rep = ref.run_kascade(t, plan)
    hm = np.array([maps[l].map if l in maps else [-1, -1] for l in range(4)], np.int32)
    np.savez_compressed(os.path.join(HERE, "kascade_prefill.npz"), Q=orc.bf16_bits(Q), K=orc.bf16_bits(K),
                        V=orc.bf16_bits(V), outs=outs, head_maps=hm, anchors=np.array(anchors),
                        tile=np.array(64), fraction=np.array(0.1), k_min=np.array(16),
                        rel=np.array([r.output_rel_err_l2 for r in rep.per_layer]),
                        mass=np.array([r.mass_recovered_mean for r in rep.per_layer]),
                        fallback=np.array([r.fallback_rows for r in rep.per_layer]))

    # 6. pooling / mode variants: pre-softmax pooling and all-heads-pooled
    Q, K, V = bf16_trace_random(27, 3, 4, 2, 128, 64)
    t = trace_of(Q, K, V)
    core = ref.AnchorPlanCore(anchors=[0, 1], budget=2, objective_value=0.0)
    var = {"Q": orc.bf16_bits(Q), "K": orc.bf16_bits(K), "V": orc.bf16_bits(V)}
    pol = ref.KBudgetPolicy(fraction=0.5, k_min=4)
    plan = ref.AnchorPlan(core=core, mode="all_heads_pooled", k_policy=pol, tile_size=16)
    var["outs_allheads"], _ = ref.run_kascade(t, plan)
    maps = {2: ref.identity_head_map(2, reuse_layer=2, anchor_layer=1)}
    plan = ref.AnchorPlan(core=core, head_maps=maps, pooling="pre", k_policy=pol, tile_size=16)
    var["outs_pre"], _ = ref.run_kascade(t, plan)
    np.savez_compressed(os.path.join(HERE, "variants.npz"), **var)

    # 7. config 1 (BASELINE.json configs[0]): 4 layers, 8Q/2KV, d=128, N=2048,
    #    anchors {0,2}, k=10% (k_min 128).  Decode: reference run_kascade in
    #    decode phase, last token's row; prefill: last tile rows + all sets.
    c1 = gens["config1"]
    Q, K, V = orc.synth_qkv(c1["L"], c1["Hq"], c1["Hkv"], c1["d"], c1["N"], seed=c1["seed"], rho=c1["rho"])
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    t = trace_of(Q, K, V, "config1")
    anchors = [0, 2]
    maps = ref.compute_head_maps(t, anchors, k=64)
    core = ref.AnchorPlanCore(anchors=anchors, budget=2, objective_value=0.0)
    plan = ref.AnchorPlan(core=core, head_maps=maps, k_policy=ref.KBudgetPolicy(0.1, 128), tile_size=128)
    hm = np.array([maps[l].map if l in maps else [-1, -1] for l in range(4)], np.int32)
    outs_d, rep_d = ref.run_kascade(t, plan, phase="decode")
    N = c1["N"]
    last = TileSpec(phase="decode", tile_size=4,
                    tiles=[Tile(start=N - 1, end=N, kv_head=gg, tile_id=N - 1) for gg in range(2)])
    dec_sel = np.zeros((4, 2, ref.k_budget(plan.k_policy, N)), np.int32)
    cur = None
    for l in range(4):
        if l in anchors:
            P, _ = ref.dense_attention(t, l)
            cur = ref_runner._anchor_selections(t, l, P, last, plan)
            s = cur
        else:
            s = ref_runner._routed_selections(cur, maps[l], 2)
        for gg in range(2):
            dec_sel[l, gg] = s[(gg, N - 1)].indices
    outs_p, rep_p = ref.run_kascade(t, plan, phase="prefill")
    tiles = ref.make_tiles(N, "prefill", 8, 2, 128)
    pre_idx = []
    for a in anchors:
        P, _ = ref.dense_attention(t, a)
        sels = ref_runner._anchor_selections(t, a, P, tiles, plan)
        idx, cnt = sels_to_arrays(sels, 2, list(range(N // 128)))
        pre_idx.append(idx)
    np.savez_compressed(os.path.join(HERE, "config1.npz"), head_maps=hm, anchors=np.array(anchors),
                        dec_Y=outs_d[:, :, -1], dec_sel=dec_sel,
                        dec_rel=np.array([r.output_rel_err_l2 for r in rep_d.per_layer]),
                        dec_mass=np.array([r.mass_recovered_mean for r in rep_d.per_layer]),
                        pre_last_tile=outs_p[:, :, N - 128:], pre_idx=np.stack(pre_idx),
                        pre_rel=np.array([r.output_rel_err_l2 for r in rep_p.per_layer]),
                        pre_mass=np.array([r.mass_recovered_mean for r in rep_p.per_layer]))

    # 8. trace I/O and the `run` CLI (traceio.py:44-156, cli.py:216-233).
    #    conformance_v1.kscd is the reference's own conformance trace
    #    (test_traceio.py:39-40 pins its sha256); the CLI cases run the
    #    reference `kascade run` on traces written by the reference writer and
    #    freeze its report JSON and stdout.  The GPU tests regenerate the same
    #    trace bytes with the oracle generator + our writer (sha-checked).
    import contextlib
    import io
    import tempfile
    from kascade import cli as ref_cli
    from kascade import traceio as ref_io
    cfg = ref.SynthConfig(num_layers=2, num_query_heads=2, num_kv_heads=1, head_dim=4, seq_len=3, seed=42,
                          layer_correlation=0.5, include_xy=True, prompt_id="conformance-v1")
    conf = os.path.join(HERE, "conformance_v1.kscd")
    ref_io.write_trace(conf, ref.generate_synthetic(cfg))
    with open(conf, "rb") as f:
        meta["conformance_sha256"] = hashlib.sha256(f.read()).hexdigest()
    # format-error messages and offsets of the reference reader on corrupted copies
    with open(conf, "rb") as f:
        good = f.read()
    corrupt = {"magic": b"NOPE" + good[4:], "version": good[:4] + (999).to_bytes(2, "little") + good[6:],
               "dtype": good[:26] + bytes([7]) + good[27:], "truncated": good[:-5], "header": b"KSCD\x01",
               "trailing": good + b"xx", "heads": good[:10] + (3).to_bytes(4, "little") + good[14:],
               "zero_dim": good[:6] + (0).to_bytes(4, "little") + good[10:],
               "prompt_utf8": good[:28] + b"\xff" + good[29:]}
    errs = {}
    with tempfile.TemporaryDirectory() as td:
        for name, blob in corrupt.items():
            p = os.path.join(td, name + ".kscd")
            with open(p, "wb") as f:
                f.write(blob)
            try:
                ref_io.read_trace(p)
                errs[name] = None
            except ref.FormatError as e:
                errs[name] = {"message": str(e), "offset": e.offset}
        cli_cases = {}
        c = dict(L=4, Hq=8, Hkv=2, d=128, N=512, seed=3, rho=0.9, perms=[[0, 1], [1, 0], [1, 0], [0, 1]])
        g = ref.generate_synthetic(ref.SynthConfig(num_layers=c["L"], num_query_heads=c["Hq"],
                                                   num_kv_heads=c["Hkv"], head_dim=c["d"], seq_len=c["N"],
                                                   seed=c["seed"], layer_correlation=c["rho"],
                                                   head_permutations=c["perms"], prompt_id="cli-small"))
        t = trace_of(*(orc.bf16_round(x) for x in (g.Q, g.K, g.V)), pid="cli-small")
        tpath = os.path.join(td, "t.kscd")
        ref_io.write_trace(tpath, t)
        with open(tpath, "rb") as f:
            trace_sha = hashlib.sha256(f.read()).hexdigest()
        anchors = [0, 2]
        maps = ref.compute_head_maps(t, anchors, k=32)
        for tile in (128, 32):
            core = ref.AnchorPlanCore(anchors=anchors, budget=2, objective_value=0.0)
            plan = ref.AnchorPlan(core=core, head_maps=maps, k_policy=ref.KBudgetPolicy(0.1, 16), tile_size=tile)
            ppath = os.path.join(HERE, f"cli_plan_t{tile}.json")
            ref_io.write_plan(ppath, plan)
            for phase, mode in (("prefill", None), ("prefill", "all-heads-pooled"), ("decode", None)):
                if tile == 32 and mode is not None:
                    continue
                rpath = os.path.join(td, "r.json")
                argv = ["run", "--trace", tpath, "--plan", ppath, "--phase", phase, "--out", rpath]
                if mode:
                    argv += ["--mode", mode]
                buf = io.StringIO()
                with contextlib.redirect_stdout(buf):
                    code = ref_cli.main(argv)
                with open(rpath) as f:
                    rep = json.load(f)
                cli_cases[f"t{tile}_{phase}_{mode or 'remapped'}"] = {
                    "plan": os.path.basename(ppath), "phase": phase, "mode": mode, "exit": code,
                    "report": rep, "stdout": buf.getvalue()}
    with open(os.path.join(HERE, "cli_cases.json"), "w") as f:
        json.dump({"trace_args": c, "trace_prompt_id": "cli-small", "trace_sha256": trace_sha,
                   "format_errors": errs, "cases": cli_cases}, f, indent=1, sort_keys=True)
        f.write("\n")

    # 9. offline calibration: head similarity and head
    #    maps (heads.py:67-143, pipeline.py:31-73) and the layer similarity
    #    matrix in both modes (metrics.py:205-335), on the kascade_prefill
    #    trace (section 5) and on config 1 (section 7).
    import time
    from kascade import metrics as ref_metrics
    from kascade import heads as ref_heads
    z5 = np.load(os.path.join(HERE, "kascade_prefill.npz"))
    tA = trace_of(*(orc.from_bf16_bits(z5[n]) for n in ("Q", "K", "V")))
    cal = {}
    for agg in ("mean", "min"):
        for a, b in ((0, 1), (0, 3), (2, 3), (1, 1)):
            cal[f"hs_{agg}_{a}_{b}"] = ref_heads.head_similarity(tA, a, b, k=16, token_agg=agg)
        for mode, extra in (("planning", dict(tile_size=64)), ("diagnostic", {})):
            S = ref_metrics.similarity_matrix(tA, k=16, token_agg=agg, mode=mode, **extra)
            cal[f"S_{mode}_{agg}"] = S.S
            cal[f"und_{mode}_{agg}"] = np.array(S.undefined_scores)
    S = ref_metrics.similarity_matrix(tA, k=16, token_agg="min", mode="planning", tile_size=64, phase="decode")
    cal["S_planning_decode_min"], cal["und_planning_decode_min"] = S.S, np.array(S.undefined_scores)
    maps = ref.compute_head_maps(tA, [0, 2], k=16)
    cal["maps_A"] = np.array([maps[l].map if l in maps else [-1, -1] for l in range(4)], np.int32)
    # config 1: the BASELINE planning pass (k=64, tile 128, min over tiles)
    t1 = trace_of(*(orc.bf16_round(x) for x in orc.synth_qkv(c1["L"], c1["Hq"], c1["Hkv"], c1["d"], c1["N"],
                                                             seed=c1["seed"], rho=c1["rho"])), "config1")
    t0 = time.perf_counter()
    S1 = ref_metrics.similarity_matrix(t1, k=64, token_agg="min", mode="planning", tile_size=128)
    meta["ref_seconds_config1_planning_matrix"] = round(time.perf_counter() - t0, 2)
    t0 = time.perf_counter()
    maps1 = ref.compute_head_maps(t1, [0, 2], k=64)
    meta["ref_seconds_config1_head_maps"] = round(time.perf_counter() - t0, 2)
    cal["S1_planning_min"], cal["und1"] = S1.S, np.array(S1.undefined_scores)
    cal["maps1"] = np.array([maps1[l].map if l in maps1 else [-1, -1] for l in range(4)], np.int32)
    cal["hs1_0_1"] = ref_heads.head_similarity(t1, 0, 1, k=64)
    np.savez_compressed(os.path.join(HERE, "calibration.npz"), **cal)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
        f.write("\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
