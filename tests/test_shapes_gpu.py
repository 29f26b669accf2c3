"""Head-group shapes beyond the bench's GQA-4: MHA (G = 1), odd groups
(G = 3), G = 8, 16, 24 and 32 (MQA-style) through the decode and prefill executors, against
the oracle (decode_step / run_kascade) on the same bf16 inputs, with
non-identity head maps and ragged lengths.  Needs a B200."""
import numpy as np
import pytest

from oracle import kascade_oracle as orc
from parity import assert_outputs_close

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# G = 24 and 32 exceed the decode kernel's 16-row MMA tile and run as 2
# virtual kv heads per kv head (kscd_internal.h DecodeArgs.kv_rep)
SHAPES = [(2, 2), (6, 2), (8, 1), (16, 1), (12, 4), (32, 1), (48, 2)]


def _maps(Hkv):
    """A non-identity map for layer 1 (a reuse layer) when Hkv > 1."""
    return list(reversed(range(Hkv)))


@pytest.mark.parametrize("Hq,Hkv", SHAPES)
def test_decode_engine_head_groups(cuda_ok, Hq, Hkv):
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, B, n = 3, 2, 1531
    rng = np.random.default_rng(Hq * 31 + Hkv)
    hm = _maps(Hkv)
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, hm)},
                      k_policy=KBudgetPolicy(0.1, 16))
    q = orc.bf16_round((rng.standard_normal((L, B, Hq, 128)) * 2.5).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((L, B, Hkv, n, 128)).astype(np.float32))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)  # noqa: E731
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n)
    out = dec.step(dev(q), [dev(K[l]) for l in range(L)], [dev(V[l]) for l in range(L)], n).cpu().numpy()
    for b in range(B):
        Y, _, _ = orc.decode_step(q[:, b], K[:, b], V[:, b], [0, 2], {1: hm}, 0.1, 16, want_mass=False)
        assert_outputs_close(out[:, b], Y)


@pytest.mark.parametrize("Hq,Hkv", SHAPES)
def test_prefill_engine_head_groups(cuda_ok, Hq, Hkv):
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, N = 3, 601
    rng = np.random.default_rng(Hq * 17 + Hkv)
    hm = _maps(Hkv)
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, hm)},
                      k_policy=KBudgetPolicy(0.2, 32), tile_size=128)
    Q = orc.bf16_round((rng.standard_normal((L, Hq, N, 128)) * 2.0).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((L, Hkv, N, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((L, Hkv, N, 128)).astype(np.float32))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)  # noqa: E731
    eng = engine.KascadePrefill(plan, L, Hq, Hkv, N)
    out = eng.forward([dev(Q[l]) for l in range(L)], [dev(K[l]) for l in range(L)],
                      [dev(V[l]) for l in range(L)]).float().cpu().numpy()
    want, _ = orc.run_kascade(Q, K, V, [0, 2], {1: hm}, 0.2, 32, tile_size=128)
    assert_outputs_close(out, want)


def test_decode_engine_ragged_batch(cuda_ok):
    """Serving batches hold sequences of different lengths: seq_lens[b]
    bounds sequence b's keys and its k_budget.  Each sequence equals the
    oracle's decode step over its own prefix; a captured graph reads the
    lengths at replay time."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, Hq, Hkv, n_cap = 3, 8, 2, 1600
    lens = [1531, 977, 64, 1]
    B = len(lens)
    rng = np.random.default_rng(41)
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, [1, 0])},
                      k_policy=KBudgetPolicy(0.1, 16))
    q = orc.bf16_round((rng.standard_normal((L, B, Hq, 128)) * 2.5).astype(np.float32))
    K = orc.bf16_round(rng.standard_normal((L, B, Hkv, n_cap, 128)).astype(np.float32))
    V = orc.bf16_round(rng.standard_normal((L, B, Hkv, n_cap, 128)).astype(np.float32))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)  # noqa: E731
    qd, Kd, Vd = dev(q), [dev(K[l]) for l in range(L)], [dev(V[l]) for l in range(L)]
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n_cap)
    out = dec.step(qd, Kd, Vd, max(lens), seq_lens=sl).cpu().numpy()

    def check(out, lens):
        for b, n in enumerate(lens):
            Y, _, _ = orc.decode_step(q[:, b], K[:, b, :, :n], V[:, b, :, :n], [0, 2], {1: [1, 0]}, 0.1, 16,
                                      want_mass=False)
            assert_outputs_close(out[:, b], Y)
            k = orc.k_budget(0.1, 16, n)
            assert (dec.counts[b].cpu().numpy() == k).all()

    check(out, lens)
    # a graph reads the lengths at replay: new lengths up to the captured
    # seq_len (which bounds every sequence) need no recapture
    g = dec.capture(qd, Kd, Vd, n_cap, seq_lens=sl)
    lens2 = [700, 1600, 5, 1200]
    sl.copy_(torch.tensor(lens2, dtype=torch.int32))
    g.replay()
    torch.cuda.synchronize()
    check(dec.out.cpu().numpy(), lens2)


def test_host_step_graph_ragged_batch(cuda_ok):
    """capture_host_step with seq_lens: every sequence's new K/V rows land at
    its own seq_lens[b] - 1, and the outputs equal appending by hand and
    running the ragged eager step."""
    from paper_2512_16391_b200 import engine
    from paper_2512_16391_b200.host_types import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy
    L, Hq, Hkv, n_cap = 3, 8, 2, 900
    lens = [700, 33, 899]
    B = len(lens)
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps={1: HeadMap(1, 0, [1, 0])},
                      k_policy=KBudgetPolicy(0.1, 16))
    g = torch.Generator(device="cuda").manual_seed(9)
    Ks = [torch.randn(B, Hkv, n_cap, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    Vs = [torch.randn(B, Hkv, n_cap, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
    Kr, Vr = [x.clone() for x in Ks], [x.clone() for x in Vs]
    q_host = torch.randn(L, B, Hq, 128).to(torch.bfloat16).pin_memory()
    kv_host = torch.randn(L, 2, B, Hkv, 128).to(torch.bfloat16).pin_memory()
    out_host = torch.zeros(L, B, Hq, 128).pin_memory()
    sl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    dec = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n_cap)
    q = torch.empty(L, B, Hq, 128, dtype=torch.bfloat16, device="cuda")
    graph = dec.capture_host_step(q_host, kv_host, out_host, q, Ks, Vs, n_cap, seq_lens=sl)
    for l in range(L):                       # the capture's warm-up run appended once; restore
        Ks[l].copy_(Kr[l])
        Vs[l].copy_(Vr[l])
    out_host.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for l in range(L):
        for b, n in enumerate(lens):
            assert torch.equal(Ks[l][b, :, n - 1].cpu(), kv_host[l, 0, b])
            assert torch.equal(Vs[l][b, :, n - 1].cpu(), kv_host[l, 1, b])
            Kr[l][b, :, n - 1] = kv_host[l, 0, b].cuda()
            Vr[l][b, :, n - 1] = kv_host[l, 1, b].cuda()
        assert torch.equal(Ks[l], Kr[l]) and torch.equal(Vs[l], Vr[l])
    ref = engine.KascadeDecoder(plan, L, B, Hq, Hkv, n_cap)
    want = ref.step(q_host.cuda(), Kr, Vr, n_cap, seq_lens=sl).cpu()
    assert torch.equal(out_host, want)
