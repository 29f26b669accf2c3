"""Parity comparators.

* outputs: max-abs <= 2e-2 and mean-abs <= 1e-3 against the reference's fp32
  output on identical (bf16-representable) inputs; rel-L2 reported.  Outputs
  of magnitude ~1 (heavy-tailed synthetic traces) use the magnitude-relative
  form (assert_outputs_close_rel): bf16 output rounding alone is 2^-9 of |O|.
* Top-k sets: equal, except that every element of the symmetric difference
  must carry a reference pooled score within 1e-5 relative of the reference
  k-th largest score (a documented fp32 near-tie).  The swap count is
  returned so tests can report / bound it.
* head-map and gather indices: bit-exact (plain equality).
"""

import numpy as np

OUT_MAX_ABS = 2e-2
OUT_MEAN_ABS = 1e-3
TIE_REL = 1e-5


def assert_outputs_close(got, ref, max_abs=OUT_MAX_ABS, mean_abs=OUT_MEAN_ABS, what="output"):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    err = np.abs(got - ref)
    rel = np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-30)
    assert err.max() <= max_abs, f"{what}: max-abs {err.max():.3e} > {max_abs} (rel-L2 {rel:.2e})"
    assert err.mean() <= mean_abs, f"{what}: mean-abs {err.mean():.3e} > {mean_abs} (rel-L2 {rel:.2e})"
    return float(err.max()), float(err.mean()), float(rel)


def assert_outputs_close_rel(got, ref, rel_l2=5e-3, what="output"):
    """For outputs of magnitude ~1 (heavy-tailed synthetic traces), where the
    bf16 OUTPUT rounding alone is 2^-9 of |O|: max-abs 2e-2 plus 8e-3 of the
    reference magnitude per element, and rel-L2 below ``rel_l2``."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    err = np.abs(got - ref)
    worst = float((err - 8e-3 * np.abs(ref)).max())
    rel = float(np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-30))
    assert worst <= 2e-2, f"{what}: error {worst:.3e} above 2e-2 + 8e-3|ref| (rel-L2 {rel:.2e})"
    assert rel < rel_l2, f"{what}: rel-L2 {rel:.2e} >= {rel_l2}"
    return rel


def topk_swaps(got, ref, ref_scores, rel=TIE_REL):
    """Number of near-tie swaps between two sorted index sets; raises if a
    differing element is not a near-tie of the reference k-th score."""
    got = np.asarray(got, dtype=np.int64)
    ref = np.asarray(ref, dtype=np.int64)
    assert got.size == ref.size, f"set sizes differ: {got.size} vs {ref.size}"
    assert (np.diff(got) > 0).all(), "indices not strictly ascending"
    diff = np.setxor1d(got, ref)
    if diff.size == 0:
        return 0
    s = np.asarray(ref_scores, dtype=np.float64)
    kth = np.sort(s[ref])[0]
    bad = [int(j) for j in diff if abs(s[j] - kth) > rel * abs(kth)]
    assert not bad, f"{len(bad)} non-tie differences, e.g. {bad[:5]} (k-th score {kth:.9g})"
    return diff.size // 2
