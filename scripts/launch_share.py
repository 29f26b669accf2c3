"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
of a bench.py run: per-kernel launch counts and mean durations, and the
share of the reuse-layer sparse decode kernel in one composed Kascade decode
step (cold-cache, serialised times -- compare the SHARE with bench.py's
event-timed step, not the absolute).  python scripts/launch_share.py list.csv"""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    name = name.replace("(int)", "").replace("(bool)", "")
    m = re.match(r"(?:void )?(?:kscd::)?([A-Za-z0-9_]+)(<[^()]*>)?", name)
    if not m:
        return name[:60]
    base = m.group(1)
    if base.startswith(("decode_attn", "decode_tc", "prefill_attn", "topk", "pool", "append", "probs", "pool_rows")):
        return base + (m.group(2) or "")
    return "torch/other: " + base[:40]


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
        rows.append((short(r["Kernel Name"]), r["Grid Size"], float(r["Metric Value"].replace(",", "")) * scale))
    agg = collections.OrderedDict()
    for name, grid, us in rows:
        key = (name, grid)
        c, t = agg.get(key, (0, 0.0))
        agg[key] = (c + 1, t + us)
    total = sum(t for _, t in agg.values())
    print(f"{len(rows)} launches, {total / 1e3:.1f} ms total kernel time")
    print(f"{'kernel':44s} {'grid':>16s} {'count':>6s} {'mean us':>10s} {'total ms':>10s} {'share':>6s}")
    for (name, grid), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:44s} {grid:>16s} {c:6d} {t / c:10.1f} {t / 1e3:10.2f} {t / total:6.1%}")

    def mean(prefix, grid=None):
        hits = [(c, t) for (n, g), (c, t) in agg.items() if n.startswith(prefix) and (grid is None or g == grid)]
        c = sum(h[0] for h in hits)
        return sum(h[1] for h in hits) / c if c else float("nan")

    def by_grid(prefix, grid):
        return mean(prefix, grid)

    # composed 32-layer step of bench.py's default plan (anchors 0, 2, 8, 13,
    # 14; 16 launches): layer 0 dense + scores, 3 score launches (groups [2],
    # [8], [13, 14]), 4 + 1 pooling and Top-k launches, and the sparse
    # launches (reuse layer 1; groups with their reuse runs 2-7, 8-12, 13-31)
    dense0 = by_grid("decode_tc_kernel<0, 4>", "(1214, 1, 1)")
    score1 = by_grid("decode_tc_kernel<2, 4>", "(1214, 1, 1)")
    score2 = by_grid("decode_tc_kernel<2, 4>", "(2428, 1, 1)")
    pool1, pool2 = by_grid("pool_decode", "(128, 8, 8)"), by_grid("pool_decode", "(128, 8, 16)")
    topk1, topk2 = by_grid("topk_kernel<4>", "(256, 1, 1)"), by_grid("topk_kernel<4>", "(512, 1, 1)")
    sp = {g: by_grid("decode_attn_kernel<0>", g) for g in ("(9, 8, 8)", "(9, 8, 48)", "(9, 8, 40)", "(9, 8, 152)")}
    select = 3 * (pool1 + topk1) + pool2 + topk2
    sparse = sum(sp.values())
    step = dense0 + 2 * score1 + score2 + select + sparse
    print(f"\ncomposed decode step (ncu, serialised, cold caches): {step:.0f} us = dense0 {dense0:.0f} + score passes "
          f"{2 * score1 + score2:.0f} + selections {select:.0f} + sparse launches {sparse:.0f} "
          f"(longest run, layers 13-31: {sp['(9, 8, 152)']:.0f})")
    print(f"shares: sparse {sparse / step:.1%}, dense + score passes {(dense0 + 2 * score1 + score2) / step:.1%}, "
          f"selections {select / step:.1%} (overlapped with the attention on a side stream in the step)")


if __name__ == "__main__":
    main()
