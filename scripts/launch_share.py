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
    m = re.match(r"(?:void )?(?:kscd::)?([A-Za-z0-9_]+)(<[^()]*>)?", name)
    if not m:
        return name[:60]
    base = m.group(1)
    if base.startswith(("decode_attn", "prefill_attn", "topk", "pool", "append", "probs", "pool_rows")):
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

    # composed 32-layer step of bench.py's default plan: 27 reuse + 4 anchors
    # (scores, pool, top-k, sparse) + anchor 0 (dense with scores, pool, top-k)
    sparse = mean("decode_attn_kernel<1")
    scores = mean("decode_attn_kernel<2")
    dense = mean("decode_attn_kernel<0")
    pool = mean("pool_decode")
    topk = mean("topk_kernel<4")   # decode rows run as 4-CTA clusters
    step = 27 * sparse + 4 * (scores + pool + topk + sparse) + (dense + pool + topk)
    print(f"\ncomposed decode step (ncu, serialised): {step:.0f} us; reuse sparse_decode {sparse:.1f} us/launch, "
          f"27 launches = {27 * sparse / step:.1%} of the step; all sparse_decode = {31 * sparse / step:.1%}")


if __name__ == "__main__":
    main()
