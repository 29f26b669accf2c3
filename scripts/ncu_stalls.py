"""Per-instruction warp-stall summary of an ncu report's SASS source page (dev tool).
python scripts/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    body = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = Counter()
    op_samples = Counter()
    for r in body:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        op_samples[op.split(".")[0]] += s
        for c in stall_cols:
            tot[c] += int(float(r[c] or 0))
    n = sum(tot.values())
    print(f"total samples {n}")
    for c, v in tot.most_common(12):
        print(f"  {c:28s} {v:8d} {100 * v / max(n, 1):5.1f}%")
    print("samples by opcode:")
    for op, v in op_samples.most_common(15):
        print(f"  {op:20s} {v:8d} {100 * v / max(n, 1):5.1f}%")
    print("hottest instructions:")
    body.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in body[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        st = sorted(((int(float(r[c] or 0)), c) for c in stall_cols), reverse=True)[:2]
        print(f"  {r['Address']:>6s} {s:6d}  {r['Source'][:60]:60s} {st[0][1]}={st[0][0]} {st[1][1]}={st[1][0]}")


if __name__ == "__main__":
    main()
