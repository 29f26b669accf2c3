"""Per-kernel instruction summary of the built library (cuobjdump -sass):
the Blackwell tensor-core / TMEM / TMA / async-copy mnemonics that show
which hardware path each kernel uses, plus the register and shared-memory
footprint (cuobjdump -res-usage).  No GPU needed.

    python scripts/sass_summary.py > profiles/sass_summary_r02.txt
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2512_16391_b200", "libkascade_b200.so")
GROUPS = [
    ("UTCHMMA", "tcgen05.mma kind::f16 (5th-gen tensor core)"),
    ("UTCBAR", "tcgen05.commit -> mbarrier"),
    ("LDTM", "tcgen05.ld (TMEM -> registers)"),
    ("STTM", "tcgen05.st (registers -> TMEM)"),
    ("UTMALDG", "TMA tensor load (cp.async.bulk.tensor)"),
    ("HMMA", "mma.sync (warp-level tensor core)"),
    ("LDGSTS", "cp.async (global -> shared)"),
    ("MUFU.EX2", "MUFU exp2"),
    ("ATOMS", "shared-memory atomics"),
    ("SYNCS", "mbarrier ops"),
    ("UCGABAR", "cluster barrier"),
]


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
        if m and cur:
            usage[cur] = (int(m.group(1)), int(m.group(2)))
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for key, _ in GROUPS:
                if op.startswith(key):
                    counts[cur][key] += 1
            counts[cur]["_total"] += 1
    names = list(counts)
    pretty = dict(zip(names, demangle(names)))
    print(f"# SASS summary of {os.path.basename(lib)} (cuobjdump -sass / -res-usage, sm_100a)")
    print("# columns: static instruction counts per kernel")
    for key, what in GROUPS:
        print(f"#   {key:9s} {what}")
    hdr = ["kernel", "regs", "smem"] + [k for k, _ in GROUPS] + ["total"]
    print("\t".join(hdr))
    for n in names:
        c = counts[n]
        reg, shm = usage.get(n, ("?", "?"))
        print("\t".join([pretty[n], str(reg), str(shm)] + [str(c[k]) for k, _ in GROUPS] + [str(c["_total"])]))


if __name__ == "__main__":
    main()
