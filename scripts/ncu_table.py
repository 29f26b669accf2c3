"""One markdown row per kernel launch of an ncu report (dev tool):
python scripts/ncu_table.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %pk"),
        ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
        ("sm__cycles_elapsed.avg.per_second", "SM clk"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs")]


def scale(v, u):
    x = float(v.replace(",", ""))
    return x * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                "Gbyte": 1e9}.get(u, 1.0)


def main():
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM GB/s |")
    print("|---" * (len(COLS) + 2) + "|")
    for rep in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("kscd::", "")
            t_us = scale(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
            rd = scale(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
            wr = scale(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
            cells = []
            for k, _ in COLS:
                if k == "gpu__time_duration.sum":
                    cells.append(f"{t_us:.1f} us")
                elif k.startswith("dram__bytes"):
                    cells.append(f"{scale(d[k], u[k]) / 1e6:.1f} MB")
                elif k == "sm__cycles_elapsed.avg.per_second":
                    cells.append(f"{scale(d[k], u[k]) / 1e9 if u[k] == 'hz' else float(d[k]):.2f} {'' if u[k] == 'hz' else u[k]}".strip())
                else:
                    cells.append(d.get(k, "-"))
            print(f"| `{name}` | " + " | ".join(cells) + f" | {(rd + wr) / (t_us * 1e-6) / 1e9:.0f} |")


if __name__ == "__main__":
    main()
