"""Summarise an ncu --set full report into a few lines (dev tool; the output
goes to profiles/).  python scripts/ncu_summary.py report.ncu-rep [algo_bytes] [algo_flops]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(f"report: {rep}")
    for k in KEYS:
        if k in d:
            print(f"  {k:92s} {d[k]:>20s} {u.get(k, '')}")
    t_us = float(d["gpu__time_duration.sum"]) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u["gpu__time_duration.sum"], 1.0)
    rd = float(d["dram__bytes_read.sum"]) * (1e6 if u["dram__bytes_read.sum"] == "Mbyte" else
                                              1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1e3)
    wr = float(d["dram__bytes_write.sum"]) * (1e6 if u["dram__bytes_write.sum"] == "Mbyte" else
                                               1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1e3)
    print(f"  traffic (dram read+write) = {(rd + wr) / 1e6:.1f} MB; achieved dram {(rd + wr) / t_us / 1e3:.1f} GB/s")
    if len(sys.argv) > 2 and float(sys.argv[2]) > 0:
        ab = float(sys.argv[2])
        print(f"  algorithmic bytes {ab / 1e6:.1f} MB -> {ab / t_us / 1e3:.1f} GB/s; traffic/algorithmic = {(rd + wr) / ab:.3f}")
    if len(sys.argv) > 3:
        fl = float(sys.argv[3])
        print(f"  algorithmic flops {fl / 1e12:.3f} TFLOP -> {fl / t_us / 1e6:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
