"""Summarise `ncu --set full` reports (.ncu-rep) into a text table for profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep [label] [--algo-bytes B1,B2,...] [--algo-flops F1,F2,...]
"""
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
METRICS = [   # (metric, column, scale applied to the value converted to seconds / bytes)
    ("gpu__time_duration.sum", "dur_us", 1e6),
    ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
    ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1),
    # tcgen05 (UTCHMMA) issue is counted by the tensor pipe's HMMA sub-pipe; the
    # legacy tensor_% / op-path columns do not see tcgen05 MMAs on sm_100
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", "hmma_subpipe_%", 1),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tc_pipe_%", 1),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tmem_%", 1),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.sum", "utchmma_inst", 1),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    path = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else path
    algo = flops = None
    if "--algo-bytes" in sys.argv:
        algo = [float(x) for x in sys.argv[sys.argv.index("--algo-bytes") + 1].split(",")]
    if "--algo-flops" in sys.argv:
        flops = [float(x) for x in sys.argv[sys.argv.index("--algo-flops") + 1].split(",")]
    h, units, rows = load(path)
    idx = {n: i for i, n in enumerate(h)}
    kcol = idx.get("Kernel Name", idx.get("Function Name"))
    print(f"# {label}")
    cols = ["kernel"] + [m[1] for m in METRICS if any(n.endswith(m[0]) for n in h)]
    if algo:
        cols += ["algo_MB", "achieved_GB/s", "traffic/algo"]
    if flops:
        cols += ["algo_GFLOP", "achieved_TFLOP/s"]
    print(" | ".join(cols))
    for li, r in enumerate(rows):
        vals = [r[kcol].split("(")[0][-40:]]
        got = {}
        for m, short, sc in METRICS:
            name = next((n for n in h if n.endswith(m)), None)
            if name is None:
                continue
            try:
                v = float(r[idx[name]].replace(",", "")) * UNIT.get(units[idx[name]], 1.0) * sc
            except ValueError:
                v = float("nan")
            got[short] = v
            vals.append(f"{v:.2f}" if abs(v) < 1e6 else f"{v:.3e}")
        if algo and li < len(algo):
            a = algo[li]
            traffic = (got.get("dram_rd_MB", 0) + got.get("dram_wr_MB", 0)) * 1e6
            vals += [f"{a / 1e6:.2f}", f"{a / (got['dur_us'] * 1e-6) / 1e9:.1f}", f"{traffic / a:.3f}"]
        if flops and li < len(flops):
            f = flops[li]
            vals += [f"{f / 1e9:.1f}", f"{f / (got['dur_us'] * 1e-6) / 1e12:.1f}"]
        print(" | ".join(vals))


if __name__ == "__main__":
    main()
