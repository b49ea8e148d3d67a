"""Summarise an ncu --set full report (one kernel) into a short text block,
and an ncu launch-list CSV into per-kernel shares.  Output goes to profiles/.

    python tools/ncu_summary.py report <file.ncu-rep> [algorithmic_bytes]
    python tools/ncu_summary.py launches <launches.csv>
"""
import collections
import csv
import io
import signal
import subprocess
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def report(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]:>16s} {u.get(k, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(u["dram__bytes_read.sum"], 1)
            wr *= scale.get(u["dram__bytes_write.sum"], 1)
            print(f"  dram traffic (read+write) = {(rd + wr) / 1e6:.1f} MB")
            if alg_bytes:
                print(f"  algorithmic bytes = {alg_bytes / 1e6:.1f} MB -> traffic/algorithmic = "
                      f"{(rd + wr) / alg_bytes:.4f}")
        except (KeyError, ValueError):
            pass


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hd = rows[h]
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) != len(hd):
            continue
        d = dict(zip(hd, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
        agg[d["Kernel Name"].split("(")[0][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8s} {'mean us':>10s} {'total us':>11s} {'share':>6s}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{len(v):8d} {sum(v) / len(v):10.1f} {sum(v):11.1f} {100 * sum(v) / tot:5.1f}%  {k}")
    print(f"total device time {tot:.1f} us (ncu-serialised, cold caches)")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
    else:
        launches(sys.argv[2])
