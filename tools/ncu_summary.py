"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep / csv
brought back in gpurun_out/)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                print(f"   {k:80s} {row[hdr.index(k)]:>14s} {units[hdr.index(k)]}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        d[r[ki].split("(")[0].split("::")[-1]][r[mi]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(m["gpu__time_duration.sum"]) for m in d.values())
    for k, m in sorted(d.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = m["gpu__time_duration.sum"]
        rd = sum(m.get("dram__bytes_read.sum", [0])) / len(t)
        wr = sum(m.get("dram__bytes_write.sum", [0])) / len(t)
        print(f"{k:24s} launches={len(t):4d} avg={sum(t) / len(t) / 1e3:8.2f} us share={sum(t) / tot * 100:5.1f}% "
              f"dram_rd={rd / 1e6:7.1f} MB dram_wr={wr / 1e6:6.1f} MB")


if __name__ == "__main__":
    (full if sys.argv[1] == "full" else launches)(sys.argv[2])
