"""Summarise ncu --set full reports (raw page) into the handful of metrics the roofline needs."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d.get("Kernel Name", "")[:90], {k: f"{d.get(k, '')} {u.get(k, '')}".strip() for k in KEYS}))
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for name, m in summarise(p):
            print(f"## {p.split('/')[-1]}: {name}")
            for k, v in m.items():
                print(f"  {k:90s} {v}")
