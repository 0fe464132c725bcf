"""Summarise one kernel of an ncu --set full report into JSON (profiles/)."""
import csv
import io
import json
import subprocess
import sys

METRICS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
           "dram__bytes_write.sum", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_barrier"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {m: [v[h.index(m)], u[h.index(m)]] for m in METRICS if m in h}


if __name__ == "__main__":
    json.dump(summary(sys.argv[1]), open(sys.argv[2], "w"), indent=1)
