"""Summarise an ncu --set full report into a text table (per kernel)."""
import csv, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
idx = {w: h.index(w) for w in want if w in h}
with open(out, "w") as fh:
    fh.write("kernel," + ",".join(f"{w} [{units[idx[w]]}]" for w in idx) + "\n")
    for row in r[2:]:
        fh.write(row[h.index("Kernel Name")].split("(")[0] + "," + ",".join(row[idx[w]] for w in idx) + "\n")
print(open(out).read())
