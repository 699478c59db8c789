"""Summarise an ncu report: headline metrics + per-source-line instructions/stall samples."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for k, v in zip(r[0], r[2]):
    if k in want:
        print(f"  {k:80s} {v[:70]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = None; fname = None; out = []; ti = ts = 0
for row in rows:
    if row and row[0] == "File Path":
        fname = row[1].split("/")[-1]; continue
    if row and row[0] == "Line No":
        hdr = row; continue
    if not row or row[0] == "Function Name" or hdr is None:
        continue
    if row[2] == "-" and row[0].isdigit():
        def g(k):
            x = row[hdr.index(k)]
            return float(x.replace(",", "")) if x not in ("", "-") else 0.0
        ie, ss = g("Instructions Executed"), g("Warp Stall Sampling (All Samples)")
        sec = g("L2 Theoretical Sectors Global")
        ti += ie; ts += ss
        out.append((ss, ie, sec, fname, row[0], row[1][:88]))
out.sort(reverse=True)
print(f"  total warp-inst {ti/1e6:.2f}M  samples {ts:.0f}")
for ss, ie, sec, f, ln, s in out[:top]:
    print(f"  {100*ss/max(ts,1):5.1f}% {ie/1e6:7.2f}Mi {sec*32/1e6:7.1f}MB  {f}:{ln} {s}")
