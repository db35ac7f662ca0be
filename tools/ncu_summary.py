"""Summarise an ncu --set full report: headline metrics + SASS lines by instructions / stall samples.
    python tools/ncu_summary.py report.ncu-rep [units_per_launch] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, unit, val = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for h in want:
    if h in hdr:
        i = hdr.index(h)
        print(f"{h:70s} {val[i]:>18s} {unit[i]}")
stall = [(h, val[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
stall = sorted(((float(v.replace(",", "")), h) for h, v in stall if v not in ("", "n/a")), reverse=True)[:8]
for v, h in stall:
    print(f"  stall {h.replace('smsp__average_warp_latency_issue_stalled_', ''):50s} {v:8.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
ia, isrc, ist = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia]) for r in data if r[ia].isdigit())
stot = sum(int(r[ist]) for r in data if r[ist].isdigit()) or 1
print(f"instructions {tot} = {tot / units:.1f} per unit; stall samples {stot}")
ranked = sorted(((int(r[ist]) if r[ist].isdigit() else 0, k, r) for k, r in enumerate(data)), reverse=True)[:top]
for sv, k, r in sorted(ranked, key=lambda x: x[1]):
    print(f"{k:5d} {int(r[ia]) / units:7.3f}/u st={sv / stot * 100:5.1f}%  {r[isrc].strip()[:100]}")
