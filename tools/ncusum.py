"""Profiling aid: key metrics + top stall reasons per kernel from an ncu report (raw page csv)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
st = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("----", d["Kernel Name"][:70])
    print("   ", {w.split("__", 1)[1][:34]: d.get(w) for w in want if w in d})
    tot = sum(float(d[k] or 0) for k in st) or 1
    top = sorted(((float(d[k] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in st), reverse=True)[:8]
    print("    stalls", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))
