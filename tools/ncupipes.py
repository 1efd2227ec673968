"""Profiling aid: pipe utilisation per kernel from an ncu --set full report
(tensor / FMA / ALU / FP64 pipes, L1 and L2 throughput, DRAM bytes)."""
import csv
import subprocess
import sys

KEYS = {
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_hmma_inst_pct": "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "time_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
}

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    vals = {k: d.get(v) for k, v in KEYS.items() if d.get(v) not in (None, "", "n/a")}
    print(f"{d['Kernel Name'].split('(')[0][-40:]:40s} " + "  ".join(f"{k}={v}" for k, v in vals.items()))
