"""Key metrics of one kernel in an ncu report (dev tool): duration, DRAM bytes and
throughput, tensor-pipe activity, occupancy, issue, stall mix.

usage: python tools/ncu_summary.py report.ncu-rep
"""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA subpipe active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "UMMA (tcgen05) pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "CTAs"),
    ("launch__block_size", "threads / CTA"),
]

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}
print(f"kernel: {vals[col['Kernel Name']]}")
for key, label in WANT:
    if key in col:
        print(f"  {label:28s} {vals[col[key]]:>16s} {units[col[key]]}")
stalls = []
for h, i in col.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
        try:
            stalls.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(s for s, _ in stalls) or 1.0
print("  stall mix (pc sampling):", ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:6]))
