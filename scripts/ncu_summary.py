"""Summarise an ncu --set full raw CSV (scripts/gpu.sh prof) into a short text file for profiles/."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(f"Kernel Name: {d.get('Kernel Name', '')}")
    for k in KEYS:
        if k in d:
            print(f"{k}: {d[k]} {units[hdr.index(k)]}")
    top = sorted(((float(d[s] or 0), s) for s in stall), reverse=True)[:6]
    for v, s in top:
        print(f"{s}: {v:.3f}")
    print()
