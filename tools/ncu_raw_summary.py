"""Summarise one kernel of an `ncu --page raw --csv` dump: the metrics profiles/*.md quote
(duration, DRAM bytes, launch shape, issue, stall reasons). Usage: ncu_raw_summary.py raw.csv"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, units, val = rows[hi], rows[hi + 1], rows[hi + 2]
d = {h: (v, u) for h, u, v in zip(hdr, units, val)}
print("Kernel:", d["Kernel Name"][0])
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__cycles_active.max", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct"]
print("| metric | value |\n|---|---|")
for k in keys:
    if k in d:
        print(f"| {k} | {d[k][0]} {d[k][1]} |")
pre = "smsp__average_warps_issue_stalled_"
suf = "_per_issue_active.ratio"
st = sorted(((float(v[0].replace(",", "")), k[len(pre):-len(suf)]) for k, v in d.items()
             if k.startswith(pre) and k.endswith(suf) and v[0]), reverse=True)
print("\nTop stall reasons (warps stalled per issue-active cycle):\n")
for v, k in st[:8]:
    print(f"- {k}: {v:.6f}")
