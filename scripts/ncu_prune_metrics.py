"""Parse an ncu --csv metrics capture of ONE prune_kernel launch over N cfg5
nodes (scripts/cfg5_one_launch.py N lb) into profiles/prune_kernel_ncu.json:
executed warp instructions and DRAM bytes per node -- the per-launch figures
bench.py's roofline scales by its node count.

    python scripts/ncu_prune_metrics.py gpurun_out/ncu_cfg5_metrics.csv N
"""
import csv
import json
import os
import sys

path, n = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and "prune_kernel" in r[4]]
m = {r[12]: float(r[14].replace(",", "")) for r in rows}
out = {
    "nodes": n,
    "warp_inst_per_node": m["smsp__inst_executed.sum"] / n,
    "dram_bytes_per_node": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / n,
    "duration_ms_under_ncu": m["gpu__time_duration.sum"] / 1e6,
    "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "source": os.path.basename(path) + " (ncu --metrics, --clock-control none, one launch over the first N nodes "
              "of the cfg5 stream, lb mode)",
}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "prune_kernel_ncu.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out))
