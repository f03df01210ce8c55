"""Parse an ncu --csv capture of scripts/cfg4_one.py (two cfg4 checks) into
profiles/cfg4_wide_ncu.json: per-kernel duration / warp instructions / DRAM
bytes of the SECOND check's launch sequence (wide_init .. wide_finish) and the
wide_units totals bench.py's cfg4 roofline uses.

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum --clock-control none --csv \
        python scripts/cfg4_one.py > gpurun_out/ncu_cfg4_metrics.csv
"""
import collections
import csv
import json
import os
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
launches = collections.OrderedDict()
for r in rows:
    lid = int(r[0])
    d = launches.setdefault(lid, {"kernel": r[4].split("(")[0]})
    d[r[12]] = float(r[14].replace(",", ""))
seq = list(launches.values())
starts = [i for i, d in enumerate(seq) if "wide_init" in d["kernel"]]
second = seq[starts[-1]:]
units = [d for d in second if "wide_units" in d["kernel"]]
out = {
    "kernels": [{"kernel": d["kernel"], "us": d.get("gpu__time_duration.sum", 0) / 1e3,
                 "warp_inst": d.get("smsp__inst_executed.sum"),
                 "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)} for d in second],
    "wide_units_warp_inst": sum(d["smsp__inst_executed.sum"] for d in units),
    "wide_units_us": sum(d["gpu__time_duration.sum"] for d in units) / 1e3,
    "wide_units_dram_bytes": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in units),
    "wide_units_l2_sectors": sum(d.get("l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum", 0) for d in units),
    "sequence_us_serialised": sum(d.get("gpu__time_duration.sum", 0) for d in second) / 1e3,
    "source": os.path.basename(path) + " (ncu --metrics, --clock-control none, second of two cfg4 checks)",
}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "cfg4_wide_ncu.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
