"""Summarise an ncu report (.ncu-rep) as markdown: duration, issue/pipe
utilisation, occupancy, DRAM traffic, top stall reasons, instruction mix.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [title] [kernel-regex] > profiles/x.md
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def _csv(path, *args):
    out = subprocess.run(["ncu", "-i", path, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path, title="", kernel=""):
    flt = ["--kernel-name", f"regex:{kernel}"] if kernel else []
    raw = _csv(path, "--page", "raw", *flt)
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def g(name):
        v = m.get(name)
        return f"{v[0]} {v[1]}".strip() if v else "n/a"

    kname = g("Kernel Name").replace(" ", "")
    print(f"### {title or kname}\n")
    print(f"kernel `{m.get('Kernel Name', ('?',))[0][:120]}`\n")
    rows = [
        ("duration", "gpu__time_duration.sum"),
        ("SM frequency", "smsp__cycles_elapsed.avg.per_second"),
        ("elapsed cycles", "sm__cycles_elapsed.max"),
        ("SM active cycles (avg)", "sm__cycles_active.avg"),
        ("issue slots busy", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("executed IPC (active)", "sm__inst_executed.avg.per_cycle_active"),
        ("warp instructions executed", "smsp__inst_executed.sum"),
        ("ALU pipe", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        ("FMA pipe", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        ("FMA-heavy pipe (elapsed)", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("LSU pipe", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        ("uniform pipe", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"),
        ("achieved occupancy", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("registers / thread", "launch__registers_per_thread"),
        ("grid x block", "launch__grid_size"),
        ("DRAM read bytes", "dram__bytes_read.sum"),
        ("DRAM write bytes", "dram__bytes_write.sum"),
        ("DRAM throughput", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
        ("tensor pipe", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ]
    print("| metric | value |\n|---|---|")
    for label, key in rows:
        print(f"| {label} | {g(key)} |")
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
              for h, v in zip(hdr, vals)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    print("\nwarp-state samples (top):\n")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
        print(f"- {k}: {100 * v / tot:.1f}%")
    src = _csv(path, "--page", "source", "--print-source", "sass", *flt)
    if len(src) > 2:
        h = src[1]
        data = [dict(zip(h, r)) for r in src[2:] if len(r) == len(h) and r != h]
        data = [d for d in data if (d.get("Instructions Executed") or "0").isdigit()]
        key = "Instructions Executed"
        tot_i = sum(int(d.get(key) or 0) for d in data) or 1
        op = collections.Counter()
        for d in data:
            t = d["Source"].split()
            o = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
            op[o.split(".")[0]] += int(d.get(key) or 0)
        print("\ninstruction mix (share of executed warp instructions):\n")
        print(", ".join(f"{o} {100 * n / tot_i:.1f}%" for o, n in op.most_common(10)))
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", sys.argv[3] if len(sys.argv) > 3 else "")
