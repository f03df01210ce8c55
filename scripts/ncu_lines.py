"""Attribute an ncu SASS profile to CUDA source lines.

ncu's CSV source export carries no per-line metrics here, so this joins the
per-instruction SASS page (exec counts, warp-state samples) with nvdisasm's
line table of the SAME build (-lineinfo):

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep <kernel-regex> [libbplb.so] [mangled-substring] [frame-file]

Only valid when the report was captured from the library passed in.
"""

from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_rows(rep, kernel_sub=""):
    flt = ["--kernel-name", f"regex:{kernel_sub}"] if kernel_sub else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", *flt],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r != hdr]


def line_table(lib, kernel_sub, frame_file=None):
    """SASS offset -> (file, line).  nvdisasm prints an instruction's inline
    chain innermost first; by default the OUTERMOST frame is used (the line in
    the kernel body), with ``frame_file`` the innermost frame in that file
    (e.g. bplb_prune.cuh: lines inside the inlined device functions)."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    table = {}
    func = None
    chain, cur, fresh = [], None, True
    for line in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", line)
        if m:
            func = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            if fresh:
                chain, fresh = [], False
            chain.append((os.path.basename(m.group(1)), int(m.group(2))))
            cur = chain[-1]
            if frame_file:
                inner = [fr for fr in chain if fr[0] == frame_file]
                if inner:
                    cur = inner[0]
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
        if m:
            fresh = True
            if func and kernel_sub in func:
                table[int(m.group(1), 16)] = cur
    return table


def main(rep, kernel_sub, lib="paper_2402_14821_b200/libbplb.so", mangled=None, frame_file=None):
    """kernel_sub filters the ncu report (demangled name regex); mangled (or
    kernel_sub) selects the function in the library's line table."""
    rows = sass_rows(rep, kernel_sub)
    base = int(rows[0]["Address"], 16)
    table = line_table(lib, mangled or kernel_sub, frame_file)
    S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    agg_s, agg_i = collections.Counter(), collections.Counter()
    reasons = collections.defaultdict(collections.Counter)
    for d in rows:
        off = int(d["Address"], 16) - base
        key = table.get(off, ("?", 0))
        agg_s[key] += int(d[S] or 0)
        agg_i[key] += int(d[I] or 0)
        for col, v in d.items():
            if col.startswith("stall_") and "Not Issued" not in col and v and v.isdigit():
                reasons[key][col[6:]] += int(v)
    ts, ti = sum(agg_s.values()) or 1, sum(agg_i.values()) or 1
    srcs = {}
    for (f, ln) in agg_s:
        if f != "?" and f not in srcs:
            for root in ("paper_2402_14821_b200/csrc",):
                p = os.path.join(root, f)
                if os.path.exists(p):
                    srcs[f] = open(p).read().splitlines()
    print(f"{'samples':>8} {'instr':>7}  location")
    for key, s in sorted(agg_s.items(), key=lambda kv: -kv[1])[:45]:
        f, ln = key
        text = srcs.get(f, [""] * (ln + 1))[ln - 1].strip() if ln and f in srcs else ""
        top = ",".join(f"{r}:{100 * n / max(s, 1):.0f}" for r, n in reasons[key].most_common(3))
        print(f"{100 * s / ts:7.1f}% {100 * agg_i[key] / ti:6.1f}%  {f}:{ln}  {text[:70]:70s} [{top}]")


if __name__ == "__main__":
    main(*sys.argv[1:])
