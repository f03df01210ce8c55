"""Build libbplb.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbplb.so")
GEN_OUT = os.path.join(HERE, "libbplb_gen.so")  # synthetic node generator (workload data, not the path)
PEAKS_OUT = os.path.join(HERE, "libbplb_peaks.so")  # measured issue-rate denominators (bench.py only)
SOURCES = ["bplb_capi.cu"]
HEADERS = ["bplb_core.h", "bplb_device.cuh", "bplb_node.cuh", "bplb_prune.cuh", "bplb_ubound.cuh", "bplb_warp.cuh", "bplb_wide.cuh", "bplb_tab.cuh", "bplb_reduce.cuh", "bplb_knap.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "bplb.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build_gen(force: bool = False, src_name: str = "bplb_gen.cu", out: str = GEN_OUT) -> str:
    src = os.path.join(CSRC, src_name)
    GEN_OUT = out  # noqa: N806
    if not force and os.path.exists(GEN_OUT) and os.path.getmtime(GEN_OUT) > os.path.getmtime(src):
        return GEN_OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared", "-o", GEN_OUT + ".tmp", src,
           "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(GEN_OUT)}")
    os.replace(GEN_OUT + ".tmp", GEN_OUT)
    return GEN_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    build_gen(force)
    build_gen(force, "bplb_peaks.cu", PEAKS_OUT)
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", OUT + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES], "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libbplb.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
