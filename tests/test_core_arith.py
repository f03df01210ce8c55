"""Host-compiled check of the integer core shared with the kernels
(paper_2402_14821_b200/csrc/bplb_core.h) against brute force.  CPU only."""

import os
import subprocess

from conftest import ROOT


def test_core_arith(tmp_path):
    exe = tmp_path / "core_arith_test"
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe),
                    os.path.join(ROOT, "tests", "core_arith_test.cpp")], check=True)
    res = subprocess.run([str(exe), "1500"], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK" in res.stdout
