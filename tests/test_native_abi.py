"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/bplb.h declares (no compute calls: CPU only)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "bplb.h")).read()
    return sorted(set(re.findall(r"BPLB_API\s+[\w\s\*]+?\b(bplb_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for want in ("bplb_engine_create", "bplb_engine_destroy", "bplb_check", "bplb_dff_bound_batch",
                 "bplb_check_batch", "bplb_check_batch_device", "bplb_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2402_14821_b200 import build_native, _native

    path = build_native.build()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    # ctypes signatures cover every declared symbol
    assert set(_declared()) == set(_native.SIGNATURES)
    lib = _native.load_library(path)
    assert b"sm_100a" in lib.bplb_version()


def test_library_is_sm100a_code():
    from paper_2402_14821_b200 import build_native

    path = build_native.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "VIADDMNMX" in sass  # the modular walk's DPX min-add


def test_engine_create_without_gpu_fails_cleanly():
    import torch

    from paper_2402_14821_b200 import _native

    if torch.cuda.is_available():
        return
    lib = _native.load_library()
    h = ctypes.c_void_p()
    rc = lib.bplb_engine_create(0, ctypes.byref(h))
    assert rc == _native.E_NODEV
    assert lib.bplb_last_error()
