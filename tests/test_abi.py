"""C-ABI checks that need no GPU (-m "not gpu"): libddh.so loads, exports
every function include/ddh.h declares, the ctypes mirror of ddh_params has
the C layout, defaults match the paper, and ddh_create fails cleanly (no CPU
fallback) when no CUDA device is present."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest
import torch

from paper_2305_03284_b200 import build as B
from paper_2305_03284_b200 import ddh as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ddh.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return D.load_library()


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ddh_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_expected_entry_points():
    fns = header_functions()
    for f in ["ddh_create", "ddh_bootstrap", "ddh_step", "ddh_strehl", "ddh_destroy", "ddh_step_host"]:
        assert f in fns
    assert sorted(D.EXPORTS) == fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", D.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(\w+)", out))
    for f in header_functions():
        assert f in exported, f
        assert hasattr(lib, f)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", D.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_params_layout_matches_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "ddh.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(ddh_params), offsetof(ddh_params, aperture_mask),"
        " offsetof(ddh_params, r_min), offsetof(ddh_params, boot_alpha), offsetof(ddh_params, chunk_streams),"
        " offsetof(ddh_params, flags)); return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    P = D.DdhParams
    assert vals == [ctypes.sizeof(P), P.aperture_mask.offset, P.r_min.offset, P.boot_alpha.offset,
                    P.chunk_streams.offset, P.flags.offset]


def test_default_params_follow_paper(lib):
    p = D.default_params()
    assert p.lam == 0.45 and p.alpha == 0.025
    assert p.boot_period == 200
    assert p.n_k == 1 and p.r_min == 1e-4


def test_create_rejects_bad_params_without_gpu(lib):
    p = D.default_params()
    h = ctypes.c_void_p()
    p.n = 100
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 1
    assert b"n must be" in lib.ddh_last_error(None)
    p = D.default_params()
    p.lam = 1.5
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 1
    p = D.default_params()
    assert p.aperture_diam == 0.0  # default: D = N (whatever N is)
    p.aperture_diam = -1.0  # a mask is required then
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 1
    p = D.default_params()
    p.n, p.aperture_diam = 64, 65.0  # wider than the grid
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 1
    assert b"aperture_diam" in lib.ddh_last_error(None)
    p = D.default_params()
    p.flags = 4  # the retired cluster path
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_create_fails_loudly_without_gpu(lib):
    p = D.default_params()
    h = ctypes.c_void_p()
    assert lib.ddh_create(ctypes.byref(p), None, ctypes.byref(h)) == 2  # DDH_E_CUDA, no CPU fallback
    assert h.value is None


def test_null_ctx_is_rejected(lib):
    assert lib.ddh_step(None, None, 0, None, None, None) == 1
    assert lib.ddh_sync(None) == 1
    assert lib.ddh_kernel_launches(None) == 0
