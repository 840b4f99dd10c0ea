"""Sanitizer substitute (SURVEY 4.2 "S", 5 race detection): compute-sanitizer
is not available on the GPU pool, so the bounds-checked build
(lib/libddh_debug.so, -DDDH_DEBUG_BOUNDS=1) runs the parity tests at small N
in a child process.  Every shared-memory tile index of the ICD kernels is
checked to lie inside the tile and outside its padding; every neighbour read
of a colour phase must come from another colour sub-grid (no read of a pixel
the phase writes: the colour-phase race condition), the own pixel from the
phase's colour; global indices of the tiles and the halo lie inside the
frame.  A violation traps the kernel (the test then fails with a CUDA error
and the printed location)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_build_runs_parity_tests():
    from paper_2305_03284_b200 import build
    lib = build.build(debug=True)
    env = dict(os.environ, DDH_LIB=lib)
    sel = ("ricd_stage or ricd_large_launch or phiicd_stage or chain_step_parity or step_parity_priors_on and (64 or 128) or step_parity_masked "
           "or kernel_variants or degenerate or end_to_end_c1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "tests/test_gpu_parity.py", "-k", sel]
    pr = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert pr.returncode == 0, (pr.stdout[-4000:], pr.stderr[-2000:])
    assert "passed" in pr.stdout and "DDH_DEBUG_BOUNDS" not in pr.stdout


def test_bounds_checked_build_traps_an_injected_violation():
    """The checks are live: DDH_DEBUG_FAULT=1 makes the r-ICD assert that its
    own pixel is NOT of the phase's colour; the kernel must trap with the
    DDH_DEBUG_BOUNDS message (and the release library ignores the variable)."""
    from paper_2305_03284_b200 import build
    lib = build.build(debug=True)
    code = ("import torch, numpy as np; from paper_2305_03284_b200 import DDH; "
            "c = DDH(64, 1, noise_var=0.1); r = torch.rand(1, 64, 64, device='cuda') + 0.1; "
            "out = c.test_ricd(r, r.clone()); torch.cuda.synchronize(); print('RAN', float(out.sum()))")
    bad = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, DDH_LIB=lib, DDH_DEBUG_FAULT="1"),
                         capture_output=True, text=True, timeout=300)
    assert bad.returncode != 0 and "DDH_DEBUG_BOUNDS" in bad.stdout + bad.stderr, (bad.stdout[-2000:], bad.stderr[-2000:])
    ok = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, DDH_DEBUG_FAULT="1"),
                        capture_output=True, text=True, timeout=300)
    assert ok.returncode == 0 and "RAN" in ok.stdout, ok.stderr[-2000:]
