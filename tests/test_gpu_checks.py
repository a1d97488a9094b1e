"""Bounds-checked kernel build (CSENC_CHECKS=1: every bulk copy, converter SMEM read, TMEM column
range and output store is range-checked on the device; a violation traps).  compute-sanitizer is
not available on the GPU pool, so this is the memory-safety gate: small cases covering every
block size, key mode, folds, partial blocks and ragged GOPs for the top plans of each, every q16
mode, closed-loop / chained keys, per-GOP Phi, the adjoint and the frame-level GEMM (single CTA,
2-CTA cluster, split-K) -- tools/sanitize_cases.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_build_runs_clean():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1311_1419_b200 import _build
    lib = os.path.join(_build.LIB_DIR, "libcsenc_checks.so")
    deps = [os.path.join(_build.CSRC, f) for f in os.listdir(_build.CSRC)]
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(d) for d in deps):
        _build.build(out=lib, defines=("CSENC_CHECKS=1",))
    env = dict(os.environ, CSENC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert "CSENC_CHECK failed" not in r.stdout + r.stderr, r.stdout + r.stderr
    assert r.returncode == 0 and "ALL_OK" in r.stdout, r.stdout + r.stderr
