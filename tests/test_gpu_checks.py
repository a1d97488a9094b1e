"""Bounds-checked kernel build (CSENC_CHECKS=1: every bulk copy, converter SMEM read, TMEM column
range and output store is range-checked on the device; a violation traps).  compute-sanitizer is
not available on the GPU pool, so this is the memory-safety gate: small cases covering every
block size, key mode, folds, partial blocks and ragged GOPs for the top plans of each (and every
KEY_CHUNK / streamed-Phi plan), every q16 mode, closed-loop / chained keys, per-GOP Phi, the adjoint
and the frame-level GEMM -- tools/sanitize_cases.py.

The same build is the race gate: with CSENC_STRESS set, every mbarrier wait of K1 is followed (one
time in four) by a pseudo-random delay of up to ~2 us (ptx::stress_point), so producer, converters,
MMA issuer and epilogue interleave in orders the normal schedule never shows; a missing wait, a
wrong phase or a buffer recycled early gives wrong measurements or a hang (the 20 s watchdog
traps).  Every candidate plan of every case runs under two seeds."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def checks_lib():
    from paper_1311_1419_b200 import _build
    lib = os.path.join(_build.LIB_DIR, "libcsenc_checks.so")
    deps = [os.path.join(_build.CSRC, f) for f in os.listdir(_build.CSRC)]
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(d) for d in deps):
        _build.build(out=lib, defines=("CSENC_CHECKS=1",))
    return lib


def run_cases(extra_env, timeout=900):
    env = dict(os.environ, CSENC_LIB=checks_lib(), **extra_env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert "CSENC_CHECK failed" not in r.stdout + r.stderr, r.stdout + r.stderr
    assert r.returncode == 0 and "ALL_OK" in r.stdout, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_bounds_checked_build_runs_clean(gpu):
    run_cases({})


@pytest.mark.parametrize("seed", ["12345", "987654321"])
def test_mbarrier_race_gate(gpu, seed):
    out = run_cases({"CSENC_STRESS": seed, "SANITIZE_K1_ONLY": "1"})
    assert out.count(" True") >= 50


def test_race_gate_has_teeth(gpu):
    """The gate catches a real synchronisation bug: a build with the converters' A-buffer-empty wait
    removed (CSENC_INJECT_RACE, KEY_CHUNK plans) passes without the random delays and fails with them."""
    from paper_1311_1419_b200 import _build
    lib = os.path.join(_build.LIB_DIR, "libcsenc_race.so")
    deps = [os.path.join(_build.CSRC, f) for f in os.listdir(_build.CSRC)]
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(d) for d in deps):
        _build.build(out=lib, defines=("CSENC_CHECKS=1", "CSENC_INJECT_RACE=1"))
    env = dict(os.environ, CSENC_LIB=lib, CSENC_STRESS="12345", SANITIZE_K1_ONLY="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.stdout.count(" False") > 0, r.stdout[-3000:]
