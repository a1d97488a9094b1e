"""bench.py's JSON line keeps the driver's contract: the reference arm (the CPU oracle, runs here) and,
on a B200, the device arm with roofline / clocks / e2e / cpu_baseline / gpu_launches."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config")


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def check_base(d):
    for k in BASE_KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["config"]["workload"] == "C4"


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    check_base(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_device_arm_contract():
    d = run_bench("--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--cpu-budget", "2")
    check_base(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    # time base: the timed region (step bytes / step time); the per-launch event pairs are reported beside it
    alg = sum(m["alg_bytes"] for m in d["per_M"].values())
    assert abs(r["achieved"] - alg / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    assert 0 < r["achieved_event_pairs"] < 1.5 * r["peak"] and "timed region" in r["time_base"]
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 240 * 1920 * 1080
    assert e["d2h_bytes_per_step"] == 4 * 210 * 8160 * (16 + 32 + 64 + 128)
    assert d["gpu_launches"] == 3 * 4
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert d["parity"]["ok"] is True and d["parity"]["entries"] == 4 * 400
    for m in d["per_M"].values():
        assert m["ms_mean_l2clean"] > 0


def test_self_launch_n_ranks():
    """--gpus N without torchrun re-runs bench.py under torch.distributed.run with N ranks; the
    launcher check (gloo, no GPU) proves every rank joined and rank 0 reports n_gpus == N."""
    d = run_bench("--gpus", "2", "--launcher-check", timeout=300)
    assert d["n_gpus"] == 2 and d["max_ms_over_ranks"] == 2.0 and d["streams"] == [0, 1]


@pytest.mark.gpu
def test_multi_gpu_bench():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    d = run_bench("--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--M", "16",
                  "--tune-candidates", "2")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity"]["ok"] is True


@pytest.mark.gpu
@pytest.mark.parametrize("args,bound", [(("--op", "adjoint"), "hbm"), (("--op", "closed_loop"), "hbm"),
                                        (("--output", "q16row"), "hbm"), (("--op", "frame"), "tensor")])
def test_device_arm_variants(args, bound):
    d = run_bench(*args, "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--tune-candidates", "2")
    for k in BASE_KEYS:
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == bound and 0 < r["frac"] < 1.5 and d["gpu_launches"] > 0
    if "parity" in d and d["parity"]["ok"] is not None:
        assert d["parity"]["ok"] is True, d["parity"]


@pytest.mark.gpu
def test_device_arm_q16_e2e():
    """--output q16row: the host-buffer e2e goes through cs_encode_batch_host_multi_q16 and copies
    back int16 codes + per-row fp32 scales."""
    d = run_bench("--output", "q16row", "--steps", "2", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline",
                  "--tune-candidates", "2")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 240 * 1920 * 1080
    assert e["d2h_bytes_per_step"] == 2 * 210 * 8160 * (16 + 32 + 64 + 128) + 4 * 4 * 210 * 68
    assert d["parity"]["ok"] is True
