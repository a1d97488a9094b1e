"""The C ABI used from plain C (examples/encode_host.c, built by __graft_entry__.build()): it links
against libcsenc.so, encodes host frames and checks every measurement against its own double sum."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "encode_host.c")


def test_example_compiles_against_the_header(tmp_path):
    """CPU: the example compiles and links with the public header and library only."""
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    lib_dir = os.path.join(ROOT, "paper_1311_1419_b200", "_lib")
    if not os.path.exists(os.path.join(lib_dir, "libcsenc.so")):
        pytest.skip("libcsenc.so not built")
    exe = str(tmp_path / "encode_host")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
                           "-L", lib_dir, "-lcsenc", f"-Wl,-rpath,{lib_dir}", "-lm", "-o", exe])
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_example_runs_on_the_gpu(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_1311_1419_b200", "_lib")
    exe = str(tmp_path / "encode_host")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), SRC, "-L", lib_dir,
                           "-lcsenc", f"-Wl,-rpath,{lib_dir}", "-lm", "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("encode_host OK"), r.stdout
