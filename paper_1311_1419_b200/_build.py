"""Build libcsenc.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.environ.get("CSENC_LIB") or os.path.join(LIB_DIR, "libcsenc.so")
SOURCES = ["cs_common.cu", "cs_encoder.cu", "cs_adjoint.cu", "cs_keys.cu", "cs_frame.cu"]
HEADERS = ["cs_measure_kernel.cuh", "ptx_sm100.cuh", "cs_adjoint_kernel.cuh", "cs_key_codec_kernel.cuh",
           "cs_frame_kernel.cuh", "cs_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "cs_encoder.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every translation unit (in parallel) and link libcsenc.so."""
    if out is None and not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    target = out or LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    flags = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    flags += [f"-D{d}" for d in defines]
    if verbose:
        flags += ["-Xptxas", "-v"]
    with tempfile.TemporaryDirectory(prefix="csenc_build_") as tmp:
        objs = [os.path.join(tmp, f.replace(".cu", ".o")) for f in SOURCES]

        def compile_one(i):
            subprocess.check_call([NVCC, *flags, "-c", os.path.join(CSRC, SOURCES[i]), "-o", objs[i]])

        with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            list(ex.map(compile_one, range(len(SOURCES))))
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", target + ".tmp", *objs])
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
