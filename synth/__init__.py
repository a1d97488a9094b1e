"""synth -- seeded synthetic inputs shared by the oracle and the CUDA path.

INPUT GENERATORS ONLY: this module draws the measurement matrix Phi and the
synthetic surveillance video.  It holds none of the method's arithmetic
(no residual, no measurement, no compression ratio), so importing it from both
``oracle/`` and ``paper_1311_1419_b200/`` does not couple them (DESIGN.md
"Input recipe").

* ``phi_from_seed(seed, M, N)`` -- the measurement matrix: M x N entries
  RNE_fp16(z / sqrt(M)), z ~ N(0,1) from SplitMix64 -> 53-bit uniforms in (0,1]
  -> Box-Muller pairs filled row-major.  "Gaussian random matrix is used to make
  the measurements" (sec.4, PAPER.md:25+31 sec.1); variance 1/m and
  a frozen PRNG per SPEC.md:111.  Returned as IEEE fp16 BIT
  PATTERNS (uint16), so both sides consume identical bits.
* ``gen_video(cfg, seed)`` -- uint8 [S][T][H][W] frames (C generator
  ``cs_synth.c``; scene model in its header and DESIGN.md).
* ``CONFIGS`` -- the five BASELINE.json configs (BASELINE.json:7-11).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libcssynth.so")
_SRC = os.path.join(_HERE, "cs_synth.c")

BASE_SEED = 0x13111419
MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def build(force: bool = False) -> str:
    """Compile the generator (plain C, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.cs_synth_background.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
        lib.cs_synth_frames.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p]
        lib.cs_synth_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


# ----------------------------------------------------------------------------------------------
# SplitMix64 (python ints) -- used for Phi and for the handful of object parameters
# ----------------------------------------------------------------------------------------------
def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        return _mix(self.state)

    def uniform(self) -> float:  # (0,1]
        return ((self.next() >> 11) + 1) * (1.0 / 9007199254740992.0)

    def randint(self, lo: int, hi: int) -> int:  # inclusive
        return lo + int(self.uniform() * (hi - lo + 1) - 1e-12)


def _splitmix_u01(seed: int, n: int) -> np.ndarray:
    """n SplitMix64 outputs of stream `seed` mapped to (0,1] (vectorised)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & MASK64) + i * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def phi_from_seed(seed: int, M: int, N: int) -> np.ndarray:
    """Phi as uint16 fp16 bit patterns, shape [M][N] row-major (see module doc)."""
    n = M * N
    npair = (n + 1) // 2
    u = _splitmix_u01(seed, 2 * npair)
    u1, u2 = u[0::2], u[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * npair, dtype=np.float64)
    z[0::2] = rad * np.cos(2.0 * np.pi * u2)
    z[1::2] = rad * np.sin(2.0 * np.pi * u2)
    vals = (z[:n] / math.sqrt(M)).astype(np.float16)  # IEEE RNE double -> half
    return vals.view(np.uint16).reshape(M, N).copy()


# ----------------------------------------------------------------------------------------------
# Configs (BASELINE.json:7-11).  Values BASELINE.json leaves open are marked in DESIGN.md.
# ----------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class VideoConfig:
    name: str
    W: int
    H: int
    T: int                # frames per stream
    S: int                # streams
    G: int                # GOP size
    B: int                # block size
    Ms: tuple             # measurement counts (C4 sweeps four)
    sigma: float = 2.0
    period: int = 16      # background lattice period P
    n_obj: tuple = (1, 1)     # min,max objects per stream
    size: tuple = (24, 24)    # object size range (px)
    speed: tuple = (2.0, 2.0)  # px/frame
    intensity: int = -1       # -1 => U{0..255}
    fixed_motion: tuple = ()  # explicit (x0,y0,vx,vy,w,h,I) list (C1)
    drift_amp: float = 0.0
    drift_period: int = 0
    config_id: int = 0

    @property
    def M(self) -> int:
        return self.Ms[0]

    def with_(self, **kw) -> "VideoConfig":
        return replace(self, **kw)


CONFIGS = {
    # QCIF, 1 GOP of 4, one 24x24 square of intensity 220 moving +2 px/frame in x.
    "C1": VideoConfig("C1-QCIF", 176, 144, 4, 1, 4, 16, (64,), sigma=2.0, period=16,
                      fixed_motion=((40.0, 60.0, 2.0, 0.0, 24, 24, 220),), config_id=1),
    "C2": VideoConfig("C2-CIF", 352, 288, 300, 1, 8, 16, (32,), sigma=2.0, period=16,
                      n_obj=(3, 3), size=(16, 40), speed=(1.0, 4.0), config_id=2),
    "C3": VideoConfig("C3-VGA", 640, 480, 600, 1, 16, 32, (64,), sigma=3.0, period=32,
                      n_obj=(5, 5), size=(24, 64), speed=(1.0, 4.0), drift_amp=10.0, drift_period=600,
                      config_id=3),
    "C4": VideoConfig("C4-1080p", 1920, 1080, 240, 1, 8, 16, (16, 32, 64, 128), sigma=2.0, period=32,
                      n_obj=(8, 8), size=(32, 128), speed=(1.0, 6.0), config_id=4),
    "C5": VideoConfig("C5-64x720p", 1280, 720, 128, 64, 32, 8, (4,), sigma=2.0, period=32,
                      n_obj=(2, 4), size=(24, 96), speed=(1.0, 4.0), config_id=5),
}


def stream_seed(cfg: VideoConfig, stream: int, seed: int = BASE_SEED) -> int:
    return _mix((seed ^ (cfg.config_id << 32) ^ (stream * GOLDEN)) & MASK64)


def phi_seed(seed: int = BASE_SEED) -> int:
    return (seed + 1) & MASK64


def make_objects(cfg: VideoConfig, stream: int, seed: int = BASE_SEED) -> np.ndarray:
    if cfg.fixed_motion:
        return np.asarray(cfg.fixed_motion, dtype=np.float64).reshape(-1, 7)
    rng = SplitMix64(stream_seed(cfg, stream, seed) ^ 0xAB1EC7)
    n = rng.randint(cfg.n_obj[0], cfg.n_obj[1])
    objs = []
    for _ in range(n):
        w = rng.randint(cfg.size[0], cfg.size[1])
        h = rng.randint(cfg.size[0], cfg.size[1])
        x0 = rng.uniform() * max(cfg.W - w, 1)
        y0 = rng.uniform() * max(cfg.H - h, 1)
        sp = cfg.speed[0] + rng.uniform() * (cfg.speed[1] - cfg.speed[0])
        th = 2.0 * math.pi * rng.uniform()
        inten = cfg.intensity if cfg.intensity >= 0 else rng.randint(0, 255)
        objs.append((x0, y0, sp * math.cos(th), sp * math.sin(th), w, h, inten))
    return np.asarray(objs, dtype=np.float64).reshape(-1, 7)


def gen_stream(cfg: VideoConfig, stream: int, seed: int = BASE_SEED, t0: int = 0, T: int | None = None,
               out: np.ndarray | None = None) -> np.ndarray:
    """uint8 [T][H][W] frames t0..t0+T-1 of one stream."""
    lib = _load()
    T = cfg.T - t0 if T is None else T
    ss = stream_seed(cfg, stream, seed)
    bg = np.empty((cfg.H, cfg.W), dtype=np.float32)
    lib.cs_synth_background(cfg.W, cfg.H, cfg.period, ss, bg.ctypes.data)
    objs = np.ascontiguousarray(make_objects(cfg, stream, seed))
    if out is None:
        out = np.empty((T, cfg.H, cfg.W), dtype=np.uint8)
    assert out.flags.c_contiguous and out.dtype == np.uint8 and out.shape == (T, cfg.H, cfg.W)
    lib.cs_synth_frames(cfg.W, cfg.H, T, t0, bg.ctypes.data, cfg.drift_amp, cfg.drift_period,
                        objs.shape[0], objs.ctypes.data, cfg.sigma, ss ^ 0x5EED, out.ctypes.data)
    return out


def gen_video(cfg: VideoConfig, seed: int = BASE_SEED, out: np.ndarray | None = None,
              streams: range | None = None) -> np.ndarray:
    """uint8 [S][T][H][W] for the selected streams (default all)."""
    streams = range(cfg.S) if streams is None else streams
    if out is None:
        out = np.empty((len(streams), cfg.T, cfg.H, cfg.W), dtype=np.uint8)
    for i, s in enumerate(streams):
        gen_stream(cfg, s, seed, out=out[i])
    return out


def host_threads() -> int:
    return _load().cs_synth_num_threads()
