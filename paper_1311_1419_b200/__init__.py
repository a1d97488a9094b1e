"""paper_1311_1419_b200 -- B200-native encoder hot path of arXiv 1311.1419 (CS surveillance video).

Thin Python binding over the C ABI in ``include/cs_encoder.h`` (libcsenc.so): argument
marshalling only.  Every step of the path (GOP partition, block loads, residual, measurement,
output) runs in the sm_100a kernel; there is no CPU fallback -- importing this package without
the built library raises, and encoding on a machine without a B200 returns an error.

PyTorch is used for device memory and streams only: ``Encoder.encode_batch`` takes CUDA uint8
frame tensors and fills a CUDA float32 tensor on the current (or given) stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB, build as build_library

__all__ = ["Encoder", "FrameEncoder", "encode_batch_host_multi", "encode_batch_host_multi_q16", "CSError", "total_cr", "compression_ratio_cfg", "measurement_count_cfg", "plan_cfg",
           "validate_config", "lib", "LIB", "build_library", "version"]

CS_OK, CS_ERR_ARG, CS_ERR_UNSUPPORTED, CS_ERR_PHI, CS_ERR_CUDA, CS_ERR_OOM = range(6)
_ERR_NAMES = {1: "CS_ERR_ARG", 2: "CS_ERR_UNSUPPORTED", 3: "CS_ERR_PHI", 4: "CS_ERR_CUDA", 5: "CS_ERR_OOM"}


class CSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "tile_block_rows", "folds", "lanes", "chunk_rows", "stages", "key_resident", "box_w", "smem_bytes",
        "tmem_cols", "m_pad", "chains", "prefetch_items", "a_bufs", "d_bufs", "sms", "phi_stream")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcsenc.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"libcsenc.so not built ({LIB}); run paper_1311_1419_b200.build_library() "
                              "or __graft_entry__.build()")
        L = ctypes.CDLL(LIB)
        c_int, c_i64, c_dbl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        sig = {
            "cs_encoder_create": (c_int, [c_int, c_int, c_int, c_int, c_int, vp, ctypes.POINTER(vp)]),
            "cs_encoder_destroy": (c_int, [vp]),
            "cs_encoder_plan": (c_int, [vp, ctypes.POINTER(PlanInfo)]),
            "cs_encoder_set_trace": (c_int, [vp, vp, c_int]),
            "cs_encoder_set_stable_inputs": (c_int, [vp, c_int]),
            "cs_encoder_autotune": (c_int, [vp, vp, c_int, c_int, vp, c_int, c_int, vp]),
            "cs_encoder_num_candidates": (c_int, [vp]),
            "cs_encoder_set_candidate": (c_int, [vp, c_int]),
            "cs_encoder_candidate_index": (c_int, [vp]),
            "cs_encode_gop": (c_int, [vp, vp, c_int, vp, vp]),
            "cs_encode_batch": (c_int, [vp, vp, c_int, c_int, vp, vp]),
            "cs_encode_batch_gops": (c_int, [vp, vp, c_int, c_int, c_int, c_int, vp, vp]),
            "cs_encode_batch_host": (c_int, [vp, vp, c_int, c_int, vp]),
            "cs_encode_batch_host_multi": (c_int, [vp, c_int, vp, c_int, c_int, vp]),
            "cs_encode_batch_host_q16": (c_int, [vp, vp, c_int, c_int, c_int, vp, vp]),
            "cs_encode_batch_host_multi_q16": (c_int, [vp, c_int, vp, c_int, c_int, c_int, vp, vp]),
            "cs_encode_batch_q16": (c_int, [vp, vp, c_int, c_int, c_int, vp, vp, vp]),
            "cs_q16_scale_count": (c_i64, [vp, c_int, c_int, c_int]),
            "cs_adjoint": (c_int, [vp, vp, c_i64, vp, vp]),
            "cs_frame_encoder_create": (c_int, [c_int, c_int, c_int, c_int, vp, ctypes.POINTER(vp)]),
            "cs_frame_encoder_destroy": (c_int, [vp]),
            "cs_frame_measurement_count": (c_i64, [vp, c_int, c_int]),
            "cs_frame_encode_batch": (c_int, [vp, vp, c_int, c_int, vp, vp]),
            "cs_frame_encoder_set_trace": (c_int, [vp, vp, c_int]),
            "cs_key_qsteps": (c_int, [c_dbl, vp]),
            "cs_key_dct_basis": (None, [vp]),
            "cs_key_coef_count": (c_i64, [vp, c_int, c_int]),
            "cs_key_codec": (c_int, [vp, vp, c_int, c_int, vp, vp, vp, vp]),
            "cs_encode_batch_keys": (c_int, [vp, vp, c_int, c_int, vp, vp, vp]),
            "cs_encode_batch_chained": (c_int, [vp, vp, c_int, c_int, vp, vp]),
            "cs_encoder_set_gop_phis": (c_int, [vp, c_int, vp]),
            "cs_measurement_count": (c_i64, [vp, c_int, c_int]),
            "cs_compression_ratio": (c_dbl, [vp, c_int, c_dbl, c_int]),
            "cs_compression_ratio_cfg": (c_dbl, [c_int, c_int, c_int, c_int, c_int, c_int, c_dbl, c_int]),
            "cs_measurement_count_cfg": (c_i64, [c_int] * 7),
            "cs_total_cr": (c_dbl, [c_int, c_dbl, c_dbl]),
            "cs_validate_config": (c_int, [c_int] * 5 + [vp]),
            "cs_plan_cfg": (c_int, [c_int] * 7 + [ctypes.POINTER(PlanInfo)]),
            "cs_last_error": (ctypes.c_char_p, []),
            "cs_version": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != CS_OK:
        raise CSError(rc, lib().cs_last_error().decode())


def version() -> str:
    return lib().cs_version().decode()


def total_cr(G: int, key_cr: float, cs_cr: float) -> float:
    return lib().cs_total_cr(G, key_cr, cs_cr)


def compression_ratio_cfg(W, H, gop, B, M, T=0, key_cr=1.0, bits_per_measurement=8) -> float:
    return lib().cs_compression_ratio_cfg(W, H, gop, B, M, T, key_cr, bits_per_measurement)


def measurement_count_cfg(W, H, gop, B, M, n_seq, T) -> int:
    return lib().cs_measurement_count_cfg(W, H, gop, B, M, n_seq, T)


def validate_config(W, H, gop, B, M, phi_bits=None) -> int:
    """Status code of cs_validate_config (0 = OK)."""
    if phi_bits is None:
        return lib().cs_validate_config(W, H, gop, B, M, None)
    phi = np.ascontiguousarray(phi_bits, dtype=np.uint16)
    return lib().cs_validate_config(W, H, gop, B, M, phi.ctypes.data)


def plan_cfg(W, H, gop, B, M, smem_limit=232448, sms=148) -> dict:
    info = PlanInfo()
    _check(lib().cs_plan_cfg(W, H, gop, B, M, smem_limit, sms, ctypes.byref(info)))
    return info.as_dict()


def key_qsteps(quant_scale: float) -> np.ndarray:
    """cs_key_qsteps: int32 [8][8] quantiser steps of the key codec for a quant_scale."""
    out = np.zeros(64, dtype=np.int32)
    _check(lib().cs_key_qsteps(float(quant_scale), out.ctypes.data))
    return out.reshape(8, 8)


def key_dct_basis() -> np.ndarray:
    out = np.zeros(64, dtype=np.int32)
    lib().cs_key_dct_basis(out.ctypes.data)
    return out.reshape(8, 8)


def _ptr(t) -> int:
    return int(t.data_ptr())


def _stream_handle(stream, device=None) -> int:
    """cudaStream_t of `stream` (torch stream, raw handle or None = the current stream of `device`)."""
    if stream is None:
        import torch
        return int(torch.cuda.current_stream(device).cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def _dev_tensor(t, dtype, name, device=None, min_numel=None, shape=None):
    """ValueError unless t is a contiguous CUDA tensor of `dtype` (on `device`, with >= min_numel
    elements / exactly `shape`): the C ABI takes raw pointers and no lengths."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if min_numel is not None and t.numel() < min_numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {min_numel}")
    return t


def _host_buffer(a, dtype, name, min_numel=None, shape=None):
    """(pointer, array) of a contiguous HOST numpy array or CPU tensor of `dtype`; ValueError otherwise."""
    try:
        import torch
    except ImportError:   # pragma: no cover
        torch = None
    if isinstance(a, np.ndarray):
        if a.dtype != np.dtype(dtype):
            raise ValueError(f"{name} must be {np.dtype(dtype)}, got {a.dtype}")
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        ptr, n, shp = a.ctypes.data, a.size, a.shape
    elif torch is not None and isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise ValueError(f"{name} must be host memory")
        want = {np.uint8: torch.uint8, np.float32: torch.float32, np.int16: torch.int16}[dtype]
        if a.dtype != want:
            raise ValueError(f"{name} must be {want}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        ptr, n, shp = _ptr(a), a.numel(), tuple(a.shape)
    else:
        raise ValueError(f"{name} must be a numpy array or a CPU tensor")
    if shape is not None and tuple(shp) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(shp)}")
    if min_numel is not None and n < min_numel:
        raise ValueError(f"{name} has {n} elements, needs >= {min_numel}")
    return ptr


class Encoder:
    """cs_encoder_create(W, H, gop, B, M, phi) -- phi: uint16 [M][B*B] fp16 bit patterns (host)."""

    def __init__(self, W: int, H: int, gop: int, B: int, M: int, phi_bits):
        phi = np.ascontiguousarray(phi_bits, dtype=np.uint16)
        if phi.shape != (M, B * B):
            raise ValueError(f"phi must have shape ({M}, {B * B}), got {phi.shape}")
        self.W, self.H, self.G, self.B, self.M = W, H, gop, B, M
        self.nbx, self.nby = -(-W // B), -(-H // B)
        self.nblk = self.nbx * self.nby
        h = ctypes.c_void_p()
        _check(lib().cs_encoder_create(W, H, gop, B, M, phi.ctypes.data, ctypes.byref(h)))
        self._h = h
        import torch
        self.device = torch.device("cuda", torch.cuda.current_device())   # the encoder lives here (create)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().cs_encoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- tracing (debug timeline of CTA 0; see include/cs_encoder.h)
    TRACE_EVENTS = ("p_empty", "p_issued", "c_full", "c_aempty", "c_done", "m_afull", "m_issued", "e_dfull",
                    "e_done", "c_conv", "e_arrived", "e_rows", "k_start", "k_end")

    def set_trace(self, buf=None, cap: int = 0):
        """buf: CUDA int64 tensor of len(TRACE_EVENTS) * cap elements (None/0 disables)."""
        _check(lib().cs_encoder_set_trace(self._h, _ptr(buf) if buf is not None else None, cap))

    def set_stable_inputs(self, frames: bool = True, measurements: bool = False):
        """Promise that the frames of this encoder's encode calls (`frames`) / the measurements given to its
        adjoint (`measurements`) are never written by the kernel preceding the call in its stream: the
        kernel then loads and computes while that kernel drains, and only its output stores wait for it
        (cs_encoder_set_stable_inputs).  Do not promise `measurements` for adjoint(encode(x)) chains."""
        _check(lib().cs_encoder_set_stable_inputs(self._h, (1 if frames else 0) | (2 if measurements else 0)))

    # -- accounting
    def plan(self) -> dict:
        info = PlanInfo()
        _check(lib().cs_encoder_plan(self._h, ctypes.byref(info)))
        return info.as_dict()

    def measurement_count(self, n_seq: int, T: int) -> int:
        return lib().cs_measurement_count(self._h, n_seq, T)

    def compression_ratio(self, T: int = 0, key_cr: float = 1.0, bits_per_measurement: int = 8) -> float:
        return lib().cs_compression_ratio(self._h, T, key_cr, bits_per_measurement)

    def out_shape(self, n_seq: int, T: int):
        n_cs = n_seq * (T - -(-T // self.G))
        return (n_cs, self.nblk, self.M)

    # -- argument checks shared by every wrapper (the C ABI takes pointers and no lengths)
    def _frames(self, frames, name="frames"):
        """(n_seq, T) of a contiguous CUDA uint8 [n_seq][T][H][W] tensor on the encoder's device."""
        import torch
        _dev_tensor(frames, torch.uint8, name, device=self.device)
        if frames.dim() != 4 or tuple(frames.shape[2:]) != (self.H, self.W):
            raise ValueError(f"{name} must be [n_seq][T][{self.H}][{self.W}], got {tuple(frames.shape)}")
        return int(frames.shape[0]), int(frames.shape[1])

    def _out(self, out, shape, dtype, name="out"):
        import torch
        if out is None:
            return torch.empty(shape, dtype=dtype, device=self.device)
        n = 1
        for d in shape:
            n *= d
        return _dev_tensor(out, dtype, name, device=self.device, min_numel=n)

    def _call(self, fn, *args, stream=None):
        """Run a C-ABI launch with the encoder's device current, on `stream` (default: that device's
        current stream)."""
        import torch
        with torch.cuda.device(self.device):
            _check(fn(*args, _stream_handle(stream, self.device)))

    # -- encode (device tensors)
    def encode_batch(self, frames, out=None, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W] (contiguous); returns CUDA float32 [n_cs][nblk][M]."""
        import torch
        n_seq, T = self._frames(frames)
        out = self._out(out, self.out_shape(n_seq, T), torch.float32)
        self._call(lib().cs_encode_batch, self._h, _ptr(frames), n_seq, T, _ptr(out), stream=stream)
        return out

    def autotune(self, frames, out=None, max_candidates: int = 6, reps: int = 3, stream=None) -> dict:
        """Time the planner's top plans on these buffers and keep the fastest (outputs are bitwise
        identical across plans).  Returns the chosen plan."""
        import torch
        n_seq, T = self._frames(frames)
        out = self._out(out, self.out_shape(n_seq, T), torch.float32)
        self._call(lib().cs_encoder_autotune, self._h, _ptr(frames), n_seq, T, _ptr(out), max_candidates, reps,
                   stream=stream)
        return self.plan()

    def num_candidates(self) -> int:
        return lib().cs_encoder_num_candidates(self._h)

    def tuned_index(self) -> int:
        return lib().cs_encoder_candidate_index(self._h)

    def set_candidate(self, index: int) -> dict:
        _check(lib().cs_encoder_set_candidate(self._h, index))
        return self.plan()

    def gop_range_count(self, n_seq: int, T: int, gop_begin: int, gop_end: int) -> int:
        """Measurements cs_encode_batch_gops writes for GOPs [gop_begin, gop_end) of every stream."""
        n_cs = sum(max(0, min(self.G, T - g * self.G) - 1) for g in range(gop_begin, gop_end))
        return n_seq * n_cs * self.nblk * self.M

    def encode_batch_gops(self, frames, gop_begin: int, gop_end: int, out, stream=None):
        import torch
        n_seq, T = self._frames(frames)
        if not (0 <= gop_begin <= gop_end <= self.n_gops(T)):
            raise ValueError("GOP range out of bounds")
        _dev_tensor(out, torch.float32, "out", device=self.device,
                    min_numel=self.gop_range_count(n_seq, T, gop_begin, gop_end))
        self._call(lib().cs_encode_batch_gops, self._h, _ptr(frames), n_seq, T, gop_begin, gop_end, _ptr(out),
                   stream=stream)
        return out

    def encode_gop(self, frames, out=None, stream=None):
        """frames: CUDA uint8 [n][H][W], 1 <= n <= gop, frame 0 = key; returns [n-1][nblk][M]."""
        import torch
        _dev_tensor(frames, torch.uint8, "frames", device=self.device)
        if frames.dim() != 3 or tuple(frames.shape[1:]) != (self.H, self.W):
            raise ValueError(f"frames must be [n][{self.H}][{self.W}], got {tuple(frames.shape)}")
        n = int(frames.shape[0])
        out = self._out(out, (max(n - 1, 0), self.nblk, self.M), torch.float32)
        self._call(lib().cs_encode_gop, self._h, _ptr(frames), n, _ptr(out), stream=stream)
        return out

    # -- 16-bit quantisation (f1)
    Q16_FRAME, Q16_ROW = 0, 1

    def q16_scale_shape(self, n_seq: int, T: int, granularity: int = 0):
        n_cs = self.out_shape(n_seq, T)[0]
        return (n_cs, self.nby) if granularity == self.Q16_ROW else (n_cs,)

    def encode_batch_q16(self, frames, granularity: int = 0, codes=None, scales=None, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W]; returns (codes int16 [n_cs][nblk][M], scales fp32
        [n_cs] (Q16_FRAME, SPEC's per-frame scale) or [n_cs][nby] (Q16_ROW, per block row))."""
        import torch
        n_seq, T = self._frames(frames)
        codes = self._out(codes, self.out_shape(n_seq, T), torch.int16, "codes")
        scales = self._out(scales, self.q16_scale_shape(n_seq, T, granularity), torch.float32, "scales")
        self._call(lib().cs_encode_batch_q16, self._h, _ptr(frames), n_seq, T, granularity, _ptr(codes),
                   _ptr(scales), stream=stream)
        return codes, scales

    # -- closed-loop key frame (f4; Eq. 2-3)
    def n_gops(self, T: int) -> int:
        return -(-T // self.G)

    def key_codec(self, frames, qsteps, keys=None, coef=None, want_coef=True, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W]; qsteps: int [8][8] (see key_qsteps).  Returns
        (decoded keys uint8 [n_seq][ceil(T/G)][H][W], coefficients int16 [...][nby8][nbx8][8][8] or None)."""
        import torch
        n_seq, T = self._frames(frames)
        ng = self.n_gops(T)
        keys = self._out(keys, (n_seq, ng, self.H, self.W), torch.uint8, "keys")
        if coef is not None or want_coef:
            coef = self._out(coef, (n_seq, ng, -(-self.H // 8), -(-self.W // 8), 8, 8), torch.int16, "coef")
        q = np.ascontiguousarray(qsteps, dtype=np.int32).ravel()
        if q.size != 64:
            raise ValueError("qsteps must have 64 entries")
        self._call(lib().cs_key_codec, self._h, _ptr(frames), n_seq, T, q.ctypes.data,
                   _ptr(coef) if coef is not None else None, _ptr(keys), stream=stream)
        return keys, coef

    def encode_batch_keys(self, frames, keys, out=None, stream=None):
        """cs_encode_batch with residuals against keys [n_seq][ceil(T/G)][H][W] (decoded key frames)."""
        import torch
        n_seq, T = self._frames(frames)
        _dev_tensor(keys, torch.uint8, "keys", device=self.device, shape=(n_seq, self.n_gops(T), self.H, self.W))
        out = self._out(out, self.out_shape(n_seq, T), torch.float32)
        self._call(lib().cs_encode_batch_keys, self._h, _ptr(frames), n_seq, T, _ptr(keys), _ptr(out), stream=stream)
        return out

    def set_gop_phis(self, phis=None):
        """Per-GOP matrices: phis uint16 [n][M][B*B]; GOP g uses phis[g % n].  None or
        an empty list restores the single Phi."""
        import torch
        with torch.cuda.device(self.device):
            if phis is None or len(phis) == 0:
                _check(lib().cs_encoder_set_gop_phis(self._h, 0, None))
                return
            a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.uint16) for x in phis]))
            if a.shape[1:] != (self.M, self.B * self.B):
                raise ValueError(f"phis must be [n][{self.M}][{self.B * self.B}], got {a.shape}")
            _check(lib().cs_encoder_set_gop_phis(self._h, a.shape[0], a.ctypes.data))

    def encode_batch_chained(self, frames, out=None, stream=None):
        """Eq. 3 literal variant: residual of every CS frame against the previous raw frame."""
        import torch
        n_seq, T = self._frames(frames)
        out = self._out(out, self.out_shape(n_seq, T), torch.float32)
        self._call(lib().cs_encode_batch_chained, self._h, _ptr(frames), n_seq, T, _ptr(out), stream=stream)
        return out

    def encode_batch_closed_loop(self, frames, qsteps, out=None, stream=None):
        """Eq. 2-3 closed loop: key codec (decoded keys) then the measurement against them (2 launches)."""
        keys, coef = self.key_codec(frames, qsteps, stream=stream)
        return self.encode_batch_keys(frames, keys, out, stream), keys, coef

    # -- adjoint / back-projection (f3)
    def adjoint(self, meas, out=None, stream=None):
        """meas: CUDA float32 [n][nblk][M] (contiguous); returns CUDA float32 [n][H][W] = Phi^T y per
        block laid back into the frame."""
        import torch
        _dev_tensor(meas, torch.float32, "meas", device=self.device)
        n = meas.numel() // (self.nblk * self.M)
        if meas.numel() != n * self.nblk * self.M:
            raise ValueError(f"meas must hold whole frames of {self.nblk * self.M} measurements")
        out = self._out(out, (n, self.H, self.W), torch.float32)
        self._call(lib().cs_adjoint, self._h, _ptr(meas), n, _ptr(out), stream=stream)
        return out

    # -- encode (host buffers)
    def _host_frames(self, frames):
        if frames.ndim != 4 or tuple(frames.shape[2:]) != (self.H, self.W):
            raise ValueError(f"frames must be [n_seq][T][{self.H}][{self.W}], got {tuple(frames.shape)}")
        return int(frames.shape[0]), int(frames.shape[1]), _host_buffer(frames, np.uint8, "frames")

    def encode_batch_host(self, frames, out=None):
        """frames: host uint8 [n_seq][T][H][W] (numpy or CPU tensor, pinned for full bandwidth);
        copies in, encodes, copies out; returns host float32 [n_cs][nblk][M]."""
        n_seq, T, fp = self._host_frames(frames)
        if out is None:
            out = np.empty(self.out_shape(n_seq, T), dtype=np.float32)
        op = _host_buffer(out, np.float32, "out", min_numel=self.measurement_count(n_seq, T))
        _check(lib().cs_encode_batch_host(self._h, fp, n_seq, T, op))
        return out

    def encode_batch_host_q16(self, frames, granularity: int = 0, codes=None, scales=None):
        """Host-buffer form of encode_batch_q16 (f1): frames in, int16 codes + fp32 scales out; the
        device->host copy moves 2 B per measurement instead of 4."""
        n_seq, T, fp = self._host_frames(frames)
        if codes is None:
            codes = np.empty(self.out_shape(n_seq, T), dtype=np.int16)
        if scales is None:
            scales = np.empty(self.q16_scale_shape(n_seq, T, granularity), dtype=np.float32)
        cp = _host_buffer(codes, np.int16, "codes", min_numel=self.measurement_count(n_seq, T))
        sp = _host_buffer(scales, np.float32, "scales",
                          min_numel=lib().cs_q16_scale_count(self._h, n_seq, T, granularity))
        _check(lib().cs_encode_batch_host_q16(self._h, fp, n_seq, T, granularity, cp, sp))
        return codes, scales


def _multi_args(encoders, frames):
    if not encoders:
        raise ValueError("need at least one encoder")
    e0 = encoders[0]
    for e in encoders:
        if (e.W, e.H, e.G) != (e0.W, e0.H, e0.G):
            raise ValueError("encoders must share W, H and gop")
    return e0._host_frames(frames)


def encode_batch_host_multi(encoders, frames, outs=None):
    """Several encoders (same W, H, gop) over the same HOST frames [n_seq][T][H][W]: each frame group
    crosses PCIe once.  frames: numpy or (pinned) CPU tensor; returns the list of host outputs."""
    n_seq, T, fp = _multi_args(encoders, frames)
    if outs is None:
        outs = [np.empty(e.out_shape(n_seq, T), dtype=np.float32) for e in encoders]
    if len(outs) != len(encoders):
        raise ValueError("one output per encoder")
    hs = (ctypes.c_void_p * len(encoders))(*[e._h.value for e in encoders])
    ps = (ctypes.c_void_p * len(outs))(*[_host_buffer(o, np.float32, "out", min_numel=e.measurement_count(n_seq, T))
                                         for e, o in zip(encoders, outs)])
    _check(lib().cs_encode_batch_host_multi(ctypes.cast(hs, ctypes.c_void_p), len(encoders), fp, n_seq, T,
                                            ctypes.cast(ps, ctypes.c_void_p)))
    return outs


def encode_batch_host_multi_q16(encoders, frames, granularity: int = 0, outs=None):
    """cs_encode_batch_host_multi_q16: every encoder's int16 codes + fp32 scales of the same HOST frames.
    Returns the list of (codes, scales) host pairs."""
    n_seq, T, fp = _multi_args(encoders, frames)
    if outs is None:
        outs = [(np.empty(e.out_shape(n_seq, T), dtype=np.int16),
                 np.empty(e.q16_scale_shape(n_seq, T, granularity), dtype=np.float32)) for e in encoders]
    if len(outs) != len(encoders):
        raise ValueError("one (codes, scales) pair per encoder")
    hs = (ctypes.c_void_p * len(encoders))(*[e._h.value for e in encoders])
    cps = (ctypes.c_void_p * len(outs))(*[_host_buffer(c, np.int16, "codes", min_numel=e.measurement_count(n_seq, T))
                                          for e, (c, _) in zip(encoders, outs)])
    sps = (ctypes.c_void_p * len(outs))(*[_host_buffer(sc, np.float32, "scales",
                                                       min_numel=lib().cs_q16_scale_count(e._h, n_seq, T, granularity))
                                          for e, (_, sc) in zip(encoders, outs)])
    _check(lib().cs_encode_batch_host_multi_q16(ctypes.cast(hs, ctypes.c_void_p), len(encoders), fp, n_seq, T,
                                                granularity, ctypes.cast(cps, ctypes.c_void_p),
                                                ctypes.cast(sps, ctypes.c_void_p)))
    return outs


class FrameEncoder:
    """f2: paper-faithful frame-level measurement y = A vec(F_cs - F_key) (Eq. 1) with one
    dense A: uint16 [m][W*H] fp16 bit patterns (host), copied to the device."""

    def __init__(self, W: int, H: int, gop: int, m: int, A_bits):
        A = np.ascontiguousarray(A_bits, dtype=np.uint16)
        if A.shape != (m, W * H):
            raise ValueError(f"A must have shape ({m}, {W * H}), got {A.shape}")
        self.W, self.H, self.G, self.m = W, H, gop, m
        h = ctypes.c_void_p()
        _check(lib().cs_frame_encoder_create(W, H, gop, m, A.ctypes.data, ctypes.byref(h)))
        self._h = h
        import torch
        self.device = torch.device("cuda", torch.cuda.current_device())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().cs_frame_encoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def out_shape(self, n_seq: int, T: int):
        return (n_seq * (T - -(-T // self.G)), self.m)

    def set_trace(self, buf=None, cap: int = 0):
        """buf: CUDA int64 tensor of 4 * cap elements (None/0 disables); see cs_frame_encoder_set_trace."""
        _check(lib().cs_frame_encoder_set_trace(self._h, _ptr(buf) if buf is not None else None, cap))

    def encode_batch(self, frames, out=None, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W]; returns CUDA float32 [n_cs][m]."""
        import torch
        _dev_tensor(frames, torch.uint8, "frames", device=self.device)
        if frames.dim() != 4 or tuple(frames.shape[2:]) != (self.H, self.W):
            raise ValueError(f"frames must be [n_seq][T][{self.H}][{self.W}], got {tuple(frames.shape)}")
        n_seq, T = int(frames.shape[0]), int(frames.shape[1])
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=self.device)
        _dev_tensor(out, torch.float32, "out", device=self.device,
                    min_numel=lib().cs_frame_measurement_count(self._h, n_seq, T))
        with torch.cuda.device(self.device):
            _check(lib().cs_frame_encode_batch(self._h, _ptr(frames), n_seq, T, _ptr(out),
                                               _stream_handle(stream, self.device)))
        return out
