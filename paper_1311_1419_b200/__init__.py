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

__all__ = ["Encoder", "CSError", "total_cr", "compression_ratio_cfg", "measurement_count_cfg", "plan_cfg",
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
            "cs_encoder_autotune": (c_int, [vp, vp, c_int, c_int, vp, c_int, c_int, vp]),
            "cs_encoder_num_candidates": (c_int, [vp]),
            "cs_encoder_set_candidate": (c_int, [vp, c_int]),
            "cs_encoder_candidate_index": (c_int, [vp]),
            "cs_encode_gop": (c_int, [vp, vp, c_int, vp, vp]),
            "cs_encode_batch": (c_int, [vp, vp, c_int, c_int, vp, vp]),
            "cs_encode_batch_gops": (c_int, [vp, vp, c_int, c_int, c_int, c_int, vp, vp]),
            "cs_encode_batch_host": (c_int, [vp, vp, c_int, c_int, vp]),
            "cs_encode_batch_host_multi": (c_int, [vp, c_int, vp, c_int, c_int, vp]),
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


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


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
                    "e_done", "c_conv", "e_arrived", "e_rows")

    def set_trace(self, buf=None, cap: int = 0):
        """buf: CUDA int64 tensor of len(TRACE_EVENTS) * cap elements (None/0 disables)."""
        _check(lib().cs_encoder_set_trace(self._h, _ptr(buf) if buf is not None else None, cap))

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

    # -- encode (device tensors)
    def encode_batch(self, frames, out=None, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W] (contiguous); returns CUDA float32 [n_cs][nblk][M]."""
        import torch
        assert frames.is_cuda and frames.dtype == torch.uint8 and frames.is_contiguous()
        n_seq, T, H, W = frames.shape
        assert (H, W) == (self.H, self.W)
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=frames.device)
        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()
        assert out.numel() >= self.measurement_count(n_seq, T)
        _check(lib().cs_encode_batch(self._h, _ptr(frames), n_seq, T, _ptr(out), _stream_handle(stream)))
        return out

    def autotune(self, frames, out=None, max_candidates: int = 6, reps: int = 3, stream=None) -> dict:
        """Time the planner's top plans on these buffers and keep the fastest (outputs are bitwise
        identical across plans).  Returns the chosen plan."""
        import torch
        n_seq, T = frames.shape[:2]
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=frames.device)
        _check(lib().cs_encoder_autotune(self._h, _ptr(frames), n_seq, T, _ptr(out), max_candidates, reps,
                                         _stream_handle(stream)))
        return self.plan()

    def num_candidates(self) -> int:
        return lib().cs_encoder_num_candidates(self._h)

    def tuned_index(self) -> int:
        return lib().cs_encoder_candidate_index(self._h)

    def set_candidate(self, index: int) -> dict:
        _check(lib().cs_encoder_set_candidate(self._h, index))
        return self.plan()

    def encode_batch_gops(self, frames, gop_begin: int, gop_end: int, out, stream=None):
        n_seq, T = frames.shape[:2]
        _check(lib().cs_encode_batch_gops(self._h, _ptr(frames), n_seq, T, gop_begin, gop_end, _ptr(out),
                                          _stream_handle(stream)))
        return out

    def encode_gop(self, frames, out=None, stream=None):
        """frames: CUDA uint8 [n][H][W], 1 <= n <= gop, frame 0 = key; returns [n-1][nblk][M]."""
        import torch
        n = frames.shape[0]
        if out is None:
            out = torch.empty((max(n - 1, 0), self.nblk, self.M), dtype=torch.float32, device=frames.device)
        _check(lib().cs_encode_gop(self._h, _ptr(frames), n, _ptr(out), _stream_handle(stream)))
        return out

    # -- 16-bit quantisation (f1)
    Q16_FRAME, Q16_ROW, Q16_FRAME_1PASS = 0, 1, 2

    def q16_scale_shape(self, n_seq: int, T: int, granularity: int = 0):
        n_cs = self.out_shape(n_seq, T)[0]
        return (n_cs, self.nby) if granularity == self.Q16_ROW else (n_cs,)

    def encode_batch_q16(self, frames, granularity: int = 0, codes=None, scales=None, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W]; returns (codes int16 [n_cs][nblk][M], scales fp32
        [n_cs] (Q16_FRAME, SPEC's per-frame scale) or [n_cs][nby] (Q16_ROW, per block row))."""
        import torch
        assert frames.is_cuda and frames.dtype == torch.uint8 and frames.is_contiguous()
        n_seq, T, H, W = frames.shape
        assert (H, W) == (self.H, self.W)
        if codes is None:
            codes = torch.empty(self.out_shape(n_seq, T), dtype=torch.int16, device=frames.device)
        if scales is None:
            scales = torch.empty(self.q16_scale_shape(n_seq, T, granularity), dtype=torch.float32,
                                 device=frames.device)
        assert codes.is_cuda and codes.dtype == torch.int16 and codes.is_contiguous()
        assert scales.is_cuda and scales.dtype == torch.float32 and scales.is_contiguous()
        assert codes.numel() >= self.measurement_count(n_seq, T)
        assert scales.numel() >= lib().cs_q16_scale_count(self._h, n_seq, T, granularity)
        _check(lib().cs_encode_batch_q16(self._h, _ptr(frames), n_seq, T, granularity, _ptr(codes), _ptr(scales),
                                         _stream_handle(stream)))
        return codes, scales

    # -- closed-loop key frame (f4; Eq. 2-3)
    def n_gops(self, T: int) -> int:
        return -(-T // self.G)

    def key_codec(self, frames, qsteps, keys=None, coef=None, want_coef=True, stream=None):
        """frames: CUDA uint8 [n_seq][T][H][W]; qsteps: int [8][8] (see key_qsteps).  Returns
        (decoded keys uint8 [n_seq][ceil(T/G)][H][W], coefficients int16 [...][nby8][nbx8][8][8] or None)."""
        import torch
        assert frames.is_cuda and frames.dtype == torch.uint8 and frames.is_contiguous()
        n_seq, T = frames.shape[:2]
        ng = self.n_gops(T)
        if keys is None:
            keys = torch.empty((n_seq, ng, self.H, self.W), dtype=torch.uint8, device=frames.device)
        if coef is None and want_coef:
            coef = torch.empty((n_seq, ng, -(-self.H // 8), -(-self.W // 8), 8, 8), dtype=torch.int16,
                               device=frames.device)
        q = np.ascontiguousarray(qsteps, dtype=np.int32).ravel()
        assert q.size == 64
        _check(lib().cs_key_codec(self._h, _ptr(frames), n_seq, T, q.ctypes.data,
                                  _ptr(coef) if coef is not None else None, _ptr(keys), _stream_handle(stream)))
        return keys, coef

    def encode_batch_keys(self, frames, keys, out=None, stream=None):
        """cs_encode_batch with residuals against keys [n_seq][ceil(T/G)][H][W] (decoded key frames)."""
        import torch
        n_seq, T = frames.shape[:2]
        assert keys.is_cuda and keys.dtype == torch.uint8 and keys.is_contiguous()
        assert keys.shape == (n_seq, self.n_gops(T), self.H, self.W)
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=frames.device)
        _check(lib().cs_encode_batch_keys(self._h, _ptr(frames), n_seq, T, _ptr(keys), _ptr(out),
                                          _stream_handle(stream)))
        return out

    def set_gop_phis(self, phis=None):
        """Per-GOP matrices: phis uint16 [n][M][B*B]; GOP g uses phis[g % n].  None or
        an empty list restores the single Phi."""
        if phis is None or len(phis) == 0:
            _check(lib().cs_encoder_set_gop_phis(self._h, 0, None))
            return
        a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.uint16) for x in phis]))
        assert a.shape[1:] == (self.M, self.B * self.B)
        _check(lib().cs_encoder_set_gop_phis(self._h, a.shape[0], a.ctypes.data))

    def encode_batch_chained(self, frames, out=None, stream=None):
        """Eq. 3 literal variant: residual of every CS frame against the previous raw frame."""
        import torch
        n_seq, T = frames.shape[:2]
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=frames.device)
        _check(lib().cs_encode_batch_chained(self._h, _ptr(frames), n_seq, T, _ptr(out), _stream_handle(stream)))
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
        assert meas.is_cuda and meas.dtype == torch.float32 and meas.is_contiguous()
        n = meas.numel() // (self.nblk * self.M)
        assert meas.numel() == n * self.nblk * self.M
        if out is None:
            out = torch.empty((n, self.H, self.W), dtype=torch.float32, device=meas.device)
        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.numel() >= n * self.H * self.W
        _check(lib().cs_adjoint(self._h, _ptr(meas), n, _ptr(out), _stream_handle(stream)))
        return out

    # -- encode (host buffers)
    def encode_batch_host(self, frames, out=None):
        """frames: host uint8 [n_seq][T][H][W] (numpy or CPU tensor, pinned for full bandwidth);
        copies in, encodes, copies out; returns host float32 [n_cs][nblk][M]."""
        n_seq, T = frames.shape[:2]
        if out is None:
            out = np.empty(self.out_shape(n_seq, T), dtype=np.float32)
        fp = frames.ctypes.data if isinstance(frames, np.ndarray) else _ptr(frames)
        op = out.ctypes.data if isinstance(out, np.ndarray) else _ptr(out)
        _check(lib().cs_encode_batch_host(self._h, fp, n_seq, T, op))
        return out


def encode_batch_host_multi(encoders, frames, outs=None):
    """Several encoders (same W, H, gop) over the same HOST frames [n_seq][T][H][W]: each frame group
    crosses PCIe once.  frames: numpy or (pinned) CPU tensor; returns the list of host outputs."""
    n_seq, T = frames.shape[:2]
    if outs is None:
        outs = [np.empty(e.out_shape(n_seq, T), dtype=np.float32) for e in encoders]
    hs = (ctypes.c_void_p * len(encoders))(*[e._h.value for e in encoders])
    ps = (ctypes.c_void_p * len(outs))(*[o.ctypes.data if isinstance(o, np.ndarray) else _ptr(o) for o in outs])
    fp = frames.ctypes.data if isinstance(frames, np.ndarray) else _ptr(frames)
    _check(lib().cs_encode_batch_host_multi(ctypes.cast(hs, ctypes.c_void_p), len(encoders), fp, n_seq, T,
                                            ctypes.cast(ps, ctypes.c_void_p)))
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
        assert frames.is_cuda and frames.dtype == torch.uint8 and frames.is_contiguous()
        n_seq, T, H, W = frames.shape
        assert (H, W) == (self.H, self.W)
        if out is None:
            out = torch.empty(self.out_shape(n_seq, T), dtype=torch.float32, device=frames.device)
        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()
        assert out.numel() >= lib().cs_frame_measurement_count(self._h, n_seq, T)
        _check(lib().cs_frame_encode_batch(self._h, _ptr(frames), n_seq, T, _ptr(out), _stream_handle(stream)))
        return out
