"""C-ABI checks that need no GPU: libcsenc.so loads, exports every function include/cs_encoder.h
declares, validates arguments exactly as documented, and its host-only accounting matches the
oracle (the oracle is pinned to Table I in test_oracle_pins.py)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth
import paper_1311_1419_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cs_encoder.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    P.build_library()
    lib = ctypes.CDLL(P.LIB)
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n


def test_version_and_error_string():
    assert "sm_100a" in P.version()
    assert P.lib().cs_encoder_destroy(None) == P.CS_OK
    # setters validate before touching the device
    assert P.lib().cs_encoder_set_stable_inputs(None, 1) == P.CS_ERR_ARG
    assert b"NULL" in P.lib().cs_last_error()


@pytest.mark.parametrize("args,code", [
    ((176, 144, 4, 16, 64), P.CS_OK),
    ((0, 144, 4, 16, 64), P.CS_ERR_ARG),
    ((176, 144, 0, 16, 64), P.CS_ERR_ARG),
    ((176, 144, 4, 12, 64), P.CS_ERR_UNSUPPORTED),   # B not in {8,16,32}
    ((176, 144, 4, 16, 257), P.CS_ERR_ARG),          # M > N
    ((176, 144, 4, 16, 0), P.CS_ERR_ARG),
    ((180, 144, 4, 16, 64), P.CS_ERR_UNSUPPORTED),   # W % 16
    ((640, 480, 16, 32, 96), P.CS_OK),               # Phi > 160 KB: streamed in K-slices
    ((640, 480, 16, 32, 256), P.CS_OK),
    ((640, 480, 16, 32, 80), P.CS_OK),
    ((16, 16, 1, 16, 256), P.CS_OK),                 # lossless M = N
])
def test_validation_codes(args, code):
    assert P.validate_config(*args) == code


def test_phi_validation():
    phi = synth.phi_from_seed(1, 16, 256)
    assert P.validate_config(64, 32, 4, 16, 16, phi) == P.CS_OK
    bad = phi.copy()
    bad[3, 7] = 0x7E00                                  # NaN
    assert P.validate_config(64, 32, 4, 16, 16, bad) == P.CS_ERR_PHI
    big = phi.copy()
    big[0, 0] = np.float16(4096.0).view(np.uint16)     # |Phi| > 2048 breaks the oracle's exactness
    assert P.validate_config(64, 32, 4, 16, 16, big) == P.CS_ERR_PHI
    ok = phi.copy()
    ok[0, 0] = np.float16(2048.0).view(np.uint16)
    assert P.validate_config(64, 32, 4, 16, 16, ok) == P.CS_OK


def test_cr_accounting_matches_oracle():
    for name, cfg in synth.CONFIGS.items():
        for M in cfg.Ms:
            for T in (0, cfg.T, 3, 1):
                for key_cr, bits in ((1.0, 8), (23.0, 8), (1.0, 32)):
                    a = P.compression_ratio_cfg(cfg.W, cfg.H, cfg.G, cfg.B, M, T, key_cr, bits)
                    b = oracle.compression_ratio(cfg.W, cfg.H, cfg.G, cfg.B, M, T, key_cr, bits)
                    assert a == pytest.approx(b, rel=1e-12), (name, M, T)
    for G, kc, cc in ((3, 23, 40), (7, 23, 80), (1, 23, 60)):
        assert P.total_cr(G, kc, cc) == pytest.approx(oracle.total_cr(G, kc, cc), rel=1e-15)
    assert P.total_cr(0, 23, 40) < 0 and P.compression_ratio_cfg(0, 1, 1, 16, 1) < 0


def test_measurement_count():
    for cfg in synth.CONFIGS.values():
        for M in cfg.Ms:
            nblk = -(-cfg.W // cfg.B) * -(-cfg.H // cfg.B)
            want = cfg.S * oracle.cs_frame_count(cfg.T, cfg.G) * nblk * M
            assert P.measurement_count_cfg(cfg.W, cfg.H, cfg.G, cfg.B, M, cfg.S, cfg.T) == want


def test_plans_fit_b200_limits():
    """Every config's plan fits 227 KB SMEM / 512 TMEM columns with >= 2 ring slots."""
    for cfg in synth.CONFIGS.values():
        for M in cfg.Ms:
            p = P.plan_cfg(cfg.W, cfg.H, cfg.G, cfg.B, M)
            assert p["smem_bytes"] <= 232448 and p["tmem_cols"] <= 512 and p["stages"] >= 2
            assert p["folds"] * p["lanes"] >= p["tile_block_rows"] * -(-cfg.W // cfg.B)
            assert p["lanes"] <= 128
    for args in [(16, 1, 2, 16, 16), (48, 40, 3, 32, 5), (2048, 8, 2, 8, 64), (3840, 2160, 8, 16, 128),
                 (64, 64, 2, 32, 80), (16, 16, 2, 16, 256), (3840, 2160, 8, 8, 4), (640, 480, 16, 32, 96),
                 (640, 480, 16, 32, 128), (640, 480, 16, 32, 256), (96, 64, 3, 32, 256), (1920, 1080, 8, 32, 192)]:
        p = P.plan_cfg(*args)
        assert p["smem_bytes"] <= 232448 and p["tmem_cols"] <= 512


def test_key_codec_tables_match_oracle():
    """The library's fixed-point DCT basis and quantiser steps (independent copies) equal the
    oracle's definitions (R21), including round-half-even ties of quant_scale * table."""
    import oracle
    assert np.array_equal(P.key_dct_basis(), oracle.dct_basis_int())
    for qs in (0.01, 0.5, 1.0, 1.5, 2.25, 7.0, 100.0, 1000.0):
        assert np.array_equal(P.key_qsteps(qs), oracle.key_qsteps(qs)), qs
    with pytest.raises(P.CSError):
        P.key_qsteps(0.0)
