// cs_internal.h -- host-side declarations shared by the translation units of libcsenc.so
// (cs_common.cu, cs_encoder.cu, cs_adjoint.cu, cs_keys.cu, cs_frame.cu).  Not installed: the public
// contract is include/cs_encoder.h.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/cs_encoder.h"

namespace csenc {
namespace host {

// thread-local error string behind cs_last_error(); returns `code`
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
float half_bits_to_float(uint16_t h);
// Tuning / debug knobs (CSENC_* environment variables): read only in CSENC_TUNING=1 builds
// (tools/, libcsenc_checks.so); the product library always uses the defaults.
int env_int(const char* name, int dflt);
#ifndef CSENC_TUNING
#define CSENC_TUNING 0
#endif

// Device-buffer calls launch on the calling thread's current device: it must be the device the
// object was created on (Phi, workspaces and kernel attributes live there).  CS_ERR_ARG otherwise.
int check_device(int device);
// Host-buffer calls (synchronous) switch to the object's device for their duration and restore the
// caller's current device afterwards.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) == cudaSuccess) ok = prev == device || cudaSetDevice(device) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (ok && prev >= 0) cudaSetDevice(prev);
    }
};

// NVTX range around an ABI call (profiling: ncu --nvtx / nsys), when CSENC_NVTX=1 (read once);
// nvtx3 is header-only: no extra link dependency, a no-op without an attached tool
bool nvtx_enabled();
struct NvtxScope {
    bool on;
    explicit NvtxScope(const char* name) : on(nvtx_enabled()) {
        if (on) nvtxRangePushA(name);
    }
    ~NvtxScope() {
        if (on) nvtxRangePop();
    }
};

// GOP accounting (a1)
inline long long cs_frames_per_stream(int T, int G) { return (long long)T - cdiv(T, G); }
inline long long cs_frames_in_gops(int T, int G, int g0, int g1) {
    long long n = 0;
    for (int g = g0; g < g1; ++g) n += (long long)std::max(0, std::min(G, T - g * G) - 1);
    return n;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode_tiled();

// ------------------------------------------------------------------------- K1 tiling plan
struct Plan {
    int T_r = 0, F = 0, L = 0, n_tiles = 0;
    int chunk_rows = 0, n_chunks = 0, chunk_k = 0;
    int pieces = 0, piece_rows = 0, single_piece = 0;
    uint32_t piece_bytes = 0, stage_cs_bytes = 0, stage_bytes = 0, key_bytes = 0;
    int key_resident = 0, key_regs = 0, key_chunk = 0, n_stages = 0, prefetch_items = 0;
    int phi_stream = 0;                       // Phi K-slices ride in the stages instead of staying resident
    uint32_t phi_slice_bytes = 0, stage_phi_off = 0;
    uint32_t off_tab = 0, off_epi = 0, off_phi = 0, off_key = 0, off_stage = 0, smem_bytes = 0;
    int a_cols = 0, d_cols = 0, tmem_cols = 0, n_abuf = 2, n_dbuf = 2;
    double score = -1.0;
};

struct Geometry {
    int W, H, G, B, M, N, Mpad, nbx, nby, nblk;
};

}  // namespace host
}  // namespace csenc

// the opaque handle of include/cs_encoder.h
struct cs_encoder {
    csenc::host::Geometry geo{};
    csenc::host::Plan plan{};
    int device = 0;
    int sms = 0;
    int smem_limit = 0;
    void* phi_dev = nullptr;
    uint32_t phi_bytes = 0;
    uint32_t idesc = 0, lbo = 0, sbo = 0;
    std::mutex ws_mu;  // host-path workspace
    // host-path workspace
    uint8_t* ws_frames = nullptr;
    void* ws_out = nullptr;           // measurements (fp32 or int16 codes) + scales
    size_t ws_frames_bytes = 0, ws_out_bytes = 0;
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr};
    std::vector<csenc::host::Plan> candidates;  // planner's ranked plans (autotune)
    int chained_plan = -1;         // best KEY_STREAMED candidate (previous-frame reference), -1 = none
    int row_plan = -1;             // best candidate with <= kRowSlots block rows per tile (CS_Q16_ROW), -1 = none
    void* phis_dev = nullptr;      // per-GOP Phi copies (arranged like phi_dev), n_phis of phi_bytes
    int n_phis = 0;
    int tuned = -1;                // index of the autotuned plan, -1 = model choice
    void* zeros_dev = nullptr;   // piece_rows * W zero bytes: source for frame rows beyond H
    size_t zeros_bytes = 0;
    unsigned long long* trace = nullptr;  // device buffer (debug timeline), caller-owned
    int trace_cap = 0;
    int stable_inputs = 0;         // cs_encoder_set_stable_inputs flags: loads may start before the previous kernel completes
    std::vector<cudaEvent_t> hev;
    // stream-ordered scratch (q16 workspaces): the encoder's own memory pool, created on first use,
    // that keeps its memory between calls (release threshold = max) so repeated calls do not map
    // and unmap device memory
    cudaMemPool_t pool = nullptr;
    std::mutex pool_mu;
    // f3 adjoint (K3): Phi^T chunks (tf32, no-swizzle K-major), plan; phiT_dev == nullptr when M % 4 != 0
    void* phiT_dev = nullptr;
    int adj_Kc = 0, adj_n_kc = 0, adj_Nc = 0, adj_n_nc = 0, adj_stages = 0;
    uint32_t adj_chunk_bytes = 0, adj_stage_bytes = 0, adj_smem = 0;
};

// f2: frame-level measurement matrix A (m x n, n = W*H) and its geometry

namespace csenc {
namespace host {
// f3 (cs_adjoint.cu): Phi^T chunks and plan at create; per-kernel SMEM attribute
int prepare_adjoint(cs_encoder* e, const uint16_t* phi_fp16);
// stream-ordered scratch from the encoder's pool (created on first use); free with cudaFreeAsync
cudaError_t scratch_alloc(cs_encoder* e, void** ptr, size_t bytes, cudaStream_t st);
cudaError_t adjoint_set_smem_attr(int bytes);
}  // namespace host
}  // namespace csenc
