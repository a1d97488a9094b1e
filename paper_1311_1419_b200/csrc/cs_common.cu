// cs_common.cu -- error state, version string and small host utilities shared by libcsenc.so.
#include <cmath>
#include <cstdlib>
#include <string>

#include "cs_internal.h"

namespace csenc {
namespace host {

thread_local std::string g_err;   // behind cs_last_error()

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(CS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

float half_bits_to_float(uint16_t h) {
    uint32_t s = (h >> 15) & 1u, e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
    float v;
    if (e == 0)
        v = std::ldexp((float)m, -24);
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = std::ldexp((float)(m | 0x400u), (int)e - 25);
    return s ? -v : v;
}

bool nvtx_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("CSENC_NVTX");
        return v != nullptr && std::atoi(v) != 0;
    }();
    return on;
}

int check_device(int device) {
    int cur = -1;
    const cudaError_t err = cudaGetDevice(&cur);
    if (err != cudaSuccess) return cuda_fail(err, "cudaGetDevice");
    if (cur != device)
        return fail(CS_ERR_ARG, "the current device (" + std::to_string(cur) + ") is not the device the encoder was created on (" +
                                    std::to_string(device) + "): call cudaSetDevice first");
    return CS_OK;
}

int env_int(const char* name, int dflt) {
#if CSENC_TUNING
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
#else
    (void)name;   // product build: every tuning / debug knob keeps its default
    return dflt;
#endif
}

PFN_encodeTiled get_encode_tiled() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    });
    return fn;
}

}  // namespace host
}  // namespace csenc

extern "C" {

const char* cs_last_error(void) { return csenc::host::g_err.c_str(); }
const char* cs_version(void) { return "csenc 0.2 (sm_100a, tcgen05/TMEM/TMA)"; }

}  // extern "C"
