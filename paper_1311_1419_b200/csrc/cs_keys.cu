// cs_keys.cu -- host side of K5, the closed-loop key codec: quantiser
// steps, the fixed-point DCT basis, the codec launch.  (Encoding against the decoded keys is
// cs_encode_batch_keys in cs_encoder.cu.)
#include <algorithm>
#include <cmath>
#include <cstring>

#include "cs_internal.h"
#include "cs_key_codec_kernel.cuh"

using namespace csenc::host;

extern "C" {

void cs_key_dct_basis(int32_t out[64]) {
    for (int i = 0; i < 64; ++i) out[i] = csenc::kc::kDctHost[i];
}

int cs_key_qsteps(double quant_scale, int32_t out[64]) {
    if (!out) return fail(CS_ERR_ARG, "out is NULL");
    if (!(quant_scale > 0.0) || !std::isfinite(quant_scale)) return fail(CS_ERR_ARG, "quant_scale must be > 0");
    for (int i = 0; i < 64; ++i) {
        const double v = std::nearbyint(quant_scale * csenc::kc::kJpegLuma[i]);  // round half to even
        out[i] = (int32_t)std::min(4096.0, std::max(1.0, v));
    }
    return CS_OK;
}

int64_t cs_key_coef_count(const cs_encoder* e, int n_seq, int T) {
    if (!e || n_seq < 0 || T < 0) return -1;
    const Geometry& g = e->geo;
    return (int64_t)n_seq * cdiv(T, g.G) * cdiv(g.H, 8) * cdiv(g.W, 8) * 64;
}

int cs_key_codec(cs_encoder* e, const uint8_t* frames, int n_seq, int T, const int32_t* qsteps, int16_t* coef,
                 uint8_t* keys, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_key_codec");
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    if (n_seq == 0 || T == 0) return CS_OK;
    if (!frames || !keys || !qsteps) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(keys) || (coef && !aligned16(coef)))
        return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if (int rc = check_device(e->device)) return rc;
    const Geometry& g = e->geo;
    csenc::kc::KCParams kp;
    std::memset(&kp, 0, sizeof(kp));
    for (int i = 0; i < 64; ++i) {
        if (qsteps[i] < 1 || qsteps[i] > 4096) return fail(CS_ERR_ARG, "quantiser steps must be in [1, 4096]");
        kp.qsteps[i] = qsteps[i];
    }
    kp.frames = frames;
    kp.coef = coef;
    kp.keys = keys;
    kp.W = g.W;
    kp.H = g.H;
    kp.T = T;
    kp.G = g.G;
    kp.n_gops_T = cdiv(T, g.G);
    kp.nbx8 = cdiv(g.W, 8);
    kp.nby8 = cdiv(g.H, 8);
    kp.n_blocks = (long long)n_seq * kp.n_gops_T * kp.nby8 * kp.nbx8;
    const long long n_keys = (long long)n_seq * kp.n_gops_T;
    if (n_keys > 65535 || (long long)kp.nby8 * kp.nbx8 > 0x7FFFFFFFLL)
        return fail(CS_ERR_UNSUPPORTED, "key codec: more than 65535 key frames in one call");
    // ~12 CTAs per SM in total (3 resident: 4 waves of slack against imbalance), spread over the keys
    const int per_key_ctas = (int)((kp.nby8 * (long long)kp.nbx8 + csenc::kc::kThreads / 8 - 1) / (csenc::kc::kThreads / 8));
    const int gx = (int)std::max(1LL, std::min((long long)per_key_ctas, ((long long)e->sms * 12 + n_keys - 1) / n_keys));
    csenc::kc::cs_key_codec_kernel<<<dim3(gx, (unsigned)n_keys), csenc::kc::kThreads, 0, (cudaStream_t)stream>>>(kp);
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? CS_OK : cuda_fail(err, "key codec launch");
}

}  // extern "C"
