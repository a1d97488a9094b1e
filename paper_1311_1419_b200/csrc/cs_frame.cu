// cs_frame.cu -- host side of K4, the paper-faithful frame-level measurement y = A vec(F_cs - F_key)
// with one dense A: the frame encoder object, window planning (load
// balance), tensor maps, launch, split-K reduction.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "cs_internal.h"
#include "cs_frame_kernel.cuh"

using namespace csenc::host;

struct cs_frame_encoder {
    int W = 0, H = 0, G = 0, m = 0, n = 0;
    int device = 0, sms = 0, smem_limit = 0;
    void* A_dev = nullptr;   // fp16 [m][n], columns permuted within groups of 4 (converter pair order)
    unsigned long long* trace = nullptr;   // debug timeline (cs_frame_encoder_set_trace)
    int trace_cap = 0;
};

extern "C" {

int cs_frame_encoder_create(int W, int H, int gop, int m, const uint16_t* A_fp16, cs_frame_encoder** out) {
    if (!out) return fail(CS_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!A_fp16) return fail(CS_ERR_ARG, "A is NULL");
    if (W < 1 || H < 1 || gop < 1 || m < 1) return fail(CS_ERR_ARG, "W, H, gop and m must be >= 1");
    if (W % 16 != 0) return fail(CS_ERR_UNSUPPORTED, "W must be a multiple of 16 (TMA row pitch)");
    const long long n = (long long)W * H;
    if (n > (1LL << 30) || (long long)m * n > (1LL << 34)) return fail(CS_ERR_UNSUPPORTED, "A too large");
    for (long long i = 0; i < (long long)m * n; ++i) {
        const float v = half_bits_to_float(A_fp16[i]);
        if (!std::isfinite(v) || std::fabs(v) > 2048.0f) return fail(CS_ERR_PHI, "A has a non-finite entry or |entry| > 2048");
    }
    int dev = 0, major = 0, minor = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return cuda_fail(err, "cudaGetDevice");
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) return fail(CS_ERR_UNSUPPORTED, "device is not sm_100 (B200)");
    cs_frame_encoder* f = new (std::nothrow) cs_frame_encoder();
    if (!f) return fail(CS_ERR_OOM, "host allocation failed");
    f->W = W;
    f->H = H;
    f->G = gop;
    f->m = m;
    f->n = (int)n;
    f->device = dev;
    cudaDeviceGetAttribute(&f->sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&f->smem_limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    err = cudaFuncSetAttribute(csenc::frm::cs_frame_measure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               f->smem_limit);
    if (err != cudaSuccess) {
        delete f;
        return cuda_fail(err, "cudaFuncSetAttribute");
    }
    // column k of the device copy holds pixel 4(k/4) + {0,2,1,3}[k%4] (the residual4 pair order)
    static const int kPerm[4] = {0, 2, 1, 3};
    std::vector<uint16_t> perm((size_t)m * n);
    for (long long r = 0; r < m; ++r)
        for (long long k = 0; k < n; ++k) {
            const long long j = (k & ~3LL) | kPerm[k & 3];
            perm[(size_t)(r * n + k)] = j < n ? A_fp16[r * n + j] : 0;
        }
    err = cudaMalloc(&f->A_dev, perm.size() * 2);
    if (err != cudaSuccess) {
        delete f;
        return fail(CS_ERR_OOM, std::string("cudaMalloc(A): ") + cudaGetErrorString(err));
    }
    err = cudaMemcpy(f->A_dev, perm.data(), perm.size() * 2, cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
        cudaFree(f->A_dev);
        delete f;
        return cuda_fail(err, "cudaMemcpy(A)");
    }
    *out = f;
    return CS_OK;
}

int cs_frame_encoder_set_trace(cs_frame_encoder* f, unsigned long long* trace_dev, int cap) {
    if (!f || cap < 0 || (cap > 0 && !trace_dev)) return fail(CS_ERR_ARG, "bad trace arguments");
    f->trace = cap > 0 ? trace_dev : nullptr;
    f->trace_cap = cap;
    return CS_OK;
}

int cs_frame_encoder_destroy(cs_frame_encoder* f) {
    if (!f) return CS_OK;
    if (f->A_dev) cudaFree(f->A_dev);
    delete f;
    return CS_OK;
}

int64_t cs_frame_measurement_count(const cs_frame_encoder* f, int n_seq, int T) {
    if (!f || n_seq < 0 || T < 0) return -1;
    return (int64_t)n_seq * cs_frames_per_stream(T, f->G) * f->m;
}

}  // extern "C"


extern "C" {

int cs_frame_encode_batch(cs_frame_encoder* f, const uint8_t* frames, int n_seq, int T, float* y, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_frame_encode_batch");
    if (!f) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_seq < 0 || T < 0) return fail(CS_ERR_ARG, "n_seq and T must be >= 0");
    const long long cs_s = cs_frames_per_stream(T, f->G);
    if (n_seq == 0 || cs_s == 0) return CS_OK;
    if (!frames || !y) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(frames) || !aligned16(y)) return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if ((long long)n_seq * T > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many frames");
    if (int rc = check_device(f->device)) return rc;
    const cudaStream_t st = (cudaStream_t)stream;
    csenc::frm::FParams fp;
    std::memset(&fp, 0, sizeof(fp));
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int G = f->G;
    const int n_gops = cdiv(T, G);
    const int gw_max = std::max(1, 256 / G);          // box rows <= 256, CS rows <= 256
    fp.n_mp = cdiv(f->m, 256);
    if (T % G == 0) {
        // whole GOPs everywhere: windows over the concatenation, sized so the units fill the SMs in
        // whole waves (k units per SM, the smallest k whose windows fit a box)
        fp.global_win = 1;
        fp.total_gops = n_seq * n_gops;
        fp.gw = std::min(gw_max, fp.total_gops);
        for (int k = 1; k <= 16; ++k) {
            const long long want = ((long long)k * f->sms + fp.n_mp - 1) / fp.n_mp;
            const long long gw = (fp.total_gops + want - 1) / want;
            if (gw <= gw_max) {
                fp.gw = (int)std::max(1LL, gw);
                break;
            }
        }
        if (const int gwf = env_int("CSENC_FRAME_GW", 0)) fp.gw = std::max(1, std::min(gw_max, gwf));   // experiment knob
        fp.n_win_s = 0;
        fp.n_win = cdiv(fp.total_gops, fp.gw);
    } else {
        // windows inside each stream, balanced
        fp.global_win = 0;
        fp.total_gops = n_seq * n_gops;
        fp.n_win_s = cdiv(n_gops, gw_max);
        fp.gw = cdiv(n_gops, fp.n_win_s);
        fp.n_win_s = cdiv(n_gops, fp.gw);
        fp.n_win = n_seq * fp.n_win_s;
    }
    fp.nf_box = fp.gw * G;
    {
        cuuint64_t dims[2] = {(cuuint64_t)f->n, (cuuint64_t)n_seq * T};
        cuuint64_t strides[1] = {(cuuint64_t)f->n};
        cuuint32_t box[2] = {(cuuint32_t)csenc::frm::kKc, (cuuint32_t)fp.nf_box};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = enc(&fp.fmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(frames), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled(frames) failed (code " + std::to_string((int)r) + ")");
    }
    {
        cuuint64_t dims[2] = {(cuuint64_t)f->n, (cuuint64_t)f->m};
        cuuint64_t strides[1] = {(cuuint64_t)f->n * 2u};
        cuuint32_t box[2] = {(cuuint32_t)csenc::frm::kKc, 256u};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = enc(&fp.amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, f->A_dev, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed (code " + std::to_string((int)r) + ")");
    }
    fp.n = f->n;
    fp.m = f->m;
    fp.G = G;
    fp.T = T;
    fp.cs_s = (int)cs_s;

    fp.n_chunks = cdiv(f->n, csenc::frm::kKc);
    const long long n_cl = f->sms;                                      // CTAs resident at once
    const long long tiles = (long long)fp.n_win * fp.n_mp;              // work units per K split
    long long ks = (n_cl + tiles - 1) / tiles;                        // K splits to fill the SMs
    ks = std::max(1LL, std::min(ks, (long long)std::max(1, fp.n_chunks / 8)));
    if (const int ksf = env_int("CSENC_FRAME_KS", 0)) ks = std::max(1, std::min(ksf, fp.n_chunks));   // experiment knob
    // no empty K split (every unit must issue at least one chunk): ks = ceil(chunks / per-split)
    const long long per_split = (fp.n_chunks + ks - 1) / ks;
    ks = (fp.n_chunks + per_split - 1) / per_split;
    fp.n_ks = (int)ks;
    if (tiles * ks > 0x7FFFFFFFLL) return fail(CS_ERR_UNSUPPORTED, "too many work units");
    fp.n_units = (int)(tiles * ks);
    fp.fbox_bytes = (uint32_t)fp.nf_box * (uint32_t)csenc::frm::kKc;
    fp.stage_bytes = align_up(fp.fbox_bytes, 1024);                    // frames ring slot
    const uint32_t a_slot = 256u * csenc::frm::kKc * 2u;                // A ring slot (32 KB)
    fp.b_bytes = align_up((uint32_t)(fp.gw * (G - 1) + 15) / 16 * 16 * 128u, 1024);
    fp.n_b = std::max(2, std::min(4, env_int("CSENC_FRAME_BBUFS", 2)));
    fp.off_stage = csenc::frm::kOffB + (uint32_t)fp.n_b * fp.b_bytes;
    // A ring: 3 slots (A is L2-resident: short latency); frames ring: the rest, up to kMaxStages
    // (frames come from HBM and are consumed first)
    const long avail = (long)f->smem_limit - 1024 - (long)fp.off_stage;
    fp.n_a = std::max(2, std::min(csenc::frm::kMaxStages, env_int("CSENC_FRAME_ASLOTS", 3)));
    fp.n_stages = (int)std::min<long>(csenc::frm::kMaxStages, (avail - (long)fp.n_a * a_slot) / (long)fp.stage_bytes);
    while (fp.n_stages < 2 && fp.n_a > 2) {
        --fp.n_a;
        fp.n_stages = (int)std::min<long>(csenc::frm::kMaxStages, (avail - (long)fp.n_a * a_slot) / (long)fp.stage_bytes);
    }
    if (fp.n_stages < 2) return fail(CS_ERR_UNSUPPORTED, "frame measurement: rings do not fit shared memory");
    if (const int fs = env_int("CSENC_FRAME_FSLOTS", 0)) fp.n_stages = std::max(2, std::min(fp.n_stages, fs));   // knob
    fp.off_a = fp.off_stage + (uint32_t)fp.n_stages * fp.stage_bytes;   // 1024-aligned (slots are)
    const uint32_t smem = 1024 + fp.off_a + (uint32_t)fp.n_a * a_slot;
    fp.prefetch = env_int("CSENC_FRAME_PREFETCH", 0);
    fp.trace = f->trace;
    fp.trace_cap = f->trace_cap;
    fp.out_floats = (long long)n_seq * cs_s * f->m;
    fp.smem_bytes = smem - 1024;
    const long long ny = (long long)n_seq * cs_s * f->m;
    float* part = nullptr;
    cudaError_t err;
    if (fp.n_ks > 1) {
        fp.part_stride = (ny + 3) / 4 * 4;
        err = cudaMallocAsync((void**)&part, (size_t)fp.part_stride * fp.n_ks * sizeof(float), st);
        if (err != cudaSuccess) return fail(CS_ERR_OOM, std::string("partials: ") + cudaGetErrorString(err));
        fp.out = part;
    } else {
        fp.part_stride = 0;
        fp.out = y;
    }
    const int grid = (int)std::max(1LL, std::min(n_cl, (long long)fp.n_units));
    csenc::frm::cs_frame_measure_kernel<<<grid, csenc::frm::kThreads, smem, st>>>(fp);
    err = cudaGetLastError();
    if (err == cudaSuccess && fp.n_ks > 1) {
        csenc::frm::cs_frame_reduce_kernel<<<f->sms * 4, 256, 0, st>>>(part, y, ny, fp.part_stride, fp.n_ks);
        err = cudaGetLastError();
    }
    if (part) cudaFreeAsync(part, st);
    return err == cudaSuccess ? CS_OK : cuda_fail(err, "frame measurement launch");
}

}  // extern "C"
