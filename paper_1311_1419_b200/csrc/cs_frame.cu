// cs_frame.cu -- host side of K4, the paper-faithful frame-level measurement y = A vec(F_cs - F_key)
// with one dense A: the frame encoder object, window planning (load
// balance), tensor maps, launch, split-K reduction.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
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
    // stream-ordered scratch for the stream-K partial tiles: the object's own pool, which keeps its memory
    // between calls (release threshold = max), created on first use
    cudaMemPool_t pool = nullptr;
    std::mutex pool_mu;
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
    if (f->pool) cudaMemPoolDestroy(f->pool);
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
    // window: CS rows <= 256 (MMA N, TMEM columns), frame rows <= 512 (two TMA boxes per chunk)
    const int gw_max = std::max(1, std::min(G > 1 ? 256 / (G - 1) : 256, 512 / G));
    fp.n_mp = cdiv(f->m, 256);
    if (T % G == 0) {
        // whole GOPs everywhere: windows over the concatenation, as large as the MMA N / TMEM allow (the A
        // tile is reused across the window's CS frames: A traffic per flop falls with the window; the
        // stream-K split below balances the SMs whatever the unit count), equal-sized
        fp.global_win = 1;
        fp.total_gops = n_seq * n_gops;
        fp.gw = std::min(gw_max, fp.total_gops);
        fp.gw = cdiv(fp.total_gops, cdiv(fp.total_gops, fp.gw));
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
    fp.n_fbox = cdiv(fp.nf_box, 256);
    fp.fbox_rows = (int)align_up((uint32_t)cdiv(fp.nf_box, fp.n_fbox), 8);   // 512-B swizzle period per box
    {
        cuuint64_t dims[2] = {(cuuint64_t)f->n, (cuuint64_t)n_seq * T};
        cuuint64_t strides[1] = {(cuuint64_t)f->n};
        cuuint32_t box[2] = {(cuuint32_t)csenc::frm::kKc, (cuuint32_t)fp.fbox_rows};
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
    const long long tiles = (long long)fp.n_win * fp.n_mp;              // work units
    if (tiles > 0x7FFFFFFFLL / 2) return fail(CS_ERR_UNSUPPORTED, "too many work units");
    fp.n_units = (int)tiles;
    fp.total_chunks = (long long)fp.n_win * fp.n_chunks;   // per m-pair
    // stream-K grid: n_mp CTAs per range (one per m-pair, same frame boxes at the same time), as many
    // ranges as SMs allow, unless that leaves a CTA fewer than 8 chunks (pipeline fill per piece) or cuts
    // a unit into more than 8 pieces (ranges of >= n_chunks / 7 chunks)
    const long long gj = std::max(1LL, std::min({(long long)f->sms / fp.n_mp, fp.total_chunks / 8,
                                                 7 * fp.total_chunks / std::max(1, fp.n_chunks)}));
    const long long n_cl = gj * fp.n_mp;
    fp.fbox_bytes = (uint32_t)(fp.n_fbox * fp.fbox_rows) * (uint32_t)csenc::frm::kKc;
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
    fp.out = y;
    const int grid = (int)n_cl;
    // units cut by a range boundary (each boundary b = 1 .. grid-1 that is not a unit start); their
    // pieces go to partial tiles (2 per CTA) summed by the fixup kernel
    csenc::frm::FixupList fl;
    fl.n = 0;
    fl.grid = grid;
    for (long long j = 1, last = -1; j < gj; ++j) {
        const long long c = j * fp.total_chunks / gj;
        if (c % fp.n_chunks == 0) continue;
        const int win = (int)(c / fp.n_chunks);
        if (win == last) continue;
        last = win;
        for (int mp = 0; mp < fp.n_mp; ++mp) {
            if (fl.n == (int)(sizeof(fl.units) / sizeof(fl.units[0]))) return fail(CS_ERR_UNSUPPORTED, "too many split units");
            fl.units[fl.n++] = win * fp.n_mp + mp;
        }
    }
    float* part = nullptr;
    cudaError_t err;
    if (fl.n > 0) {
        {
            std::lock_guard<std::mutex> lk(f->pool_mu);
            if (!f->pool) {
                cudaMemPoolProps props;
                std::memset(&props, 0, sizeof(props));
                props.allocType = cudaMemAllocationTypePinned;
                props.location.type = cudaMemLocationTypeDevice;
                props.location.id = f->device;
                if (cudaMemPoolCreate(&f->pool, &props) != cudaSuccess) f->pool = nullptr;
                uint64_t keep = ~0ull;
                if (f->pool) cudaMemPoolSetAttribute(f->pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        err = f->pool ? cudaMallocFromPoolAsync((void**)&part, (size_t)2 * grid * 65536 * sizeof(float), f->pool, st)
                      : cudaMallocAsync((void**)&part, (size_t)2 * grid * 65536 * sizeof(float), st);
        if (err != cudaSuccess) return fail(CS_ERR_OOM, std::string("partial tiles: ") + cudaGetErrorString(err));
    }
    fp.part = part;
    csenc::frm::cs_frame_measure_kernel<<<grid, csenc::frm::kThreads, smem, st>>>(fp);
    err = cudaGetLastError();
    if (err == cudaSuccess && fl.n > 0) {
        csenc::frm::cs_frame_fixup_kernel<<<dim3((unsigned)fl.n, 32), 64, 0, st>>>(fp, fl);
        err = cudaGetLastError();
    }
    if (part) cudaFreeAsync(part, st);
    return err == cudaSuccess ? CS_OK : cuda_fail(err, "frame measurement launch");
}

}  // extern "C"
