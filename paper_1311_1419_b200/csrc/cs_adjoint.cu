// cs_adjoint.cu -- host side of K3, the block back-projection x0 = Phi^T y:
// Phi^T preparation at encoder create, per-call tensor map of y, launch, cs_adjoint.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "cs_internal.h"
#include "cs_adjoint_kernel.cuh"

namespace csenc {
namespace host {

// Plan and Phi^T for the adjoint: K chunk Kc (8/16/32 floats = the swizzle span of the Y box),
// output chunk Nc = min(N, 256) columns; Phi^T chunk (nc, kc) in the no-swizzle K-major tf32 layout
//   byte(n, k) = (k/4) * LBO + (n/8) * 128 + (n%8) * 16 + (k%4) * 4,  LBO = Nc * 16,
// value Phi[kc*Kc + k][nc*Nc + n] (0 for k >= M).  Skipped (phiT_dev stays NULL) when M % 4 != 0:
// the Y rows must be 16-byte multiples for the tensor map.
int prepare_adjoint(cs_encoder* e, const uint16_t* phi_fp16) {
    const Geometry& g = e->geo;
    if (g.M % 4 != 0) return CS_OK;
    e->adj_Kc = g.M <= 8 ? 8 : (g.M <= 16 ? 16 : 32);
    e->adj_n_kc = cdiv(g.M, e->adj_Kc);
    e->adj_Nc = std::min(g.N, 256);
    e->adj_n_nc = g.N / e->adj_Nc;
    e->adj_chunk_bytes = (uint32_t)e->adj_Nc * (uint32_t)e->adj_Kc * 4u;
    const uint32_t a_bytes = 128u * (uint32_t)e->adj_Kc * 4u;
    e->adj_stage_bytes = align_up(2 * a_bytes + e->adj_chunk_bytes, 1024);
    const long avail = (long)e->smem_limit - 1024 - (long)csenc::adj::kOffStage;
    e->adj_stages = (int)std::min<long>(csenc::adj::kMaxStages, avail / (long)e->adj_stage_bytes);
    if (e->adj_stages < 2) return fail(CS_ERR_UNSUPPORTED, "adjoint: stages do not fit shared memory");
    e->adj_smem = 1024 + csenc::adj::kOffStage + (uint32_t)e->adj_stages * e->adj_stage_bytes;
    const size_t bytes = (size_t)e->adj_n_nc * e->adj_n_kc * e->adj_chunk_bytes;
    std::vector<float> h(bytes / 4, 0.0f);
    const uint32_t lbo = (uint32_t)e->adj_Nc * 16u;
    for (int nc = 0; nc < e->adj_n_nc; ++nc)
        for (int kc = 0; kc < e->adj_n_kc; ++kc) {
            const size_t base = (size_t)(nc * e->adj_n_kc + kc) * e->adj_chunk_bytes;
            for (int n = 0; n < e->adj_Nc; ++n)
                for (int k = 0; k < e->adj_Kc; ++k) {
                    const int m = kc * e->adj_Kc + k, j = nc * e->adj_Nc + n;
                    const size_t byte = base + (size_t)(k / 4) * lbo + (size_t)(n / 8) * 128 + (size_t)(n % 8) * 16 +
                                        (size_t)(k % 4) * 4;
                    h[byte / 4] = m < g.M ? half_bits_to_float(phi_fp16[(size_t)m * g.N + j]) : 0.0f;
                }
        }
    cudaError_t err = cudaMalloc(&e->phiT_dev, bytes);
    if (err != cudaSuccess) return fail(CS_ERR_OOM, std::string("cudaMalloc(Phi^T): ") + cudaGetErrorString(err));
    err = cudaMemcpy(e->phiT_dev, h.data(), bytes, cudaMemcpyHostToDevice);
    if (err != cudaSuccess) return cuda_fail(err, "cudaMemcpy(Phi^T)");
    return CS_OK;
}

int launch_adjoint(cs_encoder* e, const float* meas, long long n_frames, float* x, cudaStream_t stream) {
    const Geometry& g = e->geo;
    csenc::adj::AParams ap;
    std::memset(&ap, 0, sizeof(ap));
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const long long rows = n_frames * g.nblk;
    cuuint64_t dims[2] = {(cuuint64_t)g.M, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)g.M * 4u};
    cuuint32_t box[2] = {(cuuint32_t)e->adj_Kc, 128u};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = e->adj_Kc == 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : (e->adj_Kc == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    CUresult r = enc(&ap.ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(meas), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CS_ERR_CUDA, "cuTensorMapEncodeTiled(y) failed (code " + std::to_string((int)r) + ")");
    ap.phiT = (const uint8_t*)e->phiT_dev;
    ap.x = x;
    ap.W = g.W;
    ap.H = g.H;
    ap.M = g.M;
    ap.nbx = g.nbx;
    ap.nby = g.nby;
    ap.nblk = g.nblk;
    ap.parts = cdiv(g.nbx, 128);
    ap.L = cdiv(g.nbx, ap.parts);
    ap.Kc = e->adj_Kc;
    ap.n_kc = e->adj_n_kc;
    ap.Nc = e->adj_Nc;
    ap.n_nc = e->adj_n_nc;
    ap.a_bytes = 128u * (uint32_t)e->adj_Kc * 4u;
    ap.chunk_bytes = e->adj_chunk_bytes;
    ap.stage_bytes = e->adj_stage_bytes;
    ap.n_stages = e->adj_stages;
    ap.n_units = (int)(n_frames * g.nby * ap.parts);
    // flat tiles (128 consecutive blocks across block rows) when every warp's 32 blocks stay in one
    // block row: fewer, fuller units for narrow-block frames (C5: 113 instead of 180 per frame)
    ap.flat = (g.nbx % 32 == 0 && env_int("CSENC_ADJ_FLAT", 1)) ? 1 : 0;
    if (ap.flat) {
        ap.tiles_pf = cdiv(g.nblk, 128);
        ap.L = 128;
        ap.n_units = (int)(n_frames * ap.tiles_pf);
    }
    // kind::tf32: D fp32 (bit 4), A/B tf32 (2 at bits 7 and 10), K-major, N>>3 at 17, M>>4 at 24
    ap.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(ap.Nc >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    ap.b_lbo = (uint32_t)ap.Nc * 16u;
    ap.a_sbo = 8u * (uint32_t)ap.Kc * 4u;
    ap.x_floats = n_frames * (long long)g.W * g.H;
    ap.smem_bytes = e->adj_smem - 1024;
    const int grid = std::max(1, std::min(e->sms, ap.n_units));
    ap.pdl_early = (e->stable_inputs & CS_STABLE_MEASUREMENTS) ? 1 : 0;
    // programmatic dependent launch, as the measurement kernel (cs_encoder.cu launch())
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)csenc::adj::kThreads);
    cfg.dynamicSmemBytes = (size_t)e->adj_smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CSENC_PDL ? 1 : 0;
    cudaError_t lerr = cudaSuccess;
    switch (g.B) {
        case 8: lerr = cudaLaunchKernelEx(&cfg, csenc::adj::cs_adjoint_kernel<8>, ap); break;
        case 16: lerr = cudaLaunchKernelEx(&cfg, csenc::adj::cs_adjoint_kernel<16>, ap); break;
        case 32: lerr = cudaLaunchKernelEx(&cfg, csenc::adj::cs_adjoint_kernel<32>, ap); break;
        default: return fail(CS_ERR_UNSUPPORTED, "block size");
    }
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) err = lerr;
    return err == cudaSuccess ? CS_OK : cuda_fail(err, "adjoint launch");
}


cudaError_t adjoint_set_smem_attr(int bytes) {
    cudaError_t e = cudaSuccess, r;
    r = cudaFuncSetAttribute(adj::cs_adjoint_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (r != cudaSuccess) e = r;
    r = cudaFuncSetAttribute(adj::cs_adjoint_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (r != cudaSuccess) e = r;
    r = cudaFuncSetAttribute(adj::cs_adjoint_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (r != cudaSuccess) e = r;
    return e;
}

}  // namespace host
}  // namespace csenc

using namespace csenc::host;

extern "C" {

int cs_adjoint(cs_encoder* e, const float* meas, int64_t n_frames, float* x, cs_stream_t stream) {
    csenc::host::NvtxScope nvtx_scope("cs_adjoint");
    if (!e) return fail(CS_ERR_ARG, "encoder is NULL");
    if (n_frames < 0) return fail(CS_ERR_ARG, "n_frames must be >= 0");
    if (n_frames == 0) return CS_OK;
    if (!meas || !x) return fail(CS_ERR_ARG, "NULL buffer");
    if (!aligned16(meas) || !aligned16(x)) return fail(CS_ERR_ARG, "buffers must be 16-byte aligned");
    if (!e->phiT_dev) return fail(CS_ERR_UNSUPPORTED, "adjoint needs M % 4 == 0 (16-byte measurement rows)");
    if (e->n_phis > 0)
        return fail(CS_ERR_UNSUPPORTED, "adjoint: per-GOP matrices are set (cs_encoder_set_gop_phis); Phi^T is that of the "
                                        "single Phi given at create -- restore it with cs_encoder_set_gop_phis(e, 0, NULL)");
    if (int rc = check_device(e->device)) return rc;
    const Geometry& g = e->geo;
    if (n_frames * (long long)g.nblk >= 0x7FFFFFFFLL || n_frames * (long long)g.nby * cdiv(g.nbx, 128) >= 0x7FFFFFFFLL)
        return fail(CS_ERR_UNSUPPORTED, "too many frames for one call");
    return launch_adjoint(e, meas, n_frames, x, (cudaStream_t)stream);
}

}  // extern "C"
