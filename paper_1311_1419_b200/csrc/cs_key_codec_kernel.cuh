// cs_key_codec_kernel.cuh -- K5: closed-loop key frame.
//
// Eq. (2)-(3): the CS frames subtract the RECONSTRUCTED key frame F-hat = F + e_coding +
// e_decoding, so the key codec's error cancels at the decoder (Eq. 4).  The key codec is SPEC's
// stand-in for H.264 intra: 8x8 block DCT, uniform quantisation by
// quant_scale * the standard luminance matrix, dequantisation, inverse DCT, clamp to [0, 255],
// edge-replication padding to multiples of 8.  The transform is fixed point (R21):
//   forward  t1 = s Ci^T, t2 = Ci t1 (exact integers; s = pixel - 128, Ci = rint(2^12 C)),
//            q = sign(t2) * floor((|t2| + qstep 2^23) / (qstep 2^24))
//   inverse  dq = q qstep, t1 = floor((dq Ci + 2^11) / 2^12), t2 = Ci^T t1,
//            pixel = clamp(floor((t2 + 2^11) / 2^12) + 128, 0, 255)
// so every integer decision is exact.  Entropy coding / rate search are host-side (out of scope).
//
// One kernel does forward + inverse for every key frame: 8 threads per 8x8 block (thread = one
// row, then one column, through a 256-byte SMEM transpose per block), 4 blocks per warp.
#pragma once

#include <cstdint>

namespace csenc {
namespace kc {

constexpr int kThreads = 256;

// rint(4096 * a(u) * cos((2x + 1) u pi / 16)), [u][x] (no entry is within 0.04 of a rounding tie)
#define CSENC_DCT_TABLE                                                                        \
    1448, 1448, 1448, 1448, 1448, 1448, 1448, 1448, 2009, 1703, 1138, 400, -400, -1138, -1703, \
        -2009, 1892, 784, -784, -1892, -1892, -784, 784, 1892, 1703, -400, -2009, -1138, 1138, \
        2009, 400, -1703, 1448, -1448, -1448, 1448, 1448, -1448, -1448, 1448, 1138, -2009, 400, \
        1703, -1703, -400, 2009, -1138, 784, -1892, 1892, -784, -784, 1892, -1892, 784, 400,     \
        -1138, 1703, -2009, 2009, -1703, 1138, -400
__device__ __constant__ int c_dct[64] = {CSENC_DCT_TABLE};
static const int kDctHost[64] = {CSENC_DCT_TABLE};   // the same table, for cs_key_dct_basis()
// ITU-T T.81 Annex K Table K.1 (luminance), [v][u]
static const int kJpegLuma[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                                  14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                                  18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                                  49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};

struct KCParams {
    const uint8_t* frames;    // [n_seq][T][H][W]
    int16_t* coef;            // [n_seq][n_gops_T][nby8][nbx8][8][8] or nullptr
    uint8_t* keys;            // [n_seq][n_gops_T][H][W]
    int W, H, T, G, n_gops_T, nbx8, nby8;
    long long n_blocks;       // n_seq * n_gops_T * nby8 * nbx8
    int qsteps[64];           // [v][u], 1..4096
};

__global__ void __launch_bounds__(kThreads) cs_key_codec_kernel(const __grid_constant__ KCParams p) {
    __shared__ int32_t sm[kThreads / 8][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane >> 3, r = lane & 7;
    int32_t* const tile = sm[warp * 4 + sub];
    const long long per_key = (long long)p.nby8 * p.nbx8;
    const long long stride = (long long)gridDim.x * (kThreads / 8);
    for (long long base = ((long long)blockIdx.x * (kThreads / 32) + warp) * 4; base < p.n_blocks; base += stride) {
        const long long gb = base + sub;
        const bool valid = gb < p.n_blocks;
        long long kk = 0;
        int by8 = 0, bx8 = 0;
        if (valid) {
            kk = gb / per_key;
            const long long rem = gb - kk * per_key;
            by8 = (int)(rem / p.nbx8);
            bx8 = (int)(rem - (long long)by8 * p.nbx8);
        }
        const int s_idx = (int)(kk / p.n_gops_T), g = (int)(kk - (long long)s_idx * p.n_gops_T);
        const size_t frame_bytes = (size_t)p.W * p.H;
        // ---- load row r (edge replication beyond H / W)
        int px[8];
        if (valid) {
            const uint8_t* src = p.frames + ((size_t)s_idx * p.T + (size_t)g * p.G) * frame_bytes;
            const int Y = min(by8 * 8 + r, p.H - 1);
            const uint8_t* row = src + (size_t)Y * p.W;
            const int X0 = bx8 * 8;
            if (X0 + 8 <= p.W) {
                const uint2 w = *reinterpret_cast<const uint2*>(row + X0);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    px[i] = (int)((w.x >> (8 * i)) & 0xFFu) - 128;
                    px[4 + i] = (int)((w.y >> (8 * i)) & 0xFFu) - 128;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) px[i] = (int)row[min(X0 + i, p.W - 1)] - 128;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) px[i] = 0;
        }
        // ---- forward pass 1 (thread = row y = r): t1[y][u] = sum_x s[y][x] Ci[u][x]
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int acc = 0;
#pragma unroll
            for (int x = 0; x < 8; ++x) acc += px[x] * c_dct[u * 8 + x];
            tile[r * 8 + u] = acc;
        }
        __syncwarp();
        // ---- forward pass 2 (thread = column u = r): t2[v][u] = sum_y Ci[v][y] t1[y][u]; quantise
        int col[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) col[y] = tile[y * 8 + r];
        int q[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            long long t2 = 0;
#pragma unroll
            for (int y = 0; y < 8; ++y) t2 += (long long)c_dct[v * 8 + y] * col[y];
            const int qs = p.qsteps[v * 8 + r];
            const long long a = (t2 < 0 ? -t2 : t2) + ((long long)qs << 23);
            const int m = (int)((a >> 24) / qs);
            q[v] = max(-32768, min(32767, t2 < 0 ? -m : m));
        }
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v) tile[v * 8 + r] = q[v];
        __syncwarp();
        // ---- coefficients out (thread = row v = r: 8 int16 = 16 bytes) and inverse pass 1
        int qrow[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) qrow[u] = tile[r * 8 + u];
        if (valid && p.coef != nullptr) {
            uint4 o;
            o.x = (uint32_t)(qrow[0] & 0xFFFF) | ((uint32_t)qrow[1] << 16);
            o.y = (uint32_t)(qrow[2] & 0xFFFF) | ((uint32_t)qrow[3] << 16);
            o.z = (uint32_t)(qrow[4] & 0xFFFF) | ((uint32_t)qrow[5] << 16);
            o.w = (uint32_t)(qrow[6] & 0xFFFF) | ((uint32_t)qrow[7] << 16);
            *reinterpret_cast<uint4*>(p.coef + gb * 64 + r * 8) = o;
        }
        int t1s[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            long long t = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) t += (long long)(qrow[u] * p.qsteps[r * 8 + u]) * c_dct[u * 8 + x];
            t1s[x] = (int)((t + 2048) >> 12);
        }
        __syncwarp();
#pragma unroll
        for (int x = 0; x < 8; ++x) tile[r * 8 + x] = t1s[x];
        __syncwarp();
        // ---- inverse pass 2 (thread = column x = r): t2[y][x] = sum_v Ci[v][y] t1[v][x]
#pragma unroll
        for (int v = 0; v < 8; ++v) col[v] = tile[v * 8 + r];
        int pix[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) {
            long long t = 0;
#pragma unroll
            for (int v = 0; v < 8; ++v) t += (long long)c_dct[v * 8 + y] * col[v];
            const long long v8 = ((t + 2048) >> 12) + 128;
            pix[y] = v8 < 0 ? 0 : (v8 > 255 ? 255 : (int)v8);
        }
        __syncwarp();
#pragma unroll
        for (int y = 0; y < 8; ++y) tile[y * 8 + r] = pix[y];
        __syncwarp();
        // ---- decoded row y = r out (cropped to H; W % 16 == 0 so the row is whole)
        const int Yo = by8 * 8 + r;
        if (valid && Yo < p.H) {
            uint2 w;
            w.x = (uint32_t)tile[r * 8 + 0] | ((uint32_t)tile[r * 8 + 1] << 8) | ((uint32_t)tile[r * 8 + 2] << 16) |
                  ((uint32_t)tile[r * 8 + 3] << 24);
            w.y = (uint32_t)tile[r * 8 + 4] | ((uint32_t)tile[r * 8 + 5] << 8) | ((uint32_t)tile[r * 8 + 6] << 16) |
                  ((uint32_t)tile[r * 8 + 7] << 24);
            *reinterpret_cast<uint2*>(p.keys + (size_t)kk * frame_bytes + (size_t)Yo * p.W + (size_t)bx8 * 8) = w;
        }
        __syncwarp();
    }
}

}  // namespace kc
}  // namespace csenc
