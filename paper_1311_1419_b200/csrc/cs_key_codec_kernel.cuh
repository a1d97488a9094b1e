// cs_key_codec_kernel.cuh -- K5: closed-loop key frame.
//
// Eq. (2)-(3): the CS frames subtract the RECONSTRUCTED key frame F-hat = F + e_coding +
// e_decoding, so the key codec's error cancels at the decoder (Eq. 4).  The key codec is SPEC's
// stand-in for H.264 intra: 8x8 block DCT, uniform quantisation by
// quant_scale * the standard luminance matrix, dequantisation, inverse DCT, clamp to [0, 255],
// edge-replication padding to multiples of 8.  The transform is fixed point (R21):
//   forward  t1 = floor((s Ci^T + 2^4) / 2^5), t2 = Ci t1 (s = pixel - 128, Ci = rint(2^12 C)),
//            q = sign(t2) * floor((|t2| + qstep 2^18) / (qstep 2^19))
//   inverse  dq = q qstep, t1 = floor((dq Ci + 2^11) / 2^12), t2 = Ci^T t1,
//            pixel = clamp(floor((t2 + 2^11) / 2^12) + 128, 0, 255)
// so every integer decision is exact, and every intermediate fits int32: |s Ci^T| < 2^21,
// |t2| < 2^30, |t2| + qstep 2^18 < 2^31, |dq| <= 2^12 (q comes from the forward pass),
// |dq Ci| sums < 2^26, inverse |t2| < 2^28.  Entropy coding / rate search are host-side (out of scope).
//
// One kernel does forward + inverse for every key frame: 8 threads per 8x8 block (thread = one
// row, then one column, through a 256-byte SMEM transpose per block), 4 blocks per warp.
#pragma once

#include <cstdint>

#include "ptx_sm100.cuh"   // CS_CHECK

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
// compile-time basis: with the loops unrolled every coefficient is an instruction immediate
__device__ __forceinline__ constexpr int dct_c(int i) {
    constexpr int t[64] = {CSENC_DCT_TABLE};
    return t[i];
}
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
    long long n_blocks;       // n_seq * n_gops_T * nby8 * nbx8 (grid.y = n_seq * n_gops_T keys)
    int qsteps[64];           // [v][u], 1..4096
};

// The basis has the DCT's even/odd symmetry, Ci[u][7-x] = (-1)^u Ci[u][x] (rint keeps it), so
// each 8-point product is formed from 4-point sums and differences: 32 multiply-adds instead of 64,
// exactly the same integers.
// out[u] = sum_x in[x] Ci[u][x]
__device__ __forceinline__ void dct8_fwd(const int (&in)[8], int (&out)[8]) {
    int e[4], o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        e[k] = in[k] + in[7 - k];
        o[k] = in[k] - in[7 - k];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        int acc = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += ((u & 1) ? o[k] : e[k]) * dct_c(u * 8 + k);
        out[u] = acc;
    }
}
// out[x] = sum_u in[u] Ci[u][x]
__device__ __forceinline__ void dct8_inv(const int (&in)[8], int (&out)[8]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int E = 0, O = 0;
#pragma unroll
        for (int u = 0; u < 8; u += 2) E += in[u] * dct_c(u * 8 + k);
#pragma unroll
        for (int u = 1; u < 8; u += 2) O += in[u] * dct_c(u * 8 + k);
        out[k] = E + O;
        out[7 - k] = E - O;
    }
}

__global__ void __launch_bounds__(kThreads, 3) cs_key_codec_kernel(const __grid_constant__ KCParams p) {
    // 8x8 transpose tiles, row pitch 9 words, 72 words per block: bank = 8*sub + 9*row + col (mod 32)
    // is distinct over the warp for both row-wise and column-wise access (conflict-free)
    __shared__ int32_t sm[kThreads / 8][72];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane >> 3, r = lane & 7;
    int32_t* const tile = sm[warp * 4 + sub];
    // quantiser steps and, per step q >= 2, the exact reciprocal m = ceil(2^32 / q):
    // floor(n / q) = umulhi(n, m) for n < 2^13 (error term n * (m * q - 2^32) < 2^13 * 2^12 < 2^32)
    __shared__ int s_q[64];
    __shared__ uint32_t s_m[64];
    if (threadIdx.x < 64) {
        const int q = p.qsteps[threadIdx.x];
        s_q[threadIdx.x] = q;
        s_m[threadIdx.x] = q == 1 ? 0u : 0xFFFFFFFFu / (uint32_t)q + 1u;
    }
    __syncthreads();
    // grid: blockIdx.y = key frame (stream s, GOP g); x-dimension strides over its 8x8 blocks
    const int per_key = p.nby8 * p.nbx8;
    const int kk = blockIdx.y;
    const int s_idx = kk / p.n_gops_T, g = kk - s_idx * p.n_gops_T;
    const int stride = gridDim.x * (kThreads / 8);
    for (int base = (blockIdx.x * (kThreads / 32) + warp) * 4; base < per_key; base += stride) {
        const int gbk = base + sub;                       // block within the key frame
        const bool valid = gbk < per_key;
        const int by8 = valid ? gbk / p.nbx8 : 0;
        const int bx8 = valid ? gbk - by8 * p.nbx8 : 0;
        const long long gb = (long long)kk * per_key + gbk;
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
        // ---- forward pass 1 (thread = row y = r): t1[y][u] = floor((sum_x s[y][x] Ci[u][x] + 16) / 32)
        {
            int t1[8];
            dct8_fwd(px, t1);
#pragma unroll
            for (int u = 0; u < 8; ++u) tile[r * 9 + u] = (t1[u] + 16) >> 5;
        }
        __syncwarp();
        // ---- forward pass 2 (thread = column u = r): t2[v][u] = sum_y Ci[v][y] t1[y][u]; quantise
        int col[8];
#pragma unroll
        for (int y = 0; y < 8; ++y) col[y] = tile[y * 9 + r];
        int t2v[8];
        dct8_fwd(col, t2v);
        int q[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int t2 = t2v[v];
            const int qs = s_q[v * 8 + r];
            const uint32_t mq = s_m[v * 8 + r];
            const uint32_t n = (uint32_t)(((t2 < 0 ? -t2 : t2) + (qs << 18)) >> 19);
            const int m = (int)(mq == 0u ? n : __umulhi(n, mq));
            q[v] = t2 < 0 ? -m : m;
        }
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v) tile[v * 9 + r] = q[v];
        __syncwarp();
        // ---- coefficients out (thread = row v = r: 8 int16 = 16 bytes) and inverse pass 1
        int qrow[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) qrow[u] = tile[r * 9 + u];
        CS_CHECK(!valid || gb * 64 + r * 8 + 8 <= p.n_blocks * 64);
        if (valid && p.coef != nullptr) {
            uint4 o;
            o.x = (uint32_t)(qrow[0] & 0xFFFF) | ((uint32_t)qrow[1] << 16);
            o.y = (uint32_t)(qrow[2] & 0xFFFF) | ((uint32_t)qrow[3] << 16);
            o.z = (uint32_t)(qrow[4] & 0xFFFF) | ((uint32_t)qrow[5] << 16);
            o.w = (uint32_t)(qrow[6] & 0xFFFF) | ((uint32_t)qrow[7] << 16);
            *reinterpret_cast<uint4*>(p.coef + gb * 64 + r * 8) = o;
        }
        int dq[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) dq[u] = qrow[u] * s_q[r * 8 + u];
        int t1s[8];
        dct8_inv(dq, t1s);
#pragma unroll
        for (int x = 0; x < 8; ++x) t1s[x] = (t1s[x] + 2048) >> 12;
        __syncwarp();
#pragma unroll
        for (int x = 0; x < 8; ++x) tile[r * 9 + x] = t1s[x];
        __syncwarp();
        // ---- inverse pass 2 (thread = column x = r): t2[y][x] = sum_v Ci[v][y] t1[v][x]
#pragma unroll
        for (int v = 0; v < 8; ++v) col[v] = tile[v * 9 + r];
        int pix[8];
        dct8_inv(col, pix);
#pragma unroll
        for (int y = 0; y < 8; ++y) pix[y] = max(0, min(255, ((pix[y] + 2048) >> 12) + 128));
        __syncwarp();
#pragma unroll
        for (int y = 0; y < 8; ++y) tile[y * 9 + r] = pix[y];
        __syncwarp();
        // ---- decoded row y = r out (cropped to H; W % 16 == 0 so the row is whole)
        const int Yo = by8 * 8 + r;
        CS_CHECK(!valid || Yo >= p.H ||
                 (long long)kk * frame_bytes + (long long)Yo * p.W + bx8 * 8 + 8 <= (p.n_blocks / per_key) * (long long)frame_bytes);
        if (valid && Yo < p.H) {
            uint2 w;
            w.x = (uint32_t)tile[r * 9 + 0] | ((uint32_t)tile[r * 9 + 1] << 8) | ((uint32_t)tile[r * 9 + 2] << 16) |
                  ((uint32_t)tile[r * 9 + 3] << 24);
            w.y = (uint32_t)tile[r * 9 + 4] | ((uint32_t)tile[r * 9 + 5] << 8) | ((uint32_t)tile[r * 9 + 6] << 16) |
                  ((uint32_t)tile[r * 9 + 7] << 24);
            *reinterpret_cast<uint2*>(p.keys + (size_t)kk * frame_bytes + (size_t)Yo * p.W + (size_t)bx8 * 8) = w;
        }
        __syncwarp();
    }
}

}  // namespace kc
}  // namespace csenc
