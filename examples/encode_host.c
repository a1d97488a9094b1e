/* encode_host.c -- the C ABI used directly from C (no Python): create an encoder, encode host
 * frames through cs_encode_batch_host, check every measurement against a plain double-precision
 * sum written here, report the compression ratio.  Build (done by __graft_entry__.build()):
 *   gcc -O2 -std=c11 -I include examples/encode_host.c -L paper_1311_1419_b200/_lib -lcsenc \
 *       -Wl,-rpath,'$ORIGIN/../paper_1311_1419_b200/_lib' -lm -o examples/encode_host
 * Run on a B200: examples/encode_host  -> prints "encode_host OK ..." and exits 0. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cs_encoder.h"

/* fp16 bit pattern of a value that is exactly representable (|v| in [2^-14, 2^15] or 0) */
static uint16_t half_bits(double v) {
    if (v == 0.0) return 0;
    uint16_t sgn = v < 0 ? 0x8000u : 0u;
    double a = fabs(v);
    int e = 0;
    double m = frexp(a, &e); /* a = m * 2^e, m in [0.5, 1) */
    int exp16 = e - 1 + 15;
    uint16_t mant = (uint16_t)((m * 2.0 - 1.0) * 1024.0 + 0.5);
    return (uint16_t)(sgn | (uint16_t)(exp16 << 10) | mant);
}

int main(void) {
    const int W = 176, H = 144, G = 4, B = 16, M = 32, T = 10; /* QCIF, short last GOP (10 = 4+4+2) */
    const int N = B * B;
    uint16_t* phi = (uint16_t*)malloc(sizeof(uint16_t) * M * N);
    double* phid = (double*)malloc(sizeof(double) * M * N);
    uint32_t lcg = 12345u;
    for (int i = 0; i < M * N; ++i) { /* multiples of 1/64 in [-0.5, 0.5]: exact in fp16 */
        lcg = lcg * 1664525u + 1013904223u;
        phid[i] = ((int)((lcg >> 16) % 65) - 32) / 64.0;
        phi[i] = half_bits(phid[i]);
    }
    uint8_t* frames = (uint8_t*)malloc((size_t)T * W * H);
    for (size_t i = 0; i < (size_t)T * W * H; ++i) {
        lcg = lcg * 1664525u + 1013904223u;
        frames[i] = (uint8_t)(lcg >> 24);
    }
    cs_encoder* enc = NULL;
    int rc = cs_encoder_create(W, H, G, B, M, phi, &enc);
    if (rc != CS_OK) {
        fprintf(stderr, "cs_encoder_create: %d %s\n", rc, cs_last_error());
        return 1;
    }
    const int64_t n_meas = cs_measurement_count(enc, 1, T);
    float* out = (float*)malloc(sizeof(float) * (size_t)n_meas);
    rc = cs_encode_batch_host(enc, frames, 1, T, out);
    if (rc != CS_OK) {
        fprintf(stderr, "cs_encode_batch_host: %d %s\n", rc, cs_last_error());
        return 1;
    }
    /* y[c][by][bx][m] = sum_j phi[m][j] * (F_cs - F_key)[block pixel j], OOB pixels 0 */
    const int nbx = (W + B - 1) / B, nby = (H + B - 1) / B;
    double worst = 0.0;
    int64_t idx = 0;
    for (int g = 0; g * G < T; ++g) {
        const int key = g * G;
        for (int t = key + 1; t < T && t < key + G; ++t)
            for (int by = 0; by < nby; ++by)
                for (int bx = 0; bx < nbx; ++bx)
                    for (int m = 0; m < M; ++m, ++idx) {
                        double y = 0.0, s = 0.0;
                        for (int yy = 0; yy < B; ++yy)
                            for (int xx = 0; xx < B; ++xx) {
                                const int r = by * B + yy, c = bx * B + xx;
                                if (r >= H || c >= W) continue;
                                const double d = (double)frames[(size_t)t * W * H + (size_t)r * W + c] -
                                                 (double)frames[(size_t)key * W * H + (size_t)r * W + c];
                                y += phid[m * N + yy * B + xx] * d;
                                s += fabs(phid[m * N + yy * B + xx] * d);
                            }
                        const double err = fabs((double)out[idx] - y);
                        const double rel = s > 0 ? err / s : (err > 0 ? INFINITY : 0.0);
                        if (rel > worst) worst = rel;
                    }
    }
    if (idx != n_meas) {
        fprintf(stderr, "count mismatch %lld vs %lld\n", (long long)idx, (long long)n_meas);
        return 1;
    }
    const double cr = cs_compression_ratio(enc, T, 1.0, 8);
    cs_encoder_destroy(enc);
    const int ok = worst <= 1e-5;
    printf("encode_host %s measurements=%lld max|dy|/S=%.3g CR(T=%d, raw key, 8 bit)=%.4f (%s)\n", ok ? "OK" : "FAIL",
           (long long)n_meas, worst, T, cr, cs_version());
    free(out);
    free(frames);
    free(phi);
    free(phid);
    return ok ? 0 : 1;
}
