/*
 * cs_synth.c -- seeded synthetic surveillance-video generator.
 *
 * INPUT GENERATOR ONLY.  This file draws pixels; it contains none of the
 * method's arithmetic (no residual, no measurement, no CR).  Both the oracle
 * (oracle/) and the CUDA path (paper_1311_1419_b200/) consume its output, and
 * neither side imports the other.
 *
 * Scene model (stand-in for the paper's QCIF "hall monitor"/"biker" clips,
 * PAPER.md:99 sec.4, which are not available and are never reproduced):
 *   - "a well defined, relatively static background" (sec.2.1):
 *     2-octave smoothstep value noise, lattice periods P and P/4 with weights
 *     0.75/0.25, mapped to [40,200]; optional slow global brightness drift.
 *   - moving objects: axis-aligned constant-intensity rectangles, sub-pixel
 *     constant velocity, reflecting off the frame edges, rasterised at
 *     rint(position).
 *   - additive per-pixel Gaussian noise N(0, sigma^2) on every frame, then
 *     rint + clamp to [0,255] (the add_noise model of SPEC.md:447-455).
 * Randomness is counter based (SplitMix64 of (seed, frame, pixel-pair)), so a
 * frame is a pure function of its arguments regardless of thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* SplitMix64 output for counter i of stream 'key' */
static inline uint64_t sm64_at(uint64_t key, uint64_t i) {
    return sm64_mix(key + (i + 1ull) * 0x9E3779B97F4A7C15ull);
}
/* uniform in (0,1] with 53 random bits */
static inline double u01(uint64_t r) { return ((double)(r >> 11) + 1.0) * (1.0 / 9007199254740992.0); }

static inline double lattice(uint64_t key, int64_t ix, int64_t iy) {
    uint64_t h = sm64_mix(key ^ sm64_mix((uint64_t)ix * 0x632BE59BD9B4E019ull ^ ((uint64_t)iy + 0x1234567ull)));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0); /* [0,1) */
}
static inline double smoothstep(double t) { return t * t * (3.0 - 2.0 * t); }

static double value_noise(uint64_t key, double x, double y, double period) {
    double gx = x / period, gy = y / period;
    double fx = floor(gx), fy = floor(gy);
    int64_t ix = (int64_t)fx, iy = (int64_t)fy;
    double tx = smoothstep(gx - fx), ty = smoothstep(gy - fy);
    double v00 = lattice(key, ix, iy), v10 = lattice(key, ix + 1, iy);
    double v01 = lattice(key, ix, iy + 1), v11 = lattice(key, ix + 1, iy + 1);
    double a = v00 + (v10 - v00) * tx, b = v01 + (v11 - v01) * tx;
    return a + (b - a) * ty;
}

/* Static background [H][W] in [40,200]. */
void cs_synth_background(int W, int H, int period, uint64_t seed, float* out) {
    if (period < 4) period = 4;
    uint64_t k0 = sm64_mix(seed ^ 0xB0B0B0B0ull), k1 = sm64_mix(seed ^ 0xC1C1C1C1ull);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double v = 0.75 * value_noise(k0, x + 0.5, y + 0.5, (double)period) +
                       0.25 * value_noise(k1, x + 0.5, y + 0.5, (double)period / 4.0);
            out[(size_t)y * W + x] = (float)(40.0 + 160.0 * v);
        }
}

/* reflect p into [0, L] (triangular wave) */
static double reflect(double p, double L) {
    if (L <= 0.0) return 0.0;
    double m = fmod(p, 2.0 * L);
    if (m < 0.0) m += 2.0 * L;
    return m > L ? 2.0 * L - m : m;
}

/*
 * Render T frames of one stream into out[T][H][W].
 *   objs: n_obj records of 7 doubles {x0, y0, vx, vy, w, h, intensity}
 *   frame t: background + drift_amp*sin(2*pi*(t0+t)/drift_period) (drift_period > 0),
 *   objects painted in order, + sigma * N(0,1), rint, clamp.
 *   t0 = index of the first rendered frame (so a stream can be rendered in pieces).
 */
void cs_synth_frames(int W, int H, int T, int t0, const float* bg, double drift_amp, int drift_period,
                     int n_obj, const double* objs, double sigma, uint64_t noise_seed, uint8_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int ti = 0; ti < T; ++ti) {
        int t = t0 + ti;
        uint8_t* f = out + (size_t)ti * W * H;
        double drift = drift_period > 0 ? drift_amp * sin(6.283185307179586 * t / (double)drift_period) : 0.0;
        uint64_t key = sm64_mix(noise_seed ^ sm64_mix(0xF00DF00Dull + (uint64_t)t));
        /* object rectangles for this frame */
        int rx0[16], ry0[16], rx1[16], ry1[16], ri[16];
        int no = n_obj > 16 ? 16 : n_obj;
        for (int o = 0; o < no; ++o) {
            const double* d = objs + 7 * o;
            int w = (int)d[4], h = (int)d[5];
            double px = reflect(d[0] + d[2] * t, (double)(W - w));
            double py = reflect(d[1] + d[3] * t, (double)(H - h));
            rx0[o] = (int)rint(px); ry0[o] = (int)rint(py);
            rx1[o] = rx0[o] + w; ry1[o] = ry0[o] + h;
            ri[o] = (int)d[6];
        }
        for (int y = 0; y < H; ++y) {
            const float* b = bg + (size_t)y * W;
            uint8_t* row = f + (size_t)y * W;
            for (int x = 0; x < W; x += 2) {
                uint64_t pair = ((uint64_t)y * (uint64_t)W + (uint64_t)x) >> 1;
                double z0 = 0.0, z1 = 0.0;
                if (sigma > 0.0) {
                    uint64_t r1 = sm64_at(key, 2 * pair), r2 = sm64_at(key, 2 * pair + 1);
                    double rad = sqrt(-2.0 * log(u01(r1)));
                    double ang = 6.283185307179586 * u01(r2);
                    z0 = rad * cos(ang);
                    z1 = rad * sin(ang);
                }
                for (int k = 0; k < 2 && x + k < W; ++k) {
                    int xx = x + k;
                    double v = (double)b[xx] + drift;
                    for (int o = 0; o < no; ++o)
                        if (xx >= rx0[o] && xx < rx1[o] && y >= ry0[o] && y < ry1[o]) v = (double)ri[o];
                    v += sigma * (k == 0 ? z0 : z1);
                    v = rint(v);
                    row[xx] = (uint8_t)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
                }
            }
        }
    }
}

int cs_synth_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
