/*
 * holo_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what the
 * hot path of arXiv 2004.04049 ("Lookup tables for phase randomisation in
 * Gerchberg-Saxton and One-Step Phase-Retrieval holography") computes.
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "R-k" = reading k of DESIGN.md §3 (same numbering as SURVEY.md §8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA library under
 * paper_2004_04049_b200/csrc, and neither side includes the other.
 *
 * Compiled with -ffp-contract=off so that every a*b+c is two roundings, as
 * the phase recipe R-5 requires.
 *
 * Conventions: images are row-major data[y][x] (R-10); complex fields are
 * interleaved (re, im) doubles (C99 double _Complex has that layout);
 * the DFT pair is unitary with 1/sqrt(Nx*Ny) in both directions (P:39-40,
 * Eqs. (1)-(2); R-9); DC sits at [0][0] with no shift (R-10).
 *
 * Every function below is pinned by tests/test_oracle_*.py except where its
 * comment says "parity unpinned".
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

#define OR_PI 3.14159265358979323846264338327950288

/* ------------------------------------------------------------------ */
/* a0: the phase pool ("Random numbers can be generated at compile  */
/* time to fill the LUT"; R-3, R-4, R-5)                                */
/* ------------------------------------------------------------------ */

/* SplitMix64 in counter form (R-4): output k of the generator seeded with
 * `seed` is mix64(seed + (k+1)*gamma).  Pinned against the published
 * first outputs for seed 0 (tests/golden/splitmix64.txt). */
uint64_t or_splitmix64(uint64_t seed, uint64_t k)
{
    uint64_t z = seed + (k + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* 32-bit angle code of pool entry k: the high word (R-3: phi = 2*pi*u/2^32). */
uint32_t or_angle_code(uint64_t seed, uint64_t k)
{
    return (uint32_t)(or_splitmix64(seed, k) >> 32);
}

/* R-5 step 3: sin and cos of x in [0, pi/4] by Taylor polynomials in Horner
 * form, sin to x^17 and cos to x^16, plain double mul/add in this order. */
static double or_sin_poly(double x)
{
    double s = x * x;
    double p = 1.0 / 355687428096000.0;        /* 1/17! */
    p = -1.0 / 1307674368000.0 + s * p;        /* 1/15! */
    p = 1.0 / 6227020800.0 + s * p;            /* 1/13! */
    p = -1.0 / 39916800.0 + s * p;             /* 1/11! */
    p = 1.0 / 362880.0 + s * p;                /* 1/9!  */
    p = -1.0 / 5040.0 + s * p;                 /* 1/7!  */
    p = 1.0 / 120.0 + s * p;                   /* 1/5!  */
    p = -1.0 / 6.0 + s * p;                    /* 1/3!  */
    p = 1.0 + s * p;
    return x * p;
}

static double or_cos_poly(double x)
{
    double s = x * x;
    double p = 1.0 / 20922789888000.0;         /* 1/16! */
    p = -1.0 / 87178291200.0 + s * p;          /* 1/14! */
    p = 1.0 / 479001600.0 + s * p;             /* 1/12! */
    p = -1.0 / 3628800.0 + s * p;              /* 1/10! */
    p = 1.0 / 40320.0 + s * p;                 /* 1/8!  */
    p = -1.0 / 720.0 + s * p;                  /* 1/6!  */
    p = 1.0 / 24.0 + s * p;                    /* 1/4!  */
    p = -1.0 / 2.0 + s * p;                    /* 1/2!  */
    p = 1.0 + s * p;
    return p;
}

/* R-5 steps 1-4: (cos phi, sin phi) in double for phi = 2*pi*u/2^32.
 * Octant o = u >> 29 covers [o*pi/4, (o+1)*pi/4); the in-octant offset is
 * reflected for odd octants so that x always lies in [0, pi/4]. */
void or_phase_f64(uint32_t u, double *c, double *s)
{
    uint32_t o = u >> 29;
    uint32_t f = u & 0x1FFFFFFFu;
    if (o & 1u)
        f = 0x20000000u - f;
    double x = (double)f * (OR_PI / 2147483648.0); /* fl(pi/2^31), one multiply */
    double S = or_sin_poly(x), C = or_cos_poly(x);
    double cc, ss;
    switch (o) {
    case 0: cc = C;  ss = S;  break;  /* phi = x           */
    case 1: cc = S;  ss = C;  break;  /* phi = pi/2 - x    */
    case 2: cc = -S; ss = C;  break;  /* phi = pi/2 + x    */
    case 3: cc = -C; ss = S;  break;  /* phi = pi - x      */
    case 4: cc = -C; ss = -S; break;  /* phi = pi + x      */
    case 5: cc = -S; ss = -C; break;  /* phi = 3pi/2 - x   */
    case 6: cc = S;  ss = -C; break;  /* phi = 3pi/2 + x   */
    default: cc = C; ss = -S; break;  /* phi = 2pi - x     */
    }
    *c = cc;
    *s = ss;
}

/* R-5 steps 5-6: round to fp32 (round-to-nearest-even) and map -0 to +0. */
void or_phase_f32(uint32_t u, float *c, float *s)
{
    double cd, sd;
    or_phase_f64(u, &cd, &sd);
    float cf = (float)cd, sf = (float)sd;
    *c = (cf == 0.0f) ? 0.0f : cf;
    *s = (sf == 0.0f) ? 0.0f : sf;
}

/* Batch form of or_phase_f64 for the tests: cs[2i], cs[2i+1] = cos, sin. */
void or_phase_f64_batch(const uint32_t *u, uint64_t m, double *cs)
{
    for (uint64_t i = 0; i < m; ++i)
        or_phase_f64(u[i], &cs[2 * i], &cs[2 * i + 1]);
}

/* Build the pool: lut[2k], lut[2k+1] = cos, sin of entry k, k < n_lut
 * (S:121-129 build_lut; S:183 stores (cos, sin) pairs). */
void or_lut_build(uint64_t seed, uint64_t n_lut, float *lut)
{
    for (uint64_t k = 0; k < n_lut; ++k)
        or_phase_f32(or_angle_code(seed, k), &lut[2 * k], &lut[2 * k + 1]);
}

/* ------------------------------------------------------------------ */
/* a1/a2: cyclic consumption and randomisation ("cycled through     */
/* sequentially with successive frames and sub-frames continuing from   */
/* where the previous left off"; Fig. 3; R-1, R-2, R-6)       */
/* ------------------------------------------------------------------ */

/* Pool index of global draw number g (cursor = g mod N_LUT). */
uint64_t or_lut_index(uint64_t g, uint64_t n_lut)
{
    return g % n_lut;
}

/* Phase factor of draw g: flat 1+0i when N_LUT = 0 (R-6), else lut[g mod N_LUT]. */
static cplx or_phase_of_draw(const float *lut, uint64_t n_lut, uint64_t g)
{
    if (n_lut == 0)
        return 1.0;
    uint64_t k = or_lut_index(g, n_lut);
    return (double)lut[2 * k] + I * (double)lut[2 * k + 1];
}

/* apply_phase: R[p] = T[p] * phase(cursor + p), p row-major.
 * The product of two fp32 numbers is exact in double. */
void or_apply_phase(const float *T, int n, const float *lut, uint64_t n_lut,
                    uint64_t cursor, cplx *R)
{
    uint64_t P = (uint64_t)n * (uint64_t)n;
    for (uint64_t p = 0; p < P; ++p)
        R[p] = (double)T[p] * or_phase_of_draw(lut, n_lut, cursor + p);
}

/* The software PRNG source of P:68 (independent phases, no LUT): draw g uses
 * the recipe on the g-th generator output.  A LUT of length >= all draws is
 * indistinguishable from it (pin c3 #15). */
void or_apply_phase_prng(const float *T, int n, uint64_t seed, uint64_t cursor, cplx *R)
{
    uint64_t P = (uint64_t)n * (uint64_t)n;
    for (uint64_t p = 0; p < P; ++p) {
        float c, s;
        or_phase_f32(or_angle_code(seed, cursor + p), &c, &s);
        R[p] = (double)T[p] * ((double)c + I * (double)s);
    }
}

/* The paper's runtime-flexible alternative ("PRNGs with LUTs for sin
 * and cosine functions"; R-25): a PRNG per draw, its phase quantised to
 * 2^q levels so that (cos, sin) comes from a 2^q-entry table.  Draw g takes
 * the top q bits of the angle code, i.e. the code truncated to a multiple of
 * 2^(32-q), and the recipe at that code -- written out here without a table:
 * phase(g) = R-5(u_g & ~(2^(32-q) - 1)), 1 <= q <= 32 (q = 32: or_apply_phase_prng). */
void or_apply_phase_prng_q(const float *T, int n, uint64_t seed, uint64_t cursor, int q, cplx *R)
{
    uint64_t P = (uint64_t)n * (uint64_t)n;
    uint32_t mask = q >= 32 ? 0xFFFFFFFFu : ~((1u << (32 - q)) - 1u);
    for (uint64_t p = 0; p < P; ++p) {
        float c, s;
        or_phase_f32(or_angle_code(seed, cursor + p) & mask, &c, &s);
        R[p] = (double)T[p] * ((double)c + I * (double)s);
    }
}

/* ------------------------------------------------------------------ */
/* A1-A3: the unitary DFT pair (Eqs. (1)-(2)) and its FFT */
/* ------------------------------------------------------------------ */

/* Eq. (1) (inverse = 0) / Eq. (2) (inverse = 1) by direct O(N^4) summation:
 * out[v][u] = 1/sqrt(NxNy) sum_y sum_x in[y][x] exp(-/+ 2 pi i (ux/Nx + vy/Ny)). */
void or_dft2_direct(const cplx *in, cplx *out, int nx, int ny, int inverse)
{
    double sg = inverse ? 1.0 : -1.0;
    double scale = 1.0 / sqrt((double)nx * (double)ny);
    for (int v = 0; v < ny; ++v)
        for (int u = 0; u < nx; ++u) {
            cplx acc = 0.0;
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    double ang = sg * 2.0 * OR_PI * ((double)u * x / nx + (double)v * y / ny);
                    acc += in[(size_t)y * nx + x] * (cos(ang) + I * sin(ang));
                }
            out[(size_t)v * nx + u] = acc * scale;
        }
}

/* 1D direct DFT of length m with stride (used by the O(N^3) separable sum). */
static void or_dft1_direct(const cplx *in, cplx *out, int m, size_t stride, int inverse)
{
    double sg = inverse ? 1.0 : -1.0;
    for (int k = 0; k < m; ++k) {
        cplx acc = 0.0;
        for (int j = 0; j < m; ++j) {
            /* reduce k*j mod m first so the angle stays small and exact */
            double ang = sg * 2.0 * OR_PI * (double)(((long long)k * j) % m) / m;
            acc += in[(size_t)j * stride] * (cos(ang) + I * sin(ang));
        }
        out[(size_t)k * stride] = acc / sqrt((double)m);
    }
}

/* Eqs. (1)-(2) evaluated separably (rows, then columns) by direct sums: O(N^3). */
void or_dft2_separable(const cplx *in, cplx *out, int nx, int ny, int inverse)
{
    cplx *tmp = malloc(sizeof(cplx) * (size_t)nx * ny);
    for (int y = 0; y < ny; ++y)
        or_dft1_direct(in + (size_t)y * nx, tmp + (size_t)y * nx, nx, 1, inverse);
    for (int x = 0; x < nx; ++x)
        or_dft1_direct(tmp + x, out + x, ny, (size_t)nx, inverse);
    free(tmp);
}

/* Iterative radix-2 FFT (bit reversal, then log2(m) butterfly stages), unitary
 * 1/sqrt(m).  `tw` holds exp(sg*2*pi*i*k/m) for k < m/2. */
static void or_fft1_pow2(cplx *x, int m, const cplx *tw)
{
    for (int i = 1, j = 0; i < m; ++i) {
        int bit = m >> 1;
        for (; j & bit; bit >>= 1)
            j ^= bit;
        j ^= bit;
        if (i < j) {
            cplx t = x[i];
            x[i] = x[j];
            x[j] = t;
        }
    }
    for (int len = 2; len <= m; len <<= 1) {
        int step = m / len;
        for (int i = 0; i < m; i += len)
            for (int k = 0; k < len / 2; ++k) {
                cplx a = x[i + k];
                cplx b = x[i + k + len / 2] * tw[k * step];
                x[i + k] = a + b;
                x[i + k + len / 2] = a - b;
            }
    }
    double sc = 1.0 / sqrt((double)m);
    for (int i = 0; i < m; ++i)
        x[i] *= sc;
}

static int or_is_pow2(int m) { return m > 0 && (m & (m - 1)) == 0; }

/* In-place unitary 2D FFT of an n x n field (rows, then columns); n a power of 2.
 * Returns 0 on success, -1 if n is not a power of two. */
int or_fft2(cplx *a, int n, int inverse)
{
    if (!or_is_pow2(n))
        return -1;
    double sg = inverse ? 1.0 : -1.0;
    cplx *tw = malloc(sizeof(cplx) * (size_t)(n / 2 + 1));
    for (int k = 0; k < n / 2; ++k)
        tw[k] = cos(sg * 2.0 * OR_PI * k / n) + I * sin(sg * 2.0 * OR_PI * k / n);
    for (int y = 0; y < n; ++y)
        or_fft1_pow2(a + (size_t)y * n, n, tw);
    cplx *col = malloc(sizeof(cplx) * (size_t)n);
    for (int x = 0; x < n; ++x) {
        for (int y = 0; y < n; ++y)
            col[y] = a[(size_t)y * n + x];
        or_fft1_pow2(col, n, tw);
        for (int y = 0; y < n; ++y)
            a[(size_t)y * n + x] = col[y];
    }
    free(col);
    free(tw);
    return 0;
}

/* ------------------------------------------------------------------ */
/* A5: quantisation to the nearest acceptable value and packing   */
/* ------------------------------------------------------------------ */

/* Binary {0, pi} SLM: nearest of {+1, -1} is the sign of Re H;
 * Re H = 0 (including -0.0) maps to +1 (R-7).  Returns 1 for +1. */
int or_quantise_binary(double re)
{
    return re >= 0.0 ? 1 : 0;
}

/* Pack +1/-1 pixels (given as 1/0) row-major, MSB first, rows padded to whole
 * bytes (R-8). */
void or_pack_bits(const uint8_t *pm, int nx, int ny, uint8_t *out)
{
    int bpr = (nx + 7) / 8;
    memset(out, 0, (size_t)bpr * ny);
    for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x)
            if (pm[(size_t)y * nx + x])
                out[(size_t)y * bpr + x / 8] |= (uint8_t)(0x80u >> (x % 8));
}

/* Phase-only constraint of GS (R-14, R-15, R-16): levels = 0 gives the
 * continuous projection h/|h| (h = 0 -> +1); levels Q > 0 gives the nearest
 * of exp(2 pi i j / Q), j = floor(wrap(arg h) * Q / 2pi + 1/2) mod Q.
 * *level receives j (0 for the continuous case). */
cplx or_gs_constrain(cplx h, int levels, int *level)
{
    double re = creal(h), im = cimag(h);
    if (levels <= 0) {
        *level = 0;
        double m = sqrt(re * re + im * im);
        if (m == 0.0)
            return 1.0;
        return h / m;
    }
    double th = atan2(im, re);
    if (th < 0.0)
        th += 2.0 * OR_PI;
    long long j = (long long)floor(th * levels / (2.0 * OR_PI) + 0.5) % levels;
    *level = (int)j;
    double a = 2.0 * OR_PI * (double)j / levels;
    return cos(a) + I * sin(a);
}

/* ------------------------------------------------------------------ */
/* a7 / g4: the error metrics ("Mean Squared Error"; R-11, R-12)    */
/* ------------------------------------------------------------------ */

/* M-1: energy-normalised intensity MSE over the half-open region
 * [r0,r1) x [c0,c1): a = sum T^2 / sum I; MSE = mean (a I - T^2)^2.
 * If sum I = 0 then a = 0 and MSE = mean T^4.  Two passes, as written. */
double or_mse_m1(const double *Iv, const float *T, int n, int r0, int r1, int c0, int c1)
{
    double sT2 = 0.0, sI = 0.0;
    for (int y = r0; y < r1; ++y)
        for (int x = c0; x < c1; ++x) {
            double t = T[(size_t)y * n + x];
            sT2 += t * t;
            sI += Iv[(size_t)y * n + x];
        }
    double a = (sI == 0.0) ? 0.0 : sT2 / sI;
    double acc = 0.0;
    for (int y = r0; y < r1; ++y)
        for (int x = c0; x < c1; ++x) {
            double t = T[(size_t)y * n + x];
            double d = a * Iv[(size_t)y * n + x] - t * t;
            acc += d * d;
        }
    return acc / ((double)(r1 - r0) * (double)(c1 - c0));
}

/* SPEC's secondary amplitude metric: A = sqrt(I), alpha = <A,T>/<A,A>
 * (0 if A = 0), MSE = mean (alpha A - T)^2.  Not exported by the GPU library. */
double or_mse_alpha(const double *Iv, const float *T, int n, int r0, int r1, int c0, int c1)
{
    double sAT = 0.0, sAA = 0.0;
    for (int y = r0; y < r1; ++y)
        for (int x = c0; x < c1; ++x) {
            double A = sqrt(Iv[(size_t)y * n + x]);
            sAT += A * T[(size_t)y * n + x];
            sAA += A * A;
        }
    double al = (sAA == 0.0) ? 0.0 : sAT / sAA;
    double acc = 0.0;
    for (int y = r0; y < r1; ++y)
        for (int x = c0; x < c1; ++x) {
            double d = al * sqrt(Iv[(size_t)y * n + x]) - T[(size_t)y * n + x];
            acc += d * d;
        }
    return acc / ((double)(r1 - r0) * (double)(c1 - c0));
}

/* ------------------------------------------------------------------ */
/* OSPR (Fig. 2 right; steps a1-a7)               */
/* ------------------------------------------------------------------ */

/* One sub-frame whose first draw is `cursor`:
 *   R = apply_phase(T)            (a2)
 *   H = F^-1{R}                   (a3, "H = F^-1{R}")
 *   H' = quantise(H)              (a4)
 *   R' = F{H'}                    (a5, "R' = F{H'}")
 *   intensity += |R'|^2           (a6, when intensity != NULL)
 * bits: packed H' [n][n/8] (nullable); h_re: Re H [n][n] (nullable).
 * Returns 0, or -1 if n is not a power of two. */
int or_ospr_subframe(const float *T, int n, const float *lut, uint64_t n_lut,
                     uint64_t cursor, uint8_t *bits, double *h_re, double *intensity)
{
    if (!or_is_pow2(n))
        return -1;
    size_t P = (size_t)n * n;
    cplx *f = malloc(sizeof(cplx) * P);
    uint8_t *pm = malloc(P);
    or_apply_phase(T, n, lut, n_lut, cursor, f);
    or_fft2(f, n, 1);
    for (size_t p = 0; p < P; ++p) {
        if (h_re)
            h_re[p] = creal(f[p]);
        pm[p] = (uint8_t)or_quantise_binary(creal(f[p]));
    }
    if (bits)
        or_pack_bits(pm, n, n, bits);
    if (intensity) {
        for (size_t p = 0; p < P; ++p)
            f[p] = pm[p] ? 1.0 : -1.0;
        or_fft2(f, n, 0);
        for (size_t p = 0; p < P; ++p)
            intensity[p] += creal(f[p]) * creal(f[p]) + cimag(f[p]) * cimag(f[p]);
    }
    free(pm);
    free(f);
    return 0;
}

/* Time-averaged replay of packed binary sub-frames:
 * intensity = (1/n_sub) sum_s |F{H'_s}|^2.  Used for the conditional parity
 * protocol P-4 (the oracle forward-propagates the GPU's bits). */
int or_replay_from_bits(const uint8_t *bits, int n, int n_sub, double *intensity)
{
    if (!or_is_pow2(n) || n % 8)
        return -1;
    size_t P = (size_t)n * n, bpr = (size_t)n / 8;
    cplx *f = malloc(sizeof(cplx) * P);
    memset(intensity, 0, sizeof(double) * P);
    for (int s = 0; s < n_sub; ++s) {
        const uint8_t *b = bits + (size_t)s * bpr * n;
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x)
                f[(size_t)y * n + x] = ((b[y * bpr + x / 8] >> (7 - x % 8)) & 1u) ? 1.0 : -1.0;
        or_fft2(f, n, 0);
        for (size_t p = 0; p < P; ++p)
            intensity[p] += creal(f[p]) * creal(f[p]) + cimag(f[p]) * cimag(f[p]);
    }
    for (size_t p = 0; p < P; ++p)
        intensity[p] /= n_sub;
    free(f);
    return 0;
}

/* Full OSPR over n_frames frames of n_sub sub-frames each.  Frame f sub-frame
 * s starts at draw cursor0 + (f*n_sub + s)*N^2 (R-2).  Outputs (nullable
 * except intensity): bits [F][n_sub][n][n/8], intensity [F][n][n] (mean over
 * sub-frames, R-18), mse [F] (M-1 over the region). */
int or_ospr(const float *T, int n, int n_frames, int n_sub, const float *lut,
            uint64_t n_lut, uint64_t cursor0, uint8_t *bits, double *intensity,
            double *mse, int r0, int r1, int c0, int c1)
{
    if (!or_is_pow2(n) || n % 8 || n_frames < 1 || n_sub < 1)
        return -1;
    size_t P = (size_t)n * n, bsz = P / 8;
    for (int fr = 0; fr < n_frames; ++fr) {
        double *Iv = intensity + (size_t)fr * P;
        memset(Iv, 0, sizeof(double) * P);
        for (int s = 0; s < n_sub; ++s) {
            uint64_t cur = cursor0 + ((uint64_t)fr * n_sub + s) * P;
            or_ospr_subframe(T + (size_t)fr * P, n, lut, n_lut, cur,
                             bits ? bits + ((size_t)fr * n_sub + s) * bsz : NULL, NULL, Iv);
        }
        for (size_t p = 0; p < P; ++p)
            Iv[p] /= n_sub;
        if (mse)
            mse[fr] = or_mse_m1(Iv, T + (size_t)fr * P, n, r0, r1, c0, c1);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* GS (Fig. 2 left; steps g0-g6; R-14..R-17)      */
/* ------------------------------------------------------------------ */

/* One GS iteration from the replay-plane field R_in = R_{k-1}:
 *   H_k  = F^-1{R_{k-1}}                         (g1)
 *   h_k  = constrain(H_k)                        (g2)
 *   R'_k = F{h_k}                                (g3)
 *   I_k = |R'_k|^2; mse = M-1 over the region; E = sum_all (|R'_k| - T)^2 (g4)
 *   R_k  = T R'_k / |R'_k|  (|R'_k| = 0 -> T)    (g5)
 * Outputs (all nullable): R_out, holo (h_k), lev (uint8 level if levels in
 * 1..256), Iv, mse, E. */
int or_gs_step(const cplx *R_in, const float *T, int n, int levels, cplx *R_out,
               cplx *holo, uint8_t *lev, double *Iv, double *mse, double *E,
               int r0, int r1, int c0, int c1)
{
    if (!or_is_pow2(n))
        return -1;
    size_t P = (size_t)n * n;
    cplx *f = malloc(sizeof(cplx) * P);
    double *Ii = malloc(sizeof(double) * P);
    memcpy(f, R_in, sizeof(cplx) * P);
    or_fft2(f, n, 1);
    for (size_t p = 0; p < P; ++p) {
        int j;
        f[p] = or_gs_constrain(f[p], levels, &j);
        if (holo)
            holo[p] = f[p];
        if (lev && levels >= 1 && levels <= 256)
            lev[p] = (uint8_t)j;
    }
    or_fft2(f, n, 0);
    double e = 0.0;
    for (size_t p = 0; p < P; ++p) {
        double re = creal(f[p]), im = cimag(f[p]);
        double m2 = re * re + im * im, m = sqrt(m2);
        Ii[p] = m2;
        double d = m - (double)T[p];
        e += d * d;
        if (R_out)
            R_out[p] = (m == 0.0) ? (cplx)(double)T[p] : (double)T[p] * (f[p] / m);
    }
    if (Iv)
        memcpy(Iv, Ii, sizeof(double) * P);
    if (mse)
        *mse = or_mse_m1(Ii, T, n, r0, r1, c0, c1);
    if (E)
        *E = e;
    free(Ii);
    free(f);
    return 0;
}

/* Full GS for one frame whose initial phase draws start at `cursor` (g0; the
 * LUT is used only for the initial random phase, BASELINE configs[1]).
 * Outputs: holo [n][n] complex final h, lev [n][n] (if 1 <= levels <= 256),
 * I_final [n][n], mse [iters], E [iters] (all nullable). */
int or_gs(const float *T, int n, int iters, const float *lut, uint64_t n_lut,
          uint64_t cursor, int levels, cplx *holo, uint8_t *lev, double *I_final,
          double *mse, double *E, int r0, int r1, int c0, int c1)
{
    if (!or_is_pow2(n) || iters < 1)
        return -1;
    size_t P = (size_t)n * n;
    cplx *R = malloc(sizeof(cplx) * P), *R2 = malloc(sizeof(cplx) * P);
    or_apply_phase(T, n, lut, n_lut, cursor, R);
    for (int k = 0; k < iters; ++k) {
        int last = (k == iters - 1);
        or_gs_step(R, T, n, levels, R2, last ? holo : NULL, last ? lev : NULL,
                   last ? I_final : NULL, mse ? &mse[k] : NULL, E ? &E[k] : NULL,
                   r0, r1, c0, c1);
        cplx *t = R;
        R = R2;
        R2 = t;
    }
    free(R);
    free(R2);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Host utilities of §5.1 and the conclusion */
/* ------------------------------------------------------------------ */

int or_is_prime(uint64_t m)
{
    if (m < 2)
        return 0;
    for (uint64_t d = 2; d * d <= m; ++d)
        if (m % d == 0)
            return 0;
    return 1;
}

uint64_t or_next_prime_above(uint64_t m)
{
    uint64_t q = m + 1;
    while (!or_is_prime(q))
        ++q;
    return q;
}
