/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. The plain, slow, CPU double-precision
 * oracle for the per-record DFT of arXiv 1407.6915. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library. It shares no code, header, table or constant with
 * the CUDA path under paper_1407_6915_b200/ and neither imports the other.
 *
 * What it computes (the paper fixes no formula for the
 * transform itself, only that it is Cooley–Tukey, §I, and that
 * each FFT segment is transformed independently, §III):
 *
 *   forward  X[k] = sum_{j<N} x[j] * exp(-2*pi*i*j*k/N)          (unnormalised)
 *   inverse  x[j] = (1/N) * sum_{k<N} X[k] * exp(+2*pi*i*j*k/N)
 *
 * Sign and normalisation are readings c2/c3 in DESIGN.md (SPEC.md:36, :55,
 * :75, :90).  Two independent algorithms are provided:
 *
 *   oracle_dft : the O(N^2) direct definition (SPEC.md:72-80 dft_oracle),
 *                any N >= 1.  The exponent j*k is reduced modulo N in integer
 *                arithmetic before the angle 2*pi*m/N is formed, and the sum
 *                is accumulated in plain j order.
 *   oracle_fft : the textbook recursive radix-2 decimation-in-time
 *                Cooley–Tukey FFT (§I "Cooley–Tukey algorithm";
 *                north_star "textbook recursive radix-2"), N a power of two.
 *                E = fft(x[0::2]), O = fft(x[1::2]);
 *                X[k] = E[k] + w_k O[k],  X[k+N/2] = E[k] - w_k O[k],
 *                w_k = cos(2*pi*k/N) - i sin(2*pi*k/N) computed directly per k
 *                (no recurrence).  Inverse = conj(fft(conj(X)))/N.
 *
 * Data layout: interleaved (re, im) doubles, record-major, as the file format
 * (SPEC.md:99, :190).  Batch entry points decode complex64 (float re, im)
 * records, promote each value exactly to double, and transform each record
 * independently ("partitioning of FFT segments").
 *
 * Build: gcc -O2 -fopenmp (no -ffast-math), see __graft_entry__.build().
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_PI 3.14159265358979323846264338327950288

static int is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

/* Direct DFT of one record (inverse per SPEC.md:90).
 * in, out: 2*n doubles each, must not alias.  dir = -1 forward, +1 inverse.
 * Returns 0, or -1 on bad arguments. */
int oracle_dft(const double *in, double *out, int64_t n, int dir)
{
    if (n < 1 || (dir != -1 && dir != 1) || in == out) return -1;
    for (int64_t k = 0; k < n; ++k) {
        double sr = 0.0, si = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            int64_t m = (j * k) % n;                 /* exact integer reduction */
            double ang = 2.0 * ORACLE_PI * (double)m / (double)n;
            double c = cos(ang);
            double s = (double)dir * sin(ang);       /* e^{dir*i*ang} */
            double xr = in[2 * j], xi = in[2 * j + 1];
            sr += xr * c - xi * s;
            si += xr * s + xi * c;
        }
        if (dir == 1) { sr /= (double)n; si /= (double)n; }
        out[2 * k] = sr;
        out[2 * k + 1] = si;
    }
    return 0;
}

/* Recursive radix-2 DIT forward transform of the n samples x[0], x[stride],
 * x[2*stride], ... written to X[0..n) (contiguous).  The even half's transform
 * E lands in X[0..n/2), the odd half's O in X[n/2..n); the butterfly then
 * combines them in place. */
static void fft_rec(const double *x, int64_t stride, double *X, int64_t n)
{
    if (n == 1) {
        X[0] = x[0];
        X[1] = x[1];
        return;
    }
    int64_t h = n / 2;
    fft_rec(x, 2 * stride, X, h);                 /* E = fft(x[0::2]) */
    fft_rec(x + 2 * stride, 2 * stride, X + 2 * h, h); /* O = fft(x[1::2]) */
    for (int64_t k = 0; k < h; ++k) {
        double ang = 2.0 * ORACLE_PI * (double)k / (double)n;
        double wr = cos(ang), wi = -sin(ang);     /* w_k = e^{-2 pi i k/n} */
        double er = X[2 * k], ei = X[2 * k + 1];
        double orr = X[2 * (k + h)], oi = X[2 * (k + h) + 1];
        double tr = wr * orr - wi * oi;           /* t = w_k * O[k] */
        double ti = wr * oi + wi * orr;
        X[2 * k] = er + tr;
        X[2 * k + 1] = ei + ti;
        X[2 * (k + h)] = er - tr;
        X[2 * (k + h) + 1] = ei - ti;
    }
}

/* Recursive radix-2 FFT of one record, n a power of two.  in, out: 2*n
 * doubles, must not alias.  Inverse = conj(fft(conj(X)))/n.
 * Returns 0, or -1 on bad arguments / allocation failure. */
int oracle_fft(const double *in, double *out, int64_t n, int dir)
{
    if (!is_pow2(n) || (dir != -1 && dir != 1) || in == out) return -1;
    if (dir == -1) {
        fft_rec(in, 1, out, n);
        return 0;
    }
    double *c = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    if (!c) return -1;
    for (int64_t j = 0; j < n; ++j) { c[2 * j] = in[2 * j]; c[2 * j + 1] = -in[2 * j + 1]; }
    fft_rec(c, 1, out, n);
    for (int64_t k = 0; k < n; ++k) {
        out[2 * k] = out[2 * k] / (double)n;
        out[2 * k + 1] = -out[2 * k + 1] / (double)n;
    }
    free(c);
    return 0;
}

/* Transform `batch` independent complex64 records of n points each.
 * in:  batch*n*2 floats (interleaved re, im), promoted exactly to double.
 * out: batch*n*2 doubles.
 * algo: 0 = recursive radix-2 (oracle_fft), 1 = direct DFT (oracle_dft).
 * nthreads: OpenMP threads over records (<= 0: library default).
 * Returns 0 on success, -1 if any record failed. */
int oracle_batch_c64(const float *in, double *out, int64_t n, int64_t batch,
                     int dir, int algo, int nthreads)
{
    if (n < 1 || batch < 0 || (algo != 0 && algo != 1)) return -1;
    if (algo == 0 && !is_pow2(n)) return -1;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
    for (int64_t r = 0; r < batch; ++r) {
        double *x = (double *)malloc(sizeof(double) * 2 * (size_t)n);
        if (!x) { bad |= 1; continue; }
        const float *src = in + (size_t)r * 2 * (size_t)n;
        for (int64_t j = 0; j < 2 * n; ++j) x[j] = (double)src[j];   /* exact */
        double *dst = out + (size_t)r * 2 * (size_t)n;
        int rc = (algo == 0) ? oracle_fft(x, dst, n, dir) : oracle_dft(x, dst, n, dir);
        if (rc) bad |= 1;
        free(x);
    }
    return bad ? -1 : 0;
}

/* Number of OpenMP threads a parallel region would use (for reporting). */
int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
