// fft_device.cuh — register-level building blocks of the sm_100a FFT kernels.
//
// Method: per-record Cooley–Tukey FFT (§I; §III),
// realised as a Stockham autosort FFT (natural-order output, no bit-reversal
// pass).  Every thread holds P (<= 16) points of a
// length-L transform in registers; a pass applies radix-R butterflies with the
// Stockham twiddles and exchanges through shared memory.
//
// Stockham pass (forward, per butterfly j < L/R, current sub-length Ns):
//     a[q]  = x[j + q*L/R]                       q = 0..R-1
//     a[q] *= W_{Ns*R}^{(j mod Ns)*q}             W_M = exp(-2 pi i / M)
//     a     = DFT_R(a)
//     y[(j div Ns)*Ns*R + (j mod Ns) + q*Ns] = a[q]
// then Ns *= R.  Schedule: a first pass of radix 2^(log2 L mod 4) (if any)
// followed by radix-16 passes (tools/proto_indexing.py checks it against
// numpy.fft).  With P = 16 points per thread and T = L/16 threads per record,
// thread t always reads x[t + s*T] (s = 0..15) and the last pass leaves
// y[t + q*T] in v[q] — consecutive threads touch consecutive elements, so the
// global load and store are coalesced.
//
// Arithmetic: fp32 with the sm_100 packed f32x2 instructions (FADD2 / FMUL2 /
// FFMA2): a complex add is one FADD2 and a complex multiply FMUL2 + FFMA2.
// Round-to-nearest, no fast-math (reading c9).  Inverse transforms reuse the
// forward kernels via  ifft(X) = conj(fft(conj(X))) / N  (negation and the
// power-of-two scale are exact).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bfft {

// ---------------------------------------------------------------- complex ops
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// a * (-i) and a * (+i): register swaps, folded by ptxas into FADD2 operand modifiers.
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
__device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }
// a * w = w.x*(a.x, a.y) + w.y*(-a.y, a.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    float2 t = __fmul2_rn(a, make_float2(w.x, w.x));
    return __ffma2_rn(make_float2(-a.y, a.x), make_float2(w.y, w.y), t);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 scale_conj(float2 a, float s) {
    return __fmul2_rn(make_float2(a.x, -a.y), make_float2(s, s));
}

// cos / sin of 2*pi*m/16 for the radix-16 inner twiddles W_16^m = (c, -s).
#define BFFT_C1 0.92387953251128674f  // cos(pi/8)
#define BFFT_S1 0.38268343236508978f  // sin(pi/8)
#define BFFT_R2 0.70710678118654752f  // sqrt(1/2)

// a * W_16^m (forward sign), m compile-time in 0..15.
template <int M>
__device__ __forceinline__ float2 mul_w16(float2 a) {
    constexpr int m = M & 15;
    if constexpr (m == 0) return a;
    else if constexpr (m == 4) return mul_mi(a);
    else if constexpr (m == 8) return make_float2(-a.x, -a.y);
    else if constexpr (m == 12) return mul_pi(a);
    else {
        // W_16^m = cos(2 pi m/16) - i sin(2 pi m/16)
        constexpr float cs[4] = {1.0f, BFFT_C1, BFFT_R2, BFFT_S1};  // cos(k pi/8), k=0..3
        constexpr int q = m & 3;         // position inside the quadrant
        constexpr int quad = m >> 2;     // multiply by (-i)^quad afterwards
        constexpr float c = cs[q], s = cs[4 - q == 4 ? 0 : 4 - q];
        // W_16^q (q in 1..3) = (cos(q pi/8), -sin(q pi/8)); sin(q pi/8) = cos((4-q) pi/8)
        float2 w = make_float2(c, -s);
        float2 r = cmul(a, w);
        if constexpr (quad == 0) return r;
        else if constexpr (quad == 1) return mul_mi(r);
        else if constexpr (quad == 2) return make_float2(-r.x, -r.y);
        else return mul_pi(r);
    }
}

// ------------------------------------------------------------ DFT_R in place
// Forward DFT of R values in registers, natural-order output:
//   X[k] = sum_n x[n] W_R^{nk}.
template <int R> struct Dft;

template <> struct Dft<1> {
    template <class A> __device__ __forceinline__ static void run(A&) {}
};

template <> struct Dft<2> {
    __device__ __forceinline__ static void run(float2 (&a)[2]) {
        float2 t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    }
};

template <> struct Dft<4> {
    __device__ __forceinline__ static void run(float2 (&a)[4]) {
        float2 s0 = cadd(a[0], a[2]), d0 = csub(a[0], a[2]);
        float2 s1 = cadd(a[1], a[3]), d1 = csub(a[1], a[3]);
        a[0] = cadd(s0, s1);
        a[2] = csub(s0, s1);
        a[1] = cadd(d0, mul_mi(d1));   // d0 - i d1
        a[3] = csub(d0, mul_mi(d1));   // d0 + i d1
    }
};

template <> struct Dft<8> {
    __device__ __forceinline__ static void run(float2 (&a)[8]) {
        // X[k] = E[k] + W_8^k O[k], X[k+4] = E[k] - W_8^k O[k]
        float2 e[4] = {a[0], a[2], a[4], a[6]};
        float2 o[4] = {a[1], a[3], a[5], a[7]};
        Dft<4>::run(e);
        Dft<4>::run(o);
        o[1] = mul_w16<2>(o[1]);
        o[2] = mul_w16<4>(o[2]);
        o[3] = mul_w16<6>(o[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = cadd(e[k], o[k]);
            a[k + 4] = csub(e[k], o[k]);
        }
    }
};

template <> struct Dft<16> {
    __device__ __forceinline__ static void run(float2 (&a)[16]) {
        // n = 4 n1 + n2, k = k1 + 4 k2:
        //   X[k1 + 4k2] = sum_n2 W_4^{n2 k2} W_16^{n2 k1} sum_n1 x[4n1+n2] W_4^{n1 k1}
        float2 b[4][4];  // b[n2][k1]
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
            float2 t[4] = {a[n2], a[4 + n2], a[8 + n2], a[12 + n2]};
            Dft<4>::run(t);
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) b[n2][k1] = t[k1];
        }
        b[1][1] = mul_w16<1>(b[1][1]);
        b[1][2] = mul_w16<2>(b[1][2]);
        b[1][3] = mul_w16<3>(b[1][3]);
        b[2][1] = mul_w16<2>(b[2][1]);
        b[2][2] = mul_w16<4>(b[2][2]);
        b[2][3] = mul_w16<6>(b[2][3]);
        b[3][1] = mul_w16<3>(b[3][1]);
        b[3][2] = mul_w16<6>(b[3][2]);
        b[3][3] = mul_w16<9>(b[3][3]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            float2 t[4] = {b[0][k1], b[1][k1], b[2][k1], b[3][k1]};
            Dft<4>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) a[k1 + 4 * k2] = t[k2];
        }
    }
};

template <> struct Dft<32> {
    __device__ __forceinline__ static void run(float2 (&a)[32]) {
        // radix-2 DIT over two DFT_16: X[k] = E[k] + W_32^k O[k], X[k+16] = E[k] - W_32^k O[k]
        float2 e[16], o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            e[i] = a[2 * i];
            o[i] = a[2 * i + 1];
        }
        Dft<16>::run(e);
        Dft<16>::run(o);
        constexpr float c[8] = {1.0f,
                                0.98078528040323043f,  // cos(pi/16)
                                0.92387953251128674f,  // cos(2pi/16)
                                0.83146961230254524f,  // cos(3pi/16)
                                0.70710678118654752f,  // cos(4pi/16)
                                0.55557023301960218f,  // cos(5pi/16)
                                0.38268343236508978f,  // cos(6pi/16)
                                0.19509032201612826f}; // cos(7pi/16)
#pragma unroll
        for (int k = 1; k < 16; ++k) {
            if (k == 8) {
                o[k] = mul_mi(o[k]);
            } else {
                // W_32^k = cos(2 pi k/32) - i sin(2 pi k/32); for k in 9..15 use W_32^{k-8} * (-i)
                const int kk = k & 7;
                const float cr = c[kk], si = c[8 - kk == 8 ? 0 : 8 - kk];
                float2 t = cmul(o[k], make_float2(cr, -si));
                o[k] = k > 8 ? mul_mi(t) : t;
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a[k] = cadd(e[k], o[k]);
            a[k + 16] = csub(e[k], o[k]);
        }
    }
};

// ------------------------------------------------------------------ schedule
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// Schedule of a length-L transform with up to PP points per thread:
// P = min(PP, L) points per thread, T = L / P threads per transform, a first
// pass of radix 2^(log2 L mod log2 P) (if nonzero) and then radix-P passes.
template <int L, int PP = 16>
struct Sched {
    static constexpr int K = ilog2(L);
    static constexpr int P = L < PP ? L : PP;           // points per thread
    static constexpr int KP = ilog2(P);
    static constexpr int T = L / P;                     // threads per record
    static constexpr int R0 = L <= PP ? L : ((K % KP) ? (1 << (K % KP)) : P);
    static constexpr int NPASS = L <= PP ? 1 : ((K % KP) ? 1 + K / KP : K / KP);
    // radix of pass p and sub-length Ns before pass p
    __host__ __device__ static constexpr int radix(int p) { return p == 0 ? R0 : P; }
    __host__ __device__ static constexpr int ns(int p) {
        return p == 0 ? 1 : R0 * (p == 1 ? 1 : (1 << (KP * (p - 1))));
    }
    // offset (in complex entries) of pass p's twiddle table inside the
    // per-length table: passes p >= 1 each own (P-1)*Ns entries, [q-1][j mod Ns].
    __host__ __device__ static constexpr int tw_off(int p) {
        return p <= 1 ? 0 : tw_off(p - 1) + (P - 1) * ns(p - 1);
    }
    __host__ __device__ static constexpr int tw_entries() { return tw_off(NPASS); }
};

// --------------------------------------------------------- shared layouts
// Row layout (engine E1): records contiguous, element e of record b at
// lin = b*L + e stored at lin + lin/16 (one pad slot per 16 elements).  The
// stride-16 writes of a first pass and the unit-stride reads land on 16
// distinct bank pairs (tools/proto_indexing.py), and every address is a
// per-thread base plus a compile-time offset.
struct RowLayout {
    __device__ __forceinline__ static int at(int lin) { return lin + (lin >> 4); }
    __host__ __device__ static constexpr int size(int n) { return n + n / 16; }
};

// Column layout (engine E2): COLS interleaved transforms, element e of column
// c at e*COLS + c.  Every engine access has a half-warp on 16 consecutive
// columns of one element row, so it is conflict-free unswizzled — and every
// address is one per-thread base plus a compile-time offset (no per-element
// address registers).
template <int COLS>
struct ColLayout {
    __device__ __forceinline__ static int at(int e, int c) { return e * COLS + c; }
};
// Column layout for tiles narrower than 16 columns: one pad slot of COLS
// entries per R0 elements (R0 = the schedule's first radix).  The first
// Stockham pass writes element 16t + q-like runs whose plain addresses fall on
// the same bank pair for every t of a warp (2-4x the minimum wavefronts at
// COLS = 8 / 4, ncu: mio-bound at 2^21 / 2^22); the pad spreads them
// (tools/bank_model.py: every pass at the minimum).  COLS >= 16: plain.
template <int COLS, int R0>
struct PadColLayout {
    static constexpr int SH = ilog2(R0);
    __device__ __forceinline__ static int at(int e, int c) {
        if constexpr (COLS >= 16) return e * COLS + c;
        else return e * COLS + c + COLS * (e >> SH);
    }
    __host__ __device__ static constexpr int size(int L) { return COLS >= 16 ? COLS * L : COLS * (L + (L >> SH)); }
};
// Swizzled column layout for transposing accesses (a half-warp on 16
// consecutive elements e of one column): c ^ (e mod COLS) spreads them over
// 16 distinct bank pairs.
template <int COLS>
struct SwzColLayout {
    __device__ __forceinline__ static int at(int e, int c) { return e * COLS + (c ^ (e & (COLS - 1))); }
};

// ---------------------------------------------------------- generic passes
// One Stockham pass for a thread holding v[P] = x[t + s*T].  Results are
// handed to `put(index, value)`; the caller stores them (shared memory, or
// registers for the last pass).  TW(q, jj) returns W_{Ns*R}^{jj*q}.
template <int L, int PP, int PASS, bool DIRECT = false, class Put, class Tw>
__device__ __forceinline__ void stockham_pass(const float2 (&v)[Sched<L, PP>::P], int t, Put&& put, Tw&& tw) {
    using S = Sched<L, PP>;
    constexpr int P = S::P, T = S::T;
    constexpr int R = S::radix(PASS);
    constexpr int Ns = S::ns(PASS);
    constexpr int NB = P / R;  // butterflies per thread
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const int j = t + m * T;
        float2 a[R];
#pragma unroll
        for (int q = 0; q < R; ++q) a[q] = v[m + q * NB];
        if constexpr (Ns > 1) {
            const int jj = j & (Ns - 1);
            if constexpr (R <= 8 || DIRECT) {
#pragma unroll
                for (int q = 1; q < R; ++q) a[q] = cmul(a[q], tw(q, jj));
            } else {
                // radix 16/32: fetch W^{jj 2^i} (i < log2 R) and build W^{jj q} as
                // w[q] = w[q with its lowest set bit cleared] * W^{jj lowbit(q)}
                // (depth <= log2 R): log2 R live factors instead of R-1 loaded
                // twiddles (registers), log2 R loads instead of R-1 (L1/LSU).
                constexpr int LR = ilog2(R);
                float2 base[LR];
#pragma unroll
                for (int i = 0; i < LR; ++i) base[i] = tw(1 << i, jj);
                float2 w[R];
#pragma unroll
                for (int q = 1; q < R; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                    w[q] = (q & (q - 1)) ? cmul(w[q & (q - 1)], base[lb]) : base[lb];
                    a[q] = cmul(a[q], w[q]);
                }
            }
        }
        Dft<R>::run(a);
        const int base = (j / Ns) * Ns * R + (j & (Ns - 1));
#pragma unroll
        for (int q = 0; q < R; ++q) put(base + q * Ns, q, m, a[q]);
    }
}

}  // namespace bfft
