// fft_kernels.cuh — the sm_100a kernels of the per-record FFT.
//
//   k_rows      engine E1: single-pass Stockham, B whole records per CTA
//               (SURVEY.md §8(a) rows a2, a3, a5, a6).
//   k_fs_cols   four-step pass A: length-N1 FFTs down the columns of the
//               record viewed as [N1][N2], times W_N^{n2 k1} (row a4).
//   k_fs_rows   four-step pass B: length-N2 FFTs along the rows, stored
//               transposed to X[k1 + N1 k2] (row a4).
//   k_cluster   cluster variant: the four-step of row a4 inside one thread
//               block cluster, the transpose an all-to-all through DSMEM
//               (row a3'), so a record is read and written once.
//   k_copy      identity kernel (SPEC.md:275 test mode).
//
// The four-step split (north_star): with
//   n = N2*n1 + n2 and k = k1 + N1*k2,
//   X[k1 + N1 k2] = sum_n2 W_N2^{n2 k2} [ W_N^{n2 k1} sum_n1 x[N2 n1 + n2] W_N1^{n1 k1} ].
#pragma once

#include <type_traits>

#include "fft_device.cuh"

namespace bfft {

// ------------------------------------------------------------ small helpers
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

__device__ __forceinline__ float2 ld_stream(const float2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float2* p, float2 v) { __stcs(p, v); }

// W_N^m = exp(-2 pi i m / N) from fp64 sincospi, rounded once to fp32.
__device__ __forceinline__ float2 twiddle_exact(uint32_t m, uint32_t n) {
    double s, c;
    sincospi(-2.0 * (double)m / (double)n, &s, &c);
    return make_float2((float)c, (float)s);
}

// Per-pass Stockham twiddle fetch: table layout [q-1][j mod Ns] per pass.
template <int L, int PP = 16>
struct TableTw {
    const float2* __restrict__ base;  // this length's table
    template <int PASS>
    __device__ __forceinline__ float2 get(int q, int jj) const {
        using S = Sched<L, PP>;
        return __ldg(base + S::tw_off(PASS) + (q - 1) * S::ns(PASS) + jj);
    }
};

// Per-pass Stockham twiddles in constant memory, for the column engines whose
// butterfly index is warp-uniform (lanes = columns): the constant cache
// broadcasts and ptxas feeds the values straight into FFMA2 operands, so they
// cost no registers.  One table per (L, P) pair, filled once per device by the
// plan layer (bfft_upload_const_twiddles) with the same fp64-computed values.
__host__ __device__ constexpr int tw_entries_rt(int L, int P) {
    if (L <= P) return 0;
    const int K = ilog2(L), KP = ilog2(P);
    const int R0 = (K % KP) ? (1 << (K % KP)) : P;
    const int npass = (K % KP) ? 1 + K / KP : K / KP;
    int tot = 0;
    for (int p = 1; p < npass; ++p) tot += (P - 1) * R0 * (1 << (KP * (p - 1)));
    return tot;
}
// Lengths with a constant table: P = 16 for L in [32, 2048], P = 32 for L in [64, 512].
__host__ __device__ constexpr int ctw_max_l(int P) { return P == 16 ? 2048 : 1024; }
constexpr int CTW_MIN_L = 32;
// offset of the (L, P) table in c_tw; pairs ordered by P in {16, 32}, then L
__host__ __device__ constexpr int const_tw_base(int L, int P) {
    int base = 0;
    for (int p = 16; p <= 32; p *= 2)
        for (int l = CTW_MIN_L; l <= ctw_max_l(p); l *= 2) {
            if (l == L && p == P) return base;
            base += tw_entries_rt(l, p);
        }
    return L < 0 ? base : -1;  // L < 0: total size
}
constexpr int CTW_TOTAL = const_tw_base(-1, 0);
static_assert(CTW_TOTAL * 8 <= 60 * 1024, "constant twiddles exceed the constant bank");

__constant__ float2 c_tw[CTW_TOTAL];

template <int L, int PP = 16>
struct ConstTw {
    static constexpr int BASE = const_tw_base(L, PP);
    static_assert(L <= PP || BASE >= 0, "no constant twiddle table for this length");
    template <int PASS>
    __device__ __forceinline__ float2 get(int q, int jj) const {
        using S = Sched<L, PP>;
        return c_tw[BASE + S::tw_off(PASS) + (q - 1) * S::ns(PASS) + jj];
    }
};

// Run every pass of a length-L transform on v (v[s] = x[t + s*T] on entry,
// v[q] = X[t + q*T] on exit).  Intermediate passes exchange through `sm`
// addressed by addr(e) (the caller's layout).  Begins each exchange with a
// CTA barrier, so the buffer may still be read by other threads on entry.
struct CtaBarrier {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// Named barrier over the first `count` threads of the CTA (warp-specialised kernels).
struct NamedBarrier {
    int id, count;
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
    }
};

// Twiddle source traits: the radix-16/32 passes build their twiddles from
// log2 R table entries by a multiply tree (fewer loads and live registers).
template <class Tw> struct tw_direct { static constexpr bool value = false; };

template <int L, int PP = 16, class Addr, class Tw, class Bar = CtaBarrier>
__device__ __forceinline__ void fft_engine(float2 (&v)[Sched<L, PP>::P], int t, float2* sm,
                                           Addr&& addr, const Tw& tw, Bar bar = Bar{}) {
    using S = Sched<L, PP>;
    constexpr int P = S::P, T = S::T;
    static_for<0, S::NPASS>([&](auto pc) {
        constexpr int PASS = decltype(pc)::value;
        auto twf = [&](int q, int jj) { return tw.template get<PASS>(q, jj); };
        if constexpr (PASS == S::NPASS - 1) {
            float2 o[P];
            stockham_pass<L, PP, PASS, tw_direct<Tw>::value>(v, t, [&](int, int q, int, float2 val) { o[q] = val; }, twf);
#pragma unroll
            for (int q = 0; q < P; ++q) v[q] = o[q];
        } else {
            bar();
            stockham_pass<L, PP, PASS, tw_direct<Tw>::value>(v, t, [&](int idx, int, int, float2 val) { sm[addr(idx)] = val; }, twf);
            bar();
#pragma unroll
            for (int s = 0; s < P; ++s) v[s] = sm[addr(t + s * T)];
        }
    });
}

// w[q] = W_N^{m0 + q*dm} for q = 0..15 (mod N), as b * s1^a * s2^b * s4^c * s8^d
// with every factor from fp64 sincospi: at most four fp32 products per value.
__device__ __forceinline__ void twiddle_row16(uint32_t m0, uint32_t dm, uint32_t nmask, uint32_t n,
                                              float2 (&w)[16]) {
    const float2 b = twiddle_exact(m0 & nmask, n);
    const float2 s1 = twiddle_exact(dm & nmask, n);
    const float2 s2 = twiddle_exact((2u * dm) & nmask, n);
    const float2 s4 = twiddle_exact((4u * dm) & nmask, n);
    const float2 s8 = twiddle_exact((8u * dm) & nmask, n);
    w[0] = b;
    w[1] = cmul(b, s1);
    w[2] = cmul(b, s2);
    w[3] = cmul(w[1], s2);
#pragma unroll
    for (int q = 4; q < 8; ++q) w[q] = cmul(w[q - 4], s4);
#pragma unroll
    for (int q = 8; q < 16; ++q) w[q] = cmul(w[q - 8], s8);
}

// ======================================================================
// E1: single-pass, B records per CTA, one record = T threads x P points.
// ======================================================================
template <int L, int B, int PP = 16>
struct RowsMinBlocks {  // CTAs per SM the register budget is sized for
    static constexpr int THREADS = B * Sched<L, PP>::T;
    static constexpr int V = PP == 32 ? (THREADS <= 256 ? 2 : 1) : (THREADS <= 256 ? 4 : 1);
};

// W_64^j = exp(-2 pi i j / 64), j = 0..63, fp64-computed and rounded to fp32
// (cos, -sin).  The real-record split / merge factors W_n^k, n = 2L, k = t + q T
// as W_n^t * W_{2P}^q (n / T = 2P): the second factor, with q unrolled, is a
// constant-bank operand (c_rw64[q * 32 / P]).
__constant__ float2 c_rw64[64] = {
    {1.0f, -0.0f}, {0.99518472f, -0.0980171412f}, {0.980785251f, -0.195090324f}, {0.956940353f, -0.290284663f},
    {0.923879504f, -0.382683426f}, {0.881921291f, -0.471396744f}, {0.831469595f, -0.555570245f}, {0.773010433f, -0.634393275f},
    {0.707106769f, -0.707106769f}, {0.634393275f, -0.773010433f}, {0.555570245f, -0.831469595f}, {0.471396744f, -0.881921291f},
    {0.382683426f, -0.923879504f}, {0.290284663f, -0.956940353f}, {0.195090324f, -0.980785251f}, {0.0980171412f, -0.99518472f},
    {0.0f, -1.0f}, {-0.0980171412f, -0.99518472f}, {-0.195090324f, -0.980785251f}, {-0.290284663f, -0.956940353f},
    {-0.382683426f, -0.923879504f}, {-0.471396744f, -0.881921291f}, {-0.555570245f, -0.831469595f}, {-0.634393275f, -0.773010433f},
    {-0.707106769f, -0.707106769f}, {-0.773010433f, -0.634393275f}, {-0.831469595f, -0.555570245f}, {-0.881921291f, -0.471396744f},
    {-0.923879504f, -0.382683426f}, {-0.956940353f, -0.290284663f}, {-0.980785251f, -0.195090324f}, {-0.99518472f, -0.0980171412f},
    {-1.0f, 0.0f}, {-0.99518472f, 0.0980171412f}, {-0.980785251f, 0.195090324f}, {-0.956940353f, 0.290284663f},
    {-0.923879504f, 0.382683426f}, {-0.881921291f, 0.471396744f}, {-0.831469595f, 0.555570245f}, {-0.773010433f, 0.634393275f},
    {-0.707106769f, 0.707106769f}, {-0.634393275f, 0.773010433f}, {-0.555570245f, 0.831469595f}, {-0.471396744f, 0.881921291f},
    {-0.382683426f, 0.923879504f}, {-0.290284663f, 0.956940353f}, {-0.195090324f, 0.980785251f}, {-0.0980171412f, 0.99518472f},
    {0.0f, 1.0f}, {0.0980171412f, 0.99518472f}, {0.195090324f, 0.980785251f}, {0.290284663f, 0.956940353f},
    {0.382683426f, 0.923879504f}, {0.471396744f, 0.881921291f}, {0.555570245f, 0.831469595f}, {0.634393275f, 0.773010433f},
    {0.707106769f, 0.707106769f}, {0.773010433f, 0.634393275f}, {0.831469595f, 0.555570245f}, {0.881921291f, 0.471396744f},
    {0.923879504f, 0.382683426f}, {0.956940353f, 0.290284663f}, {0.980785251f, 0.195090324f}, {0.99518472f, 0.0980171412f},
};

// W_n^k of a real-record plan (n = 2L real points), fp64-computed tables:
// W_n^k = hi[k >> lb] * lo[k & (2^lb - 1)] (csrc/real.cu's factors).
struct RealTw {
    const float2* hi;
    const float2* lo;
    int lb;
    const float2* src = nullptr;   // k_pipe2 RS = 2: the packed half spectra (partner reads)
    __device__ __forceinline__ float2 operator()(int k) const {
        return cmul(__ldg(hi + (k >> lb)), __ldg(lo + (k & ((1 << lb) - 1))));
    }
};

// REAL = 0: complex records.  REAL = 1: real records, forward (R2C): the
// record is the L-point complex signal x[2m] + i x[2m+1]; after its transform
// Z the split X[k] = E + W_n^k O (E = (Z[k] + conj Z[L-k])/2, O = (Z[k] -
// conj Z[L-k])/(2i)) is done in the same kernel and the packed half spectrum
// (out[0] = (X[0], X[L])) is stored.  REAL = 2: inverse (C2R): the merge
// Z[k] = E + i O (E = (X[k] + conj X[L-k])/2, O = (X[k] - conj X[L-k])
// conj(W_n^k)/2) happens on load, then the inverse transform.  Partners come
// by warp shuffle when a record's T threads share a warp (T <= 32), else
// through shared memory.  csrc/real.cu holds the same arithmetic as separate
// kernels for longer records.
template <int L, int B, bool INV, int PP = 16, int MINB = 0, int REAL = 0>   // MINB > 0 overrides the register budget
__global__ void __launch_bounds__(B * Sched<L, PP>::T, MINB > 0 ? MINB : RowsMinBlocks<L, B, PP>::V)
k_rows(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec,
       const float2* __restrict__ tw, float scale, int64_t istride, const float* __restrict__ window, RealTw rt) {
    // istride: elements between consecutive input records (L for records; the
    // hop for STFT frames); window: optional real
    // per-sample weights w[0..L) applied on load (STFT), nullptr = none
    static_assert(REAL == 0 || INV == (REAL == 2), "R2C is forward, C2R inverse");
    using S = Sched<L, PP>;
    constexpr int P = S::P, T = S::T;
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x;
    const int b = tid / T, t = tid - (tid / T) * T;
    const TableTw<L, PP> tab{tw};
    auto addr = [&](int e) { return RowLayout::at(b * L + e); };
    // real records: a thread's elements are k = t + q T, whose partners L - k are
    // (T - t) + (P - 1 - q) T — element P-1-q of thread T - t — or, for t = 0,
    // element P - q of the thread itself.  With T <= 32 a record's threads share a
    // warp and the partner comes by shuffle.  W_n^k = W_n^t W_{2P}^q (n = 2 P T).
    constexpr bool SHFL = REAL != 0 && T <= 32;
    const int src_lane = ((threadIdx.x & 31) & ~(T - 1)) | ((T - t) & (T - 1));
    float2 wt = REAL != 0 ? rt(t) : make_float2(1.f, 0.f);
    auto wk = [&](int q) { return cmul(wt, c_rw64[q * (32 / P)]); };   // W_n^{t + q T}
    auto partner = [&](const float2 (&a)[P], int q) {
        float2 c;
        c.x = __shfl_sync(0xffffffffu, a[P - 1 - q].x, src_lane);
        c.y = __shfl_sync(0xffffffffu, a[P - 1 - q].y, src_lane);
        return t == 0 ? a[(P - q) & (P - 1)] : c;
    };
    for (int64_t g = blockIdx.x; g * B < nrec; g += gridDim.x) {
        const int64_t r = g * B + b;
        const bool ok = r < nrec;
        const float2* src = in + r * istride + t;
        float2 v[P];
        // keep the P products W_n^t W_{2P}^q from being hoisted out of the loop (2P live registers)
        if constexpr (REAL != 0) asm volatile("" : "+f"(wt.x), "+f"(wt.y));
        if constexpr (REAL == 2 && SHFL) {
            // C2R merge on load, partners by shuffle: Z[k] = E + i O,
            // E = (X[k] + conj X[L-k]) / 2, O = (X[k] - conj X[L-k]) conj(W_n^k) / 2
            float2 xin[P];
#pragma unroll
            for (int s = 0; s < P; ++s) xin[s] = ok ? ld_stream(src + s * T) : make_float2(0.f, 0.f);
#pragma unroll
            for (int s = 0; s < P; ++s) {
                const float2 x = xin[s], y = partner(xin, s);
                float2 z;
                if (s == 0 && t == 0) {
                    z = make_float2(0.5f * (x.x + x.y), 0.5f * (x.x - x.y));      // (E[0], O[0])
                } else {
                    const float2 e = __fmul2_rn(cadd(x, conjf2(y)), make_float2(0.5f, 0.5f));
                    const float2 o = cmul(__fmul2_rn(csub(x, conjf2(y)), make_float2(0.5f, 0.5f)), conjf2(wk(s)));
                    z = cadd(e, mul_pi(o));
                }
                v[s] = conjf2(z);   // INV
            }
        } else if constexpr (REAL == 2) {
            // C2R merge on load, partners through shared memory (the record's
            // threads span several warps)
            float2 xin[P];
#pragma unroll
            for (int s = 0; s < P; ++s) xin[s] = ok ? ld_stream(src + s * T) : make_float2(0.f, 0.f);
            __syncthreads();   // the previous record's last exchange has been read
#pragma unroll
            for (int s = 0; s < P; ++s) sm[addr(t + s * T)] = xin[s];
            __syncthreads();
#pragma unroll
            for (int s = 0; s < P; ++s) {
                const int k = t + s * T;
                const float2 x = xin[s];
                float2 z;
                if (k == 0) {
                    z = make_float2(0.5f * (x.x + x.y), 0.5f * (x.x - x.y));      // (E[0], O[0])
                } else {
                    const float2 y = sm[addr(L - k)];
                    const float2 e = __fmul2_rn(cadd(x, conjf2(y)), make_float2(0.5f, 0.5f));
                    const float2 o = cmul(__fmul2_rn(csub(x, conjf2(y)), make_float2(0.5f, 0.5f)), conjf2(wk(s)));
                    z = cadd(e, mul_pi(o));
                }
                v[s] = conjf2(z);   // INV
            }
        } else {
#pragma unroll
        for (int s = 0; s < P; ++s) {
            float2 x = ok ? ld_stream(src + s * T) : make_float2(0.f, 0.f);
            if (window) {
                const float w = __ldg(window + t + s * T);
                x = make_float2(x.x * w, x.y * w);
            }
            v[s] = INV ? conjf2(x) : x;
        }
        }
        fft_engine<L, PP>(v, t, sm, addr, tab);
        if constexpr (REAL == 1 && SHFL) {
            // R2C split, partners by shuffle: X[k] = E + W_n^k O (packed X[0] = (X[0], X[L]))
            float2* dst = out + r * (int64_t)L + t;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const float2 a = v[q], c = partner(v, q);
                float2 x;
                if (q == 0 && t == 0) {
                    x = make_float2(a.x + a.y, a.x - a.y);
                } else {
                    const float2 e = __fmul2_rn(cadd(a, conjf2(c)), make_float2(0.5f, 0.5f));
                    const float2 o = mul_mi(__fmul2_rn(csub(a, conjf2(c)), make_float2(0.5f, 0.5f)));
                    x = cadd(e, cmul(o, wk(q)));
                }
                if (ok) st_stream(dst + q * T, x);
            }
        } else if constexpr (REAL == 1) {
            __syncthreads();   // every exchange of the engine has been read
#pragma unroll
            for (int q = 0; q < P; ++q) sm[addr(t + q * T)] = v[q];
            __syncthreads();
            if (ok) {
                float2* dst = out + r * (int64_t)L + t;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int k = t + q * T;
                    const float2 a = v[q];
                    float2 x;
                    if (k == 0) {
                        x = make_float2(a.x + a.y, a.x - a.y);                     // (X[0], X[L])
                    } else {
                        const float2 c = sm[addr(L - k)];
                        const float2 e = __fmul2_rn(cadd(a, conjf2(c)), make_float2(0.5f, 0.5f));
                        const float2 o = mul_mi(__fmul2_rn(csub(a, conjf2(c)), make_float2(0.5f, 0.5f)));
                        x = cadd(e, cmul(o, wk(q)));                               // X[k] = E + W^k O
                    }
                    st_stream(dst + q * T, x);
                }
            }
        } else if (ok) {
            float2* dst = out + r * (int64_t)L + t;
#pragma unroll
            for (int q = 0; q < P; ++q) st_stream(dst + q * T, INV ? scale_conj(v[q], scale) : v[q]);
        }
    }
}

// ======================================================================
// Four-step pass A: for a tile of COLS adjacent columns n2 of record r,
// Y[k1][n2] = W_N^{n2 k1} * FFT_N1 over n1 of x[N2 n1 + n2].
// ======================================================================
template <int N1, int COLS, bool INV>
__global__ void __launch_bounds__(COLS * Sched<N1>::T)
k_fs_cols(const float2* __restrict__ in, float2* __restrict__ y, int64_t nrec, int log2n2,
          const float2* __restrict__ tw) {
    using S = Sched<N1>;
    constexpr int P = S::P, T = S::T;
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x;
    const int col = tid % COLS, t = tid / COLS;
    const int n2 = 1 << log2n2;
    const int tiles = n2 / COLS;
    const uint32_t n = (uint32_t)N1 << log2n2, nmask = n - 1;
    const ConstTw<N1> tab{};
    auto addr = [&](int e) { return ColLayout<COLS>::at(e, col); };
    for (int64_t g = blockIdx.x; g < nrec * tiles; g += gridDim.x) {
        const int64_t r = g / tiles;
        const int c = (int)(g - r * tiles) * COLS + col;     // this thread's n2
        const float2* src = in + r * (int64_t)n + c + (int64_t)t * n2;
        float2 v[P];
#pragma unroll
        for (int s = 0; s < P; ++s) {
            float2 x = ld_stream(src + (int64_t)s * T * n2);
            v[s] = INV ? conjf2(x) : x;
        }
        fft_engine<N1>(v, t, sm, addr, tab);
        float2 w[16];
        // k1 = t + q*T  ->  W_N^{n2 (t + q T)}
        twiddle_row16((uint32_t)c * (uint32_t)t, (uint32_t)c * (uint32_t)T, nmask, n, w);
        float2* dst = y + r * (int64_t)n + c + (int64_t)t * n2;
#pragma unroll
        for (int q = 0; q < P; ++q) dst[(int64_t)q * T * n2] = cmul(v[q], w[q]);
    }
}

// ======================================================================
// Four-step pass B: for ROWS adjacent rows k1 of Y (record r), FFT_N2 along
// n2 and store X[k1 + N1 k2].  The tile is loaded coalesced along n2 and
// transposed into the column layout through shared memory.
// ======================================================================
template <int N2, int ROWS, bool INV>
__global__ void __launch_bounds__(ROWS * Sched<N2>::T)
k_fs_rows(const float2* __restrict__ y, float2* __restrict__ out, int64_t nrec, int log2n1,
          const float2* __restrict__ tw, float scale) {
    using S = Sched<N2>;
    constexpr int P = S::P, T = S::T;
    constexpr int NT = ROWS * T;
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x;
    const int col = tid % ROWS, t = tid / ROWS;
    const int n1 = 1 << log2n1;
    const int tiles = n1 / ROWS;
    const int64_t n = (int64_t)n1 * N2;
    const ConstTw<N2> tab{};
    auto addr = [&](int e) { return ColLayout<ROWS>::at(e, col); };
    for (int64_t g = blockIdx.x; g < nrec * tiles; g += gridDim.x) {
        const int64_t r = g / tiles;
        const int k0 = (int)(g - r * tiles) * ROWS;
        const float2* src = y + r * n + (int64_t)k0 * N2;
        __syncthreads();  // previous tile fully consumed
#pragma unroll
        for (int u = 0; u < P; ++u) {
            const int i = tid + u * NT;          // linear index in the ROWS x N2 tile
            const int row = i / N2, e = i - (i / N2) * N2;
            sm[SwzColLayout<ROWS>::at(e, row)] = ld_stream(src + i);
        }
        __syncthreads();
        float2 v[P];
#pragma unroll
        for (int s = 0; s < P; ++s) v[s] = sm[SwzColLayout<ROWS>::at(t + s * T, col)];
        fft_engine<N2>(v, t, sm, addr, tab);
        float2* dst = out + r * n + k0 + col + (int64_t)t * n1;
#pragma unroll
        for (int q = 0; q < P; ++q)
            st_stream(dst + (int64_t)q * T * n1, INV ? scale_conj(v[q], scale) : v[q]);
    }
}


// ======================================================================
// STFT framing: frame f of a signal,
// out[f][j] = w[j] * in[f * hop + j] (w = nullptr: rectangular), for frames
// too long for the single-pass kernel (which frames and windows on load);
// the batched transform then runs in place on `out`.
// ======================================================================
static __global__ void k_frames(const float2* __restrict__ in, float2* __restrict__ out, int64_t frames, int64_t n,
                                int64_t hop, const float* __restrict__ window) {
    const int64_t total = frames * n;
    const int lg = __ffsll((unsigned long long)n) - 1;   // n is a power of two: shift, not a 64-bit division
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i >> lg, j = i & (n - 1);
        float2 x = __ldcs(in + f * hop + j);
        if (window) {
            const float w = __ldg(window + j);
            x = make_float2(x.x * w, x.y * w);
        }
        __stcs(out + i, x);
    }
}

// ======================================================================
// Identity kernel: out = in, bit-exact, 16-byte vectors.
// ======================================================================
static __global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, int64_t n16) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x)
        __stcs(out + i, __ldcs(in + i));
}

}  // namespace bfft
