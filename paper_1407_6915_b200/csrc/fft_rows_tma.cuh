// fft_rows_tma.cuh — engine E1 (single pass) for the
// longest records that still fit one CTA, with the record loads taken off the
// compute warps' critical path: whole records are streamed into an NSTAGE-deep
// ring of shared-memory stages with bulk copies (TMA), and NGRP compute groups
// of T = L / PP threads each FFT one staged record in place (the engine's
// exchanges reuse the stage) and store the result straight from registers.
//
// Why: k_rows holds a record's loads in registers, so at 2^13 (64 KiB records,
// 96 registers x 256 threads) only two records per SM are in flight and HBM
// idles while both compute (71 % of the roofline, profiles/r01_rows_2p13_minb.txt).
// Here the next record is already in shared memory when a group finishes.
//
// Records start istride elements apart (L; the hop for STFT frames — even, so
// the bulk copies stay 16-byte aligned), optionally weighted by window[0..L) on
// read.  Records are dealt statically: CTA c takes records c, c + grid, ...; task k
// of a CTA is its k-th record, staged in stage k mod NSTAGE and computed by
// group k mod NGRP.  There is no producer warp (17 warps would cap registers
// at 96 per thread: 5 warps on one SM sub-partition): thread 0 stages the first
// NSTAGE records, and the group that has read stage s for the last time
// (group barrier) refills it with task k + NSTAGE; full[s] completes when a
// copy lands.
#pragma once

#include "fft_pipe.cuh"

namespace bfft {

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Exchange layout of the staged kernels: RowLayout (one pad entry per 16)
// plus, for engines whose second pass writes groups of Ns < 16 consecutive
// outputs G = Ns * R entries apart (2^13 with radix-32: Ns = 8, G = 256), 8 pad
// entries per G, which puts neighbouring groups on opposite bank halves
// (k_rows_tma at 2^13 spent 37 % of its store wavefronts on conflicts,
// profiles/r02_rows_tma_2p13_ncu.md; with the extra pad 82.7 vs 80.6 % on one
// box, profiles/r02_rows_tma.txt).
template <int L, int PP>
struct TmaLayout {
    using S = Sched<L, PP>;
    static constexpr int NS1 = S::NPASS > 2 ? S::ns(1) : 16;    // outputs per group in pass 1
    static constexpr int G = NS1 < 16 ? NS1 * S::radix(1) : 0;  // group spacing (0: no extra pad)
    __device__ __forceinline__ static int at(int e) {
        if constexpr (G > 0) return e + (e >> 4) + 8 * (e / G);
        else return RowLayout::at(e);
    }
    __host__ __device__ static constexpr int size(int n) { return RowLayout::size(n) + (G > 0 ? 8 * (n / G) : 0); }
};

template <int L, int PP, int NGRP, int NSTAGE>
struct RowsTmaCfg {
    using S = Sched<L, PP>;
    static constexpr int T = S::T;                                     // threads per record (one group)
    static constexpr int NT = NGRP * T;
    static constexpr int STAGE = (TmaLayout<L, PP>::size(L) + 15) / 16 * 16;  // entries per stage (padded exchanges)
    static constexpr int CHUNKS = L * 8 >= 4 * 16384 ? 4 : 1;          // bulk copies per record
    static constexpr size_t SMEM = sizeof(float2) * (size_t)STAGE * NSTAGE + 8 * NSTAGE;
    static constexpr int MINB = SMEM * 2 <= 227 * 1024 ? 2 : 1;
    static_assert(T % 32 == 0 && NGRP <= NSTAGE && (L / CHUNKS) % 2 == 0 && CHUNKS <= T, "stage geometry");
};

// REAL (as k_rows): 0 complex records; 1 real records forward (R2C split after
// the transform, partners exchanged through the stage); 2 real records inverse
// (C2R merge before it: the record is staged in natural order, so the partner
// X[L-k] is read straight from the stage).
template <int L, bool INV, int PP, int NGRP, int NSTAGE, int REAL = 0>
__global__ void __launch_bounds__(RowsTmaCfg<L, PP, NGRP, NSTAGE>::NT, RowsTmaCfg<L, PP, NGRP, NSTAGE>::MINB)
k_rows_tma(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec, const float2* __restrict__ tw,
           float scale, RealTw rt, int64_t istride, const float* __restrict__ window) {
    static_assert(REAL == 0 || INV == (REAL == 2), "R2C is forward, C2R inverse");
    using CF = RowsTmaCfg<L, PP, NGRP, NSTAGE>;
    constexpr int T = CF::T, P = CF::S::P, STAGE = CF::STAGE;
    extern __shared__ __align__(128) float2 sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)STAGE * NSTAGE);   // full[NSTAGE]
    const uint32_t full0 = smem_addr(bars);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t G = gridDim.x;
    const uint64_t pol = policy_evict_first();
    // stage task k (record blockIdx.x + k G) into stage k mod NSTAGE: CHUNKS bulk
    // copies issued by lanes 0..CHUNKS-1 of the calling warp
    auto stage_task = [&](uint32_t k) {
        const int64_t r = blockIdx.x + (int64_t)k * G;
        if (r >= nrec) return;
        const uint32_t s = k % NSTAGE;
        if (lane == 0) mbar_expect_tx(full0 + 8 * s, (uint32_t)(L * sizeof(float2)));
        __syncwarp();
        constexpr int CH = L / CF::CHUNKS;
        if (lane < CF::CHUNKS)
            bulk_g2s_hint(smem_addr(sm + (size_t)s * STAGE + lane * CH), in + r * istride + lane * CH, CH * sizeof(float2),
                          full0 + 8 * s, pol);
    };
    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) mbar_init(full0 + 8 * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0)
        for (uint32_t k = 0; k < NSTAGE; ++k) stage_task(k);
    {
        // ============================================== compute groups
        const int grp = warp / (T / 32);
        const int t = tid - grp * T;
        const NamedBarrier bar{1 + grp, T};
        const TableTw<L, PP> tab{tw};
        // real records: W_n^k = W_n^t W_{2P}^q for k = t + q T (n = 2 P T; fft_kernels.cuh)
        float2 wt = REAL != 0 ? rt(t) : make_float2(1.f, 0.f);
        auto wk = [&](int q) { return cmul(wt, c_rw64[q * (32 / P)]); };
        uint32_t k = grp;
        for (int64_t r = blockIdx.x + (int64_t)grp * G; r < nrec; r += NGRP * G, k += NGRP) {
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            float2* stage = sm + (size_t)s * STAGE;
            if constexpr (REAL != 0) asm volatile("" : "+f"(wt.x), "+f"(wt.y));   // not hoisted: 2P registers
            mbar_wait(full0 + 8 * s, u & 1);
            float2 v[P];
#pragma unroll
            for (int j = 0; j < P; ++j) {
                float2 x = stage[t + j * T];
                if (window) {   // STFT frames (istride = the hop): weights applied on read
                    const float w = __ldg(window + t + j * T);
                    x = make_float2(x.x * w, x.y * w);
                }
                if constexpr (REAL == 2) {
                    // Z[k] = E + i O, E = (X[k] + conj X[L-k]) / 2, O = (X[k] - conj X[L-k]) conj(W_n^k) / 2
                    const int kk = t + j * T;
                    float2 z;
                    if (kk == 0) {
                        z = make_float2(0.5f * (x.x + x.y), 0.5f * (x.x - x.y));
                    } else {
                        const float2 y = stage[L - kk];
                        const float2 e = __fmul2_rn(cadd(x, conjf2(y)), make_float2(0.5f, 0.5f));
                        const float2 o = cmul(__fmul2_rn(csub(x, conjf2(y)), make_float2(0.5f, 0.5f)), conjf2(wk(j)));
                        z = cadd(e, mul_pi(o));
                    }
                    v[j] = conjf2(z);
                } else {
                    v[j] = INV ? conjf2(x) : x;
                }
            }
            fft_engine<L, PP>(v, t, stage, [](int e) { return TmaLayout<L, PP>::at(e); }, tab, bar);
            float2* dst = out + r * L + t;
            if constexpr (REAL == 1) {
                // X[k] = E + W_n^k O, E = (Z[k] + conj Z[L-k]) / 2, O = (Z[k] - conj Z[L-k]) / (2i); out[0] = (X[0], X[L])
                bar();   // the engine's last exchange has been read by the whole group
#pragma unroll
                for (int q = 0; q < P; ++q) stage[RowLayout::at(t + q * T)] = v[q];
                bar();
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const float2 a = v[q], c = stage[RowLayout::at((L - (t + q * T)) & (L - 1))];
                    float2 x;
                    if (q == 0 && t == 0) {
                        x = make_float2(a.x + a.y, a.x - a.y);
                    } else {
                        const float2 e = __fmul2_rn(cadd(a, conjf2(c)), make_float2(0.5f, 0.5f));
                        const float2 o = mul_mi(__fmul2_rn(csub(a, conjf2(c)), make_float2(0.5f, 0.5f)));
                        x = cadd(e, cmul(o, wk(q)));
                    }
                    st_stream(dst + q * T, x);
                }
                fence_proxy_async_smem();   // this thread's last generic access of the stage
                bar();
                if (t < 32) stage_task(k + NSTAGE);   // the group's first warp refills it
            } else {
                fence_proxy_async_smem();   // this thread's last generic access of the stage
                bar();
                if (t < 32) stage_task(k + NSTAGE);   // the group's first warp refills it
#pragma unroll
                for (int q = 0; q < P; ++q) st_stream(dst + q * T, INV ? scale_conj(v[q], scale) : v[q]);
            }
        }
    }
}

}  // namespace bfft

namespace bfft {

// k_rows_tma2: the same idea for records too long for two stages (2^14: 128 KiB
// plus exchange padding).  The record's exchange buffer X holds its last
// L - YL points in place; the first YL points are staged in a separate buffer
// Y.  Y is refilled with the next record's head as soon as the transform's
// inputs are in registers; X's tail is refilled once the engine's last
// exchange has been read — only that tail's arrival is exposed.  One group of
// T = L / PP threads per CTA.
template <int L, int PP, int YL>
struct RowsTma2Cfg {
    using S = Sched<L, PP>;
    static constexpr int T = S::T, NT = T;
    static constexpr int XS = (RowLayout::size(L) + 15) / 16 * 16;
    static constexpr size_t SMEM = sizeof(float2) * (size_t)(XS + YL) + 16;
    static_assert(YL % T == 0 && YL % 8 == 0 && (L - YL) % 8 == 0, "head / tail split");
};

// REAL as k_rows_tma (1 R2C split through X after the transform, 2 C2R merge
// on load with the partner read from Y or X).
template <int L, bool INV, int PP, int YL, int REAL = 0>
__global__ void __launch_bounds__(RowsTma2Cfg<L, PP, YL>::NT, 1)
k_rows_tma2(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec, const float2* __restrict__ tw,
            float scale, RealTw rt, int64_t istride, const float* __restrict__ window) {
    static_assert(REAL == 0 || INV == (REAL == 2), "R2C is forward, C2R inverse");
    using CF = RowsTma2Cfg<L, PP, YL>;
    constexpr int T = CF::T, P = CF::S::P, XS = CF::XS, JY = YL / T;
    extern __shared__ __align__(128) float2 sm[];
    float2* X = sm;
    float2* Y = sm + XS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Y + YL);   // fullY, fullX
    const uint32_t fullY = smem_addr(bars), fullX = smem_addr(bars + 1);
    const int t = threadIdx.x, lane = t & 31;
    const int64_t G = gridDim.x;
    const uint64_t pol = policy_evict_first();
    // bulk copy of [lo, hi) of record r into dst, lanes 0..3 of warp 0
    auto load = [&](float2* dst, int64_t r, int lo, int hi, uint32_t bar) {
        if (lane == 0) mbar_expect_tx(bar, (uint32_t)((hi - lo) * sizeof(float2)));
        __syncwarp();
        const int ch = (hi - lo) / 4;
        if (lane < 4)
            bulk_g2s_hint(smem_addr(dst + lane * ch), in + r * istride + lo + lane * ch, ch * sizeof(float2), bar, pol);
    };
    if (t == 0) {
        mbar_init(fullY, 1);
        mbar_init(fullX, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t < 32 && (int64_t)blockIdx.x < nrec) {
        load(Y, blockIdx.x, 0, YL, fullY);
        load(X + YL, blockIdx.x, YL, L, fullX);
    }
    const CtaBarrier bar{};
    const TableTw<L, PP> tab{tw};
    // real records: W_n^k = W_n^t W_{2P}^q for k = t + q T (n = 2 P T; fft_kernels.cuh)
    float2 wt = REAL != 0 ? rt(t) : make_float2(1.f, 0.f);
    auto wk = [&](int q) { return cmul(wt, c_rw64[q * (32 / P)]); };
    uint32_t k = 0;
    for (int64_t r = blockIdx.x; r < nrec; r += G, ++k) {
        const bool more = r + G < nrec;
        if constexpr (REAL != 0) asm volatile("" : "+f"(wt.x), "+f"(wt.y));   // not hoisted: 2P registers
        mbar_wait(fullY, k & 1);
        mbar_wait(fullX, k & 1);
        float2 v[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
            float2 x = j < JY ? Y[t + j * T] : X[t + j * T];
            if (window) {   // STFT frames (istride = the hop): weights applied on read
                const float w = __ldg(window + t + j * T);
                x = make_float2(x.x * w, x.y * w);
            }
            if constexpr (REAL == 2) {
                // Z[k] = E + i O, E = (X[k] + conj X[L-k]) / 2, O = (X[k] - conj X[L-k]) conj(W_n^k) / 2
                const int kk = t + j * T;
                float2 z;
                if (kk == 0) {
                    z = make_float2(0.5f * (x.x + x.y), 0.5f * (x.x - x.y));
                } else {
                    const int pk = L - kk;
                    const float2 y = pk < YL ? Y[pk] : X[pk];
                    const float2 e = __fmul2_rn(cadd(x, conjf2(y)), make_float2(0.5f, 0.5f));
                    const float2 o = cmul(__fmul2_rn(csub(x, conjf2(y)), make_float2(0.5f, 0.5f)), conjf2(wk(j)));
                    z = cadd(e, mul_pi(o));
                }
                v[j] = conjf2(z);
            } else {
                v[j] = INV ? conjf2(x) : x;
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (t < 32 && more) load(Y, r + G, 0, YL, fullY);   // the next head, behind this transform
        fft_engine<L, PP>(v, t, X, [](int e) { return RowLayout::at(e); }, tab, bar);
        float2* dst = out + r * L + t;
        if constexpr (REAL == 1) {
            // X[k] = E + W_n^k O, E = (Z[k] + conj Z[L-k]) / 2, O = (Z[k] - conj Z[L-k]) / (2i); out[0] = (X[0], X[L]).
            // The partner of k = t + qT is element P-1-q of thread T-t (P-q of thread 0 itself): exchanged
            // in two halves through X[0, L/2), so X's tail can be refilled before the split.
            static_assert(L / 2 <= YL, "the split exchange stays below the tail");
            fence_proxy_async_smem();
            __syncthreads();   // the engine's last exchange has been read
            if (t < 32 && more) load(X + YL, r + G, YL, L, fullX);
            auto split = [&](int q, float2 c) {
                const float2 a = v[q];
                float2 x;
                if (q == 0 && t == 0) {
                    x = make_float2(a.x + a.y, a.x - a.y);
                } else {
                    if (t == 0) c = v[(P - q) & (P - 1)];
                    const float2 e = __fmul2_rn(cadd(a, conjf2(c)), make_float2(0.5f, 0.5f));
                    const float2 o = mul_mi(__fmul2_rn(csub(a, conjf2(c)), make_float2(0.5f, 0.5f)));
                    x = cadd(e, cmul(o, wk(q)));
                }
                st_stream(dst + q * T, x);
            };
#pragma unroll
            for (int q = P / 2; q < P; ++q) X[t + (q - P / 2) * T] = v[q];   // k in [L/2, L)
            __syncthreads();
#pragma unroll
            for (int q = 0; q < P / 2; ++q) split(q, X[((T - t) & (T - 1)) + (P / 2 - 1 - q) * T]);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < P / 2; ++q) X[t + q * T] = v[q];             // k in [0, L/2)
            __syncthreads();
#pragma unroll
            for (int q = P / 2; q < P; ++q) split(q, X[((T - t) & (T - 1)) + (P - 1 - q) * T]);
        } else {
            fence_proxy_async_smem();
            __syncthreads();
            if (t < 32 && more) load(X + YL, r + G, YL, L, fullX);   // the next tail, behind the stores
#pragma unroll
            for (int q = 0; q < P; ++q) st_stream(dst + q * T, INV ? scale_conj(v[q], scale) : v[q]);
        }
    }
}

}  // namespace bfft
