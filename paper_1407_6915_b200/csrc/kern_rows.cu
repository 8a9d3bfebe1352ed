// kern_rows.cu — single-pass row kernels (k_rows) and the two-kernel four-step (k_fs_cols, k_fs_rows): instantiations and pickers, compiled as its own translation unit
// (kernel instantiations dominate build time; plan.cu only dispatches).
#include "fft_kernels.cuh"
#include "fft_rows_tma.cuh"
#include "plan_internal.h"

using namespace bfft;

template <int L, int PP = 16> struct RowGeom {
    static constexpr int T = Sched<L, PP>::T;
    static constexpr int B = T >= 256 ? 1 : 256 / T;  // records per CTA
    static constexpr int THREADS = B * T;
    static constexpr size_t SMEM = Sched<L, PP>::NPASS > 1 ? sizeof(float2) * RowLayout::size(B * L) : 0;
};
template <int L> struct FsGeom {
    static constexpr int COLS = L >= 2048 ? 8 : 16;   // tile width (columns or rows)
    static constexpr int THREADS = COLS * Sched<L>::T;
    static constexpr size_t SMEM = sizeof(float2) * COLS * L;
};


template <int L, int PP = 16, int MINB = 0> static KernelSet row_real_kernel(bool inv) {
    using G = RowGeom<L, PP>;
    KernelSet k;
    k.fn = inv ? (const void*)&k_rows<L, G::B, true, PP, MINB, 2> : (const void*)&k_rows<L, G::B, false, PP, MINB, 1>;
    k.threads = G::THREADS;
    k.smem = sizeof(float2) * RowLayout::size(G::B * L);   // the partner exchange needs shared memory at any L
    k.cols = G::B;
    k.pp = PP;
    return k;
}
template <int L, int PP = 16, int MINB = 0> static KernelSet row_kernel(bool inv) {
    using G = RowGeom<L, PP>;
    KernelSet k;
    k.fn = inv ? (const void*)&k_rows<L, G::B, true, PP, MINB> : (const void*)&k_rows<L, G::B, false, PP, MINB>;
    k.threads = G::THREADS;
    k.smem = G::SMEM;
    k.cols = G::B;
    k.pp = PP;
    return k;
}
template <int L> static KernelSet fs_col_kernel(int n2, bool inv) {
    constexpr int C = FsGeom<L>::COLS;
    KernelSet k;
    k.fn = inv ? (const void*)&k_fs_cols<L, C, true> : (const void*)&k_fs_cols<L, C, false>;
    k.threads = FsGeom<L>::THREADS;
    k.smem = Sched<L>::NPASS > 1 ? FsGeom<L>::SMEM : 0;
    k.cols = C;
    (void)n2;
    return k;
}
template <int L> static KernelSet fs_row_kernel(bool inv) {
    constexpr int C = FsGeom<L>::COLS;
    KernelSet k;
    k.fn = inv ? (const void*)&k_fs_rows<L, C, true> : (const void*)&k_fs_rows<L, C, false>;
    k.threads = FsGeom<L>::THREADS;
    k.smem = FsGeom<L>::SMEM;  // the transposing tile load always uses shared memory
    k.cols = C;
    return k;
}

#define BFFT_L_CASES(M) \
    M(1, 2) M(2, 4) M(3, 8) M(4, 16) M(5, 32) M(6, 64) M(7, 128) M(8, 256) M(9, 512) M(10, 1024) \
    M(11, 2048)

KernelSet pick_row(int log2l, bool inv) {
    switch (log2l) {
#define M(k, L) case k: return row_kernel<L>(inv);
        BFFT_L_CASES(M)
#undef M
        case 12: return row_kernel<4096>(inv);
        // radix-32 engines at 2^13 and 2^14 (profiles/r01_rows_2p13_minb.txt)
        case 13: return row_kernel<8192, 32>(inv);
        case 14: return row_kernel<16384, 32>(inv);
        default: return KernelSet{};
    }
}
// k_rows_tma (fft_rows_tma.cuh): records streamed into shared-memory stages by
// bulk copies; two compute groups over three 68 KiB stages at 2^13 (85.7 % vs
// k_rows 73.9 %; 2^12 and shorter gain nothing: profiles/r02_rows_tma.txt)
template <int L, int PP, int NGRP, int NSTAGE, bool REAL = false> static KernelSet row_tma_kernel(bool inv) {
    using CF = RowsTmaCfg<L, PP, NGRP, NSTAGE>;
    KernelSet k;
    if constexpr (REAL)
        k.fn = inv ? (const void*)&k_rows_tma<L, true, PP, NGRP, NSTAGE, 2>
                   : (const void*)&k_rows_tma<L, false, PP, NGRP, NSTAGE, 1>;
    else
        k.fn = inv ? (const void*)&k_rows_tma<L, true, PP, NGRP, NSTAGE> : (const void*)&k_rows_tma<L, false, PP, NGRP, NSTAGE>;
    k.threads = CF::NT;
    k.smem = CF::SMEM;
    k.cols = 1;
    k.pp = PP;
    return k;
}
// 2^14: one record per CTA, its head staged apart from the exchange buffer
// (k_rows_tma2, 73 % vs k_pipe2 63 %: profiles/r02_rows_tma.txt)
constexpr int TMA2_HEAD = 10240;
template <int L, int PP, int YL, bool REAL = false> static KernelSet row_tma2_kernel(bool inv) {
    using CF = RowsTma2Cfg<L, PP, YL>;
    KernelSet k;
    if constexpr (REAL)
        k.fn = inv ? (const void*)&k_rows_tma2<L, true, PP, YL, 2> : (const void*)&k_rows_tma2<L, false, PP, YL, 1>;
    else
        k.fn = inv ? (const void*)&k_rows_tma2<L, true, PP, YL> : (const void*)&k_rows_tma2<L, false, PP, YL>;
    k.threads = CF::NT;
    k.smem = CF::SMEM;
    k.cols = 1;
    k.pp = PP;
    return k;
}
KernelSet pick_row_tma(int log2l, bool inv) {
    switch (log2l) {
        case 13: return row_tma_kernel<8192, 32, 2, 3>(inv);
        case 14: return row_tma2_kernel<16384, 32, TMA2_HEAD>(inv);
        default: return KernelSet{};
    }
}
// the staged kernel with the real-record split / merge fused (real records of
// 2^(log2l+1) samples), or an empty set
KernelSet pick_row_real_tma(int log2l, bool inv) {
    switch (log2l) {
        case 13: return row_tma_kernel<8192, 32, 2, 3, true>(inv);
        case 14: return row_tma2_kernel<16384, 32, TMA2_HEAD, true>(inv);
        default: return KernelSet{};
    }
}
KernelSet pick_row_real(int log2l, bool inv) {
    switch (log2l) {
#define M(k, L) case k: return row_real_kernel<L>(inv);
        BFFT_L_CASES(M)
#undef M
        case 12: return row_real_kernel<4096>(inv);
        case 13: return row_real_kernel<8192, 32>(inv);
        default: return KernelSet{};
    }
}
KernelSet pick_fs_col(int log2l, int n2, bool inv) {
    switch (log2l) {
#define M(k, L) case k: return fs_col_kernel<L>(n2, inv);
        BFFT_L_CASES(M)
#undef M
        default: return KernelSet{};
    }
}
KernelSet pick_fs_row(int log2l, bool inv) {
    switch (log2l) {
#define M(k, L) case k: return fs_row_kernel<L>(inv);
        BFFT_L_CASES(M)
#undef M
        default: return KernelSet{};
    }
}


int rows_upload_const(const float2* host, size_t count) {
    if (count != (size_t)CTW_TOTAL) return 1;
    return cudaMemcpyToSymbol(c_tw, host, count * sizeof(float2)) == cudaSuccess ? 0 : 1;
}
