// kern_pipe.cu — pipelined four-step k_pipe / k_pipe2 instantiations and the pipelined-variant picker (k_pipe3 in kern_pipe3.cu), compiled as its own translation unit
// (kernel instantiations dominate build time; plan.cu only dispatches).

#include "fft_pipe.cuh"
#include "plan_internal.h"

using namespace bfft;

template <int N1, int N2, int COLS, int ROWS, int NSTAGE, int PP = 16, int TWM = TW_SPLIT, int NGRP = 1, int CB = 1>
static PipeChoice pipe2_kernel(bool inv) {
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP>;
    PipeChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.cols = COLS;
    ch.rows = ROWS;
    ch.impl = 2;
    ch.stages = NSTAGE;
    ch.boxr = CF::BOXR;
    ch.k.fn = inv ? (const void*)&k_pipe2<N1, N2, COLS, ROWS, true, NSTAGE, PP, TWM, NGRP, CB>
                  : (const void*)&k_pipe2<N1, N2, COLS, ROWS, false, NSTAGE, PP, TWM, NGRP, CB>;
    ch.twm = TWM;
    ch.pp = PP;
    ch.k.threads = CF::NT;
    ch.k.smem = pipe2_smem<N1, N2, COLS, ROWS, NSTAGE, PP, TWM, NGRP>();
    return ch;
}
// k_pipe2 with the real split fused (RS = 1: forward real records of 2 N1 N2
// samples; two groups per task over mirrored half tiles, one CTA per SM)
template <int N1, int N2, int COLS, int ROWS, int PP = 32>
static PipeChoice pipe2_real_kernel() {
    constexpr int NSTAGE = 3, NGRP = 4, H = 2;
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP, H>;
    PipeChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.cols = H * COLS;   // a task's columns / rows (tensor-map box, tasks per round)
    ch.rows = H * ROWS;
    ch.impl = 2;
    ch.stages = NSTAGE;
    ch.boxr = CF::BOXR;
    ch.k.fn = (const void*)&k_pipe2<N1, N2, COLS, ROWS, false, NSTAGE, PP, TW_SPLIT, NGRP, 2, false, H, 1>;
    ch.twm = TW_SPLIT;
    ch.pp = PP;
    ch.k.threads = CF::NT;
    ch.k.smem = pipe2_smem<N1, N2, COLS, ROWS, NSTAGE, PP, TW_SPLIT, NGRP, H>();
    return ch;
}
// the default k_pipe2 configurations with the C2R merge fused into the A-task
// read (RS = 2: inverse real records of 2 N1 N2 samples)
template <int N1, int N2, int COLS, int ROWS, int NSTAGE, int PP, int NGRP, int TWM = TW_SPLIT, int CB = 1>
static PipeChoice pipe2_real_inv_kernel() {
    PipeChoice ch = pipe2_kernel<N1, N2, COLS, ROWS, NSTAGE, PP, TWM, NGRP, CB>(true);
    ch.k.fn = (const void*)&k_pipe2<N1, N2, COLS, ROWS, true, NSTAGE, PP, TWM, NGRP, CB, false, 1, 2>;
    return ch;
}
PipeChoice pick_pipe_real_inv(int log2n) {
    switch (log2n) {   // complex length N = n / 2; the configurations pick_pipe ships
        case 15: return pipe2_real_inv_kernel<128, 256, 32, 16, 3, 32, 2>();
        case 16: return pipe2_real_inv_kernel<256, 256, 16, 16, 3, 32, 2>();
        // (256 x 512 with table twiddles and batched claims measured slower here: 27.8 / 33.7 %)
        case 17: return pipe2_real_inv_kernel<512, 256, 8, 16, 3, 32, 2>();
        case 18: return pipe2_real_inv_kernel<512, 512, 16, 16, 3, 32, 2>();
        default: return PipeChoice{};   // longer: two kernels measured faster (the partner reads miss L2)
    }
}
PipeChoice pick_pipe_real(int log2n) {
    switch (log2n) {   // complex length N = n / 2
        case 15: return pipe2_real_kernel<128, 256, 32, 16>();
        case 16: return pipe2_real_kernel<256, 256, 16, 16>();
        case 17: return pipe2_real_kernel<256, 512, 16, 8>();
        case 18: return pipe2_real_kernel<512, 512, 8, 8>();
        default: return PipeChoice{};
    }
}
template <int N1, int N2, int COLS, int ROWS> static PipeChoice pipe_kernel(bool inv) {
    using CF = PipeCfg<N1, N2, COLS, ROWS>;
    PipeChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.cols = COLS;
    ch.rows = ROWS;
    ch.k.fn = inv ? (const void*)&k_pipe<N1, N2, COLS, ROWS, true> : (const void*)&k_pipe<N1, N2, COLS, ROWS, false>;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}
// Pipelined four-step configurations per size: N = N1 * N2 (N1 >= N2), A-tile
// COLS columns, B-tile ROWS rows, NSTAGE staged tiles per CTA, PP points per
// thread, TWM = how the four-step twiddle is applied (TW_SPLIT except at 2^18
// one-group: fft_pipe.cuh; profiles/r02_twiddle_split.txt), NGRP compute
// groups per CTA.  The default (impl 0) is the warp-specialised k_pipe2 at
// every size, in its fastest measured configuration (profiles/r02_pipe2_groups.txt:
// radix-32 engines at 2^15..2^20, radix-16 with 64 KiB tiles at 2^21..2^22);
// impl 1 = k_pipe, 2 = k_pipe2, 3 = k_pipe3 select the alternatives
// explicitly (fft_plan_opts::impl / config; parity-tested in
// tests/test_gpu_parity.py).
PipeChoice pick_pipe(int log2n, bool inv, int impl, int config) {
    if (impl == 0) impl = 2;
    if (impl == 3) return pick_pipe3(log2n, inv, config);
    // k_pipe2 configurations (fft_plan_opts::config): 1 = one compute group over two
    // stages (three CTAs per SM at 32 KiB tiles), 2 = two groups over three stages,
    // 3 = two groups over three 64 KiB stages of 16-wide tiles; 0 = the fastest
    // measured per size (profiles/r02_pipe2_groups.txt): 2 at 2^15..2^17 and
    // 2^19..2^20, 3 at 2^18, 1 elsewhere
    if (impl == 2 && config == 0)
        config = (log2n == 18) ? 3 : ((log2n >= 15 && log2n <= 20) ? 2 : 1);
    if (impl == 2 && config == 3) {
        // two groups, three 64 KiB stages of 16-wide tiles (one CTA per SM)
        switch (log2n) {
            case 17: return pipe2_kernel<512, 256, 16, 32, 3, 32, TW_SPLIT, 2>(inv);
            // claims batched two at a time: 60.3 -> 61.8 % (profiles/r02_pipe2_factorisations.txt)
            case 18: return pipe2_kernel<512, 512, 16, 16, 3, 32, TW_SPLIT, 2, 2>(inv);
            default: return PipeChoice{};
        }
    }
    if (impl == 2 && config == 2) {
        // two compute groups per CTA over three stages (two CTAs per SM: 16 compute warps)
        switch (log2n) {
            case 14: return pipe2_kernel<128, 128, 16, 16, 3, 16, TW_SPLIT, 2>(inv);
            // 2^15 as 128 x 256: 32-wide A-tiles (256-byte DRAM runs), 63.4 % vs 60.1 % for
            // 256 x 128 with 16 x 32 tiles (profiles/r02_pipe2_factorisations.txt)
            case 15: return pipe2_kernel<128, 256, 32, 16, 3, 32, TW_SPLIT, 2>(inv);
            case 16: return pipe2_kernel<256, 256, 16, 16, 3, 32, TW_SPLIT, 2>(inv);
            // 2^17 as 256 x 512: 16-wide A-tiles (128-byte runs), twiddles from the full
            // [k1][n2] table (the split tables' shared memory would cost the second CTA):
            // 61.3 % vs 57.6 % for 512 x 256 (profiles/r02_pipe2_factorisations.txt)
            case 17: return pipe2_kernel<256, 512, 16, 8, 3, 32, TW_TABLE, 2, 2>(inv);
            case 18: return pipe2_kernel<512, 512, 8, 8, 3, 32, TW_TREE, 2>(inv);
            // 2^19 as 512 x 1024: 16-wide A-tiles (128-byte runs) — 60 % vs 56.7 % for
            // 1024 x 512 with 8-wide tiles (profiles/r02_pipe2_factorisations.txt)
            case 19: return pipe2_kernel<512, 1024, 16, 8, 3, 32, TW_SPLIT, 2>(inv);
            case 20: return pipe2_kernel<1024, 1024, 8, 8, 3, 32, TW_SPLIT, 2>(inv);
            default: return PipeChoice{};
        }
    }
    if (impl == 2 && config == 1) {
        switch (log2n) {
            case 13: return pipe2_kernel<128, 64, 16, 32, 2, 16>(inv);
            case 14: return pipe2_kernel<128, 128, 16, 16, 2, 16>(inv);
            case 15: return pipe2_kernel<256, 128, 16, 32, 2, 32>(inv);
            case 16: return pipe2_kernel<256, 256, 16, 16, 2, 32>(inv);
            case 17: return pipe2_kernel<512, 256, 8, 16, 2, 32>(inv);
            // TW_TREE at 2^18: the split tables' 12 KiB would cost the third CTA per SM
            case 18: return pipe2_kernel<512, 512, 8, 8, 2, 32, TW_TREE>(inv);
            case 19: return pipe2_kernel<1024, 512, 8, 16, 2, 32>(inv);
            case 20: return pipe2_kernel<1024, 1024, 8, 8, 2, 32>(inv);
            // radix-16 engines (the constant twiddles hold L = 2048 for P = 16 only), 64 KiB tiles
            case 21: return pipe2_kernel<2048, 1024, 4, 8, 2, 16>(inv);
            case 22: return pipe2_kernel<2048, 2048, 4, 4, 2, 16>(inv);
            default: return PipeChoice{};
        }
    }
    if (impl != 1 || config != 0) return PipeChoice{};
    switch (log2n) {
        case 13: return pipe_kernel<128, 64, 16, 32>(inv);
        case 14: return pipe_kernel<128, 128, 16, 16>(inv);
        case 15: return pipe_kernel<256, 128, 32, 64>(inv);
        case 16: return pipe_kernel<256, 256, 16, 16>(inv);
        case 17: return pipe_kernel<512, 256, 16, 32>(inv);
        case 18: return pipe_kernel<512, 512, 16, 16>(inv);
        case 19: return pipe_kernel<1024, 512, 8, 16>(inv);
        case 20: return pipe_kernel<1024, 1024, 8, 8>(inv);
        case 21: return pipe_kernel<2048, 1024, 8, 16>(inv);
        case 22: return pipe_kernel<2048, 2048, 8, 8>(inv);
        default: return PipeChoice{};
    }
}


int pipe_upload_const(const float2* host, size_t count) {
    if (count != (size_t)CTW_TOTAL) return 1;
    return cudaMemcpyToSymbol(c_tw, host, count * sizeof(float2)) == cudaSuccess ? 0 : 1;
}
