// kern_pipe.cu — pipelined four-step k_pipe / k_pipe2 instantiations and the pipelined-variant picker (k_pipe3 in kern_pipe3.cu), compiled as its own translation unit
// (kernel instantiations dominate build time; plan.cu only dispatches).
#include <cstdlib>

#include "fft_pipe.cuh"
#include "plan_internal.h"

using namespace bfft;

template <int N1, int N2, int COLS, int ROWS, int NSTAGE, int PP = 16, bool TWD = false, bool TWT = false>
static PipeChoice pipe2_kernel(bool inv) {
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP>;
    PipeChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.cols = COLS;
    ch.rows = ROWS;
    ch.impl = 2;
    ch.stages = NSTAGE;
    ch.boxr = CF::BOXR;
    ch.k.fn = inv ? (const void*)&k_pipe2<N1, N2, COLS, ROWS, true, NSTAGE, PP, TWD, TWT>
                  : (const void*)&k_pipe2<N1, N2, COLS, ROWS, false, NSTAGE, PP, TWD, TWT>;
    ch.twt = TWT;
    ch.pp = PP;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}
// radix-32 k_pipe2.  TWD: Stockham twiddles read directly from the constant table;
// TWT: four-step twiddles W_N^{n2 k1} from a full [k1][n2] table (N entries, N <= 2^18).
// Env BLOCKFFT_PIPE_TWD / BLOCKFFT_PIPE_TWT = 0/1 override the per-size defaults
// (profiles/r01_twiddle_direct.txt, r01_twiddle_table.txt).
template <int N1, int N2, int COLS, int ROWS, bool TWD = false, bool TWT = false>
static PipeChoice pipe2_p32(bool inv) {
    bool twd = TWD, twt = TWT;
    if (const char* e = getenv("BLOCKFFT_PIPE_TWD")) twd = atoi(e) != 0;
    if (const char* e = getenv("BLOCKFFT_PIPE_TWT")) twt = atoi(e) != 0;
    if constexpr (N1 * N2 <= (1 << 18)) {
        if (twt)
            return twd ? pipe2_kernel<N1, N2, COLS, ROWS, 2, 32, true, true>(inv)
                       : pipe2_kernel<N1, N2, COLS, ROWS, 2, 32, false, true>(inv);
    }
    return twd ? pipe2_kernel<N1, N2, COLS, ROWS, 2, 32, true>(inv) : pipe2_kernel<N1, N2, COLS, ROWS, 2, 32>(inv);
}
template <int N1, int N2, int COLS, int ROWS> static PipeChoice pipe2_pick(bool inv) {
    int ns = 2;
    if (const char* e = getenv("BLOCKFFT_PIPE_STAGES")) ns = atoi(e);
    return ns == 3 ? pipe2_kernel<N1, N2, COLS, ROWS, 3>(inv) : pipe2_kernel<N1, N2, COLS, ROWS, 2>(inv);
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
// Pipelined four-step splits (N1 >= N2; A-tile COLS columns, B-tile ROWS rows).
PipeChoice pick_pipe(int log2n, bool inv) {
    // fastest measured per size (profiles/r01_variants_*, r01_pipe3_*, r01_pipe2_large.txt):
    // k_pipe3 (compute groups, early stage release) for 2^19 and 2^20, warp-specialised
    // k_pipe2 for 2^13..2^18 and 2^21..2^22 (radix-16, 64 KiB tiles); k_pipe on request
    int impl = (log2n >= 19 && log2n <= 20) ? 3 : (log2n >= 13 && log2n <= 22) ? 2 : 1;
    if (const char* e = getenv("BLOCKFFT_PIPE_IMPL")) impl = atoi(e);
    if (impl == 3) {
        PipeChoice ch = pick_pipe3(log2n, inv);
        if (ch.k.fn) return ch;
        impl = (log2n >= 13 && log2n <= 20) ? 2 : 1;
    }
    if (impl == 2) {
        // radix-32 engines (32 points per thread) where measured faster, else radix-16
        const bool p32 = getenv("BLOCKFFT_PIPE_P32") ? atoi(getenv("BLOCKFFT_PIPE_P32")) != 0 : (log2n >= 15);
        switch (log2n) {
            case 13: return p32 ? pipe2_kernel<128, 64, 16, 32, 2, 32>(inv) : pipe2_pick<128, 64, 16, 32>(inv);
            case 14: return p32 ? pipe2_p32<128, 128, 16, 16>(inv) : pipe2_pick<128, 128, 16, 16>(inv);
            case 15: return p32 ? pipe2_p32<256, 128, 16, 32, false, true>(inv) : pipe2_pick<256, 128, 16, 32>(inv);
            case 16:
                if (getenv("BLOCKFFT_PIPE_TINY")) return pipe2_pick<256, 256, 8, 8>(inv);
                // full four-step twiddle table (profiles/r01_twiddle_table.txt)
                return p32 ? pipe2_p32<256, 256, 16, 16, false, true>(inv) : pipe2_pick<256, 256, 16, 16>(inv);
            case 17:
                if (getenv("BLOCKFFT_PIPE_WIDE")) return pipe2_pick<512, 256, 16, 32>(inv);
                return p32 ? pipe2_p32<512, 256, 8, 16>(inv) : pipe2_pick<512, 256, 8, 16>(inv);
            case 18:
                if (getenv("BLOCKFFT_PIPE_WIDE")) return pipe2_pick<512, 512, 16, 16>(inv);
                return p32 ? pipe2_p32<512, 512, 8, 8>(inv) : pipe2_pick<512, 512, 8, 8>(inv);
            case 19:
                if (getenv("BLOCKFFT_PIPE_P16")) return pipe2_pick<1024, 512, 8, 16>(inv);
                return pipe2_kernel<1024, 512, 8, 16, 2, 32>(inv);
            case 20:
                if (getenv("BLOCKFFT_PIPE_P16")) return pipe2_pick<1024, 1024, 8, 8>(inv);
                return pipe2_kernel<1024, 1024, 8, 8, 2, 32>(inv);
            // radix-16 engines (the constant twiddles hold L = 2048 for P = 16 only), 64 KiB tiles
            case 21: return pipe2_kernel<2048, 1024, 4, 8, 2, 16>(inv);
            case 22: return pipe2_kernel<2048, 2048, 4, 4, 2, 16>(inv);
            default: return PipeChoice{};
        }
    }
    switch (log2n) {
        case 13: return pipe_kernel<128, 64, 16, 32>(inv);
        case 14: return pipe_kernel<128, 128, 16, 16>(inv);
        case 15: return pipe_kernel<256, 128, 32, 64>(inv);
        case 16:
            if (getenv("BLOCKFFT_PIPE_WIDE")) return pipe_kernel<256, 256, 32, 32>(inv);
            return pipe_kernel<256, 256, 16, 16>(inv);
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
