// kern_pipe3.cu — instantiations of k_pipe3 (fft_pipe3.cuh) and their picker,
// compiled as their own translation unit.
#include "fft_pipe3.cuh"
#include "plan_internal.h"

using namespace bfft;

template <int N1, int N2, int COLS, int ROWS, int NS, int G, int CB, bool PF = false>
static PipeChoice pipe3_kernel(bool inv) {
    using CF = Pipe3Cfg<N1, N2, COLS, ROWS, NS, G, 32>;
    PipeChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.cols = COLS;
    ch.rows = ROWS;
    ch.impl = 3;
    ch.stages = NS + G + CB;   // tasks a CTA holds besides its next claim (stages, groups, claim batch)
    ch.boxr = CF::BOXR;
    ch.k.fn = inv ? (const void*)&k_pipe3<N1, N2, COLS, ROWS, true, NS, G, 32, CB, PF>
                  : (const void*)&k_pipe3<N1, N2, COLS, ROWS, false, NS, G, 32, CB, PF>;
    ch.pp = 32;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}

// (stages, groups, claim batch) per size; fft_plan_opts::config selects the alternatives
// measured in profiles/ (32 KiB tiles: (4,3,4) / (3,4,4) / (1,2,2) x2 CTAs / (1,2,4) x2 CTAs;
// 64 KiB tiles: (1,2,1) / (1,2,2) / (1,2,1)+L2 prefetch / (1,2,2)+L2 prefetch; 4 = (1,2,2)+prefetch, 32 KiB)
template <int N1, int N2, int COLS, int ROWS>
static PipeChoice pipe3_pick(bool inv, int c) {
    constexpr size_t tile = sizeof(float2) * (size_t)Pipe3Cfg<N1, N2, COLS, ROWS, 1, 1, 32>::TILE;
    if constexpr (tile <= 36 * 1024) {
        if (c == 1) return pipe3_kernel<N1, N2, COLS, ROWS, 3, 4, 4>(inv);
        if (c == 2) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 2>(inv);   // two CTAs per SM
        if (c == 3) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 4>(inv);
        if (c == 4) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 2, true>(inv);
        return pipe3_kernel<N1, N2, COLS, ROWS, 4, 3, 4>(inv);
    } else {
        if (c == 1) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 2>(inv);
        if (c == 2) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 1, true>(inv);
        if (c == 3) return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 2, true>(inv);
        return pipe3_kernel<N1, N2, COLS, ROWS, 1, 2, 1>(inv);
    }
}

PipeChoice pick_pipe3(int log2n, bool inv, int config) {
    switch (log2n) {
        case 15: return pipe3_pick<256, 128, 16, 32>(inv, config);
        case 16: return pipe3_pick<256, 256, 16, 16>(inv, config);
        case 17: return pipe3_pick<512, 256, 8, 16>(inv, config);
        case 18: return pipe3_pick<512, 512, 8, 8>(inv, config);
        case 19: return pipe3_pick<1024, 512, 8, 16>(inv, config);
        case 20: return pipe3_pick<1024, 1024, 8, 8>(inv, config);
        default: return PipeChoice{};
    }
}

int pipe3_upload_const(const float2* host, size_t count) {
    if (count != (size_t)CTW_TOTAL) return 1;
    return cudaMemcpyToSymbol(c_tw, host, count * sizeof(float2)) == cudaSuccess ? 0 : 1;
}
