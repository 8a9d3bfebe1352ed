// Experiment (not product code): DRAM efficiency of the four-step column-tile
// access patterns at the large sizes.  A record of N = N1 x N2 complex64 is
// split into column tiles of WCOLS columns (8*WCOLS bytes per row segment, row
// stride 8*N2 bytes); each CTA owns one tile of one record.  MODE 0: tile read
// + tile write (both strided), 1: strided read + contiguous write, 2:
// contiguous read + strided write.  Consecutive tiles go to consecutive CTAs.
#include <cuda_runtime.h>
#include <stdint.h>
template <int WCOLS, int N2, int N, int MODE>
__global__ void __launch_bounds__(256) ktile(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec) {
    constexpr int N1 = N / N2;
    constexpr int TILES = N2 / WCOLS;
    constexpr int RPP = 256 / WCOLS;                    // rows per instruction
    constexpr int NP = N1 / RPP;
    const int col = threadIdx.x % WCOLS, r0 = threadIdx.x / WCOLS;
    for (int64_t g = blockIdx.x; g < nrec * TILES; g += gridDim.x) {
        const int64_t rec = g / TILES;
        const int t = (int)(g % TILES);
        const int c0 = t * WCOLS;
        const float2* srcs = in + rec * N + c0 + col;
        float2* dsts = out + rec * N + c0 + col;
        const float2* srcc = in + rec * N + (int64_t)t * N1 * WCOLS;   // contiguous tile
        float2* dstc = out + rec * N + (int64_t)t * N1 * WCOLS;
        float2 v[32];
        for (int base = 0; base < NP; base += 32) {
#pragma unroll
            for (int s = 0; s < 32; ++s)
                if (base + s < NP) {
                    const int r = r0 + (base + s) * RPP;
                    v[s] = MODE == 2 ? __ldcs(srcc + (int64_t)(base + s) * 256 + threadIdx.x)
                                     : __ldcs(srcs + (int64_t)r * N2);
                }
#pragma unroll
            for (int s = 0; s < 32; ++s)
                if (base + s < NP) {
                    const int r = r0 + (base + s) * RPP;
                    if (MODE == 1) __stcs(dstc + (int64_t)(base + s) * 256 + threadIdx.x, v[s]);
                    else __stcs(dsts + (int64_t)r * N2, v[s]);
                }
        }
    }
}
template <int W, int N2, int N, int MODE>
static float run(const float2* in, float2* out, int64_t nrec, int reps) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ktile<W, N2, N, MODE>, 256, 0);
    int grid = 148 * occ;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    ktile<W, N2, N, MODE><<<grid, 256>>>(in, out, nrec);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) ktile<W, N2, N, MODE><<<grid, 256>>>(in, out, nrec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
template <int N2, int N, int MODE>
static float by_w(int w, const float2* in, float2* out, int64_t nrec, int reps) {
    switch (w) {
        case 4: return run<4, N2, N, MODE>(in, out, nrec, reps);
        case 8: return run<8, N2, N, MODE>(in, out, nrec, reps);
        case 16: return run<16, N2, N, MODE>(in, out, nrec, reps);
        case 32: return run<32, N2, N, MODE>(in, out, nrec, reps);
    }
    return -1;
}
template <int N2, int N>
static float by_mode(int mode, int w, const float2* in, float2* out, int64_t nrec, int reps) {
    switch (mode) {
        case 0: return by_w<N2, N, 0>(w, in, out, nrec, reps);
        case 1: return by_w<N2, N, 1>(w, in, out, nrec, reps);
        case 2: return by_w<N2, N, 2>(w, in, out, nrec, reps);
    }
    return -1;
}
// shape: 0 = 2^16 as 256 x 256, 1 = 2^20 as 1024 x 1024, 2 = 2^22 as 2048 x 2048
extern "C" float exp_tile2(int shape, int mode, int w, const void* in, void* out, long long nrec, int reps) {
    const float2* i = (const float2*)in;
    float2* o = (float2*)out;
    switch (shape) {
        case 0: return by_mode<256, 1 << 16>(mode, w, i, o, nrec, reps);
        case 1: return by_mode<1024, 1 << 20>(mode, w, i, o, nrec, reps);
        case 2: return by_mode<2048, 1 << 22>(mode, w, i, o, nrec, reps);
    }
    return -1;
}
