// Experiment (not product code): DRAM efficiency of column-tile access.
// A record of R x 2 KiB rows (256 x 256 complex64) is split into column
// tiles of W bytes; each CTA copies one tile (all 256 rows) per record from
// `in` to `out` (same tile position).  Measures GB/s vs W.
#include <cuda_runtime.h>
#include <stdint.h>
template <int WCOLS>  // tile width in complex64 columns (W = 8*WCOLS bytes)
__global__ void __launch_bounds__(256) ktile(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec) {
    constexpr int N2 = 256, N1 = 256, N = N1 * N2;
    constexpr int TILES = N2 / WCOLS;
    constexpr int ROWS_PER_PASS = 256 / WCOLS;          // 256 threads cover ROWS_PER_PASS rows per instruction
    const int col = threadIdx.x % WCOLS, r0 = threadIdx.x / WCOLS;
    for (int64_t g = blockIdx.x; g < nrec * TILES; g += gridDim.x) {
        const int64_t rec = g / TILES;
        const int c0 = (int)(g % TILES) * WCOLS;
        const float2* src = in + rec * N + c0 + col;
        float2* dst = out + rec * N + c0 + col;
        float2 v[32];
        // 256 rows / ROWS_PER_PASS passes; up to 32 loads in flight per thread
        constexpr int NP = N1 / ROWS_PER_PASS;
        for (int base = 0; base < NP; base += 32) {
#pragma unroll
            for (int s = 0; s < 32; ++s)
                if (base + s < NP) v[s] = __ldcs(src + (int64_t)(r0 + (base + s) * ROWS_PER_PASS) * N2);
#pragma unroll
            for (int s = 0; s < 32; ++s)
                if (base + s < NP) __stcs(dst + (int64_t)(r0 + (base + s) * ROWS_PER_PASS) * N2, v[s]);
        }
    }
}
__global__ void kcopy(const float4* __restrict__ in, float4* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(out + i, __ldcs(in + i));
}
template <int W>
static float run(const float2* in, float2* out, int64_t nrec, int reps) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ktile<W>, 256, 0);
    int grid = 148 * occ;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    ktile<W><<<grid, 256>>>(in, out, nrec);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) ktile<W><<<grid, 256>>>(in, out, nrec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
extern "C" float exp_tile(int w, const void* in, void* out, long long nrec, int reps) {
    switch (w) {
        case 16: return run<16>((const float2*)in, (float2*)out, nrec, reps);
        case 32: return run<32>((const float2*)in, (float2*)out, nrec, reps);
        case 64: return run<64>((const float2*)in, (float2*)out, nrec, reps);
        case 128: return run<128>((const float2*)in, (float2*)out, nrec, reps);
        case 256: return run<256>((const float2*)in, (float2*)out, nrec, reps);
        case 0: {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            int64_t n = nrec * 65536 / 2;
            kcopy<<<148 * 8, 256>>>((const float4*)in, (float4*)out, n);
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i) kcopy<<<148 * 8, 256>>>((const float4*)in, (float4*)out, n);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            return ms / reps;
        }
    }
    return -1;
}
