// Experiment (not product code): phase timing of k_pipe (2^16, 256x256, 32x32 tiles).
#define BFFT_PIPE_PROF 1
#include "../../paper_1407_6915_b200/csrc/fft_pipe.cuh"
using namespace bfft;
extern "C" int exp_pipe(const void* in, void* out, void* ring, int* ctr, long long nrec, int S, int LAG,
                        const void* hi, const void* lo, int lb, unsigned long long* prof, float* ms) {
    auto fn = k_pipe<256, 256, 16, 16, false>;
    using CF = PipeCfg<256, 256, 16, 16>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, CF::NT, CF::SMEM);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_pipe_prof, z, sizeof z);
    cudaMemset(ctr, 0, sizeof(int) * (1 + 2 * S));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    fn<<<occ * 148, CF::NT, CF::SMEM>>>((const float2*)in, (float2*)out, (float2*)ring, nrec, ctr, S, LAG, 1.f,
                                        (const float2*)hi, (const float2*)lo, lb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    cudaMemcpyFromSymbol(prof, g_pipe_prof, sizeof z);
    return occ;
}
