// Experiment (not product code): phase timing of k_pipe2 g2 s3 at 2^16 (BFFT_PIPE_PROF counters:
// per task of group 0 / thread 0, clock64 cycles waiting for the staged tile and working on it).
#define BFFT_PIPE_PROF 1
#include "exp_wide.cu"
extern "C" int exp_prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_pipe_prof, 32 * sizeof(unsigned long long)) != cudaSuccess;
}
extern "C" int exp_prof_zero() {
    unsigned long long z[32] = {0};
    return cudaMemcpyToSymbol(g_pipe_prof, z, sizeof z) != cudaSuccess;
}
