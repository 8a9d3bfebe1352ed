// Experiment (not product code): phase timing of k_pipe2 (2^16 narrow tiles).
#define BFFT_PIPE_PROF 1
#include "../../paper_1407_6915_b200/csrc/fft_pipe.cuh"
#include <cudaTypedefs.h>
using namespace bfft;
extern "C" int exp_pipe2(const void* in, void* out, void* ring, int* ctr, long long nrec, int S, int LAG,
                         const void* hi, const void* lo, int lb, unsigned long long* prof, float* ms) {
    auto fn = k_pipe2<256, 256, 16, 16, false, 2>;
    using CF = Pipe2Cfg<256, 256, 16, 16, 2>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, CF::NT, CF::SMEM);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap tm;
    cuuint64_t dims[3] = {256, 256, (cuuint64_t)nrec};
    cuuint64_t strides[2] = {256 * 8, 65536 * 8};
    cuuint32_t box[3] = {16, 256, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(in), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_pipe_prof, z, sizeof z);
    cudaMemset(ctr, 0, sizeof(int) * (1 + 2 * S));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    fn<<<occ * 148, CF::NT, CF::SMEM>>>(tm, (float2*)out, (float2*)ring, nrec, ctr, S, LAG, 1.f,
                                        (const float2*)hi, (const float2*)lo, lb, nullptr, RealTw{});
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    cudaMemcpyFromSymbol(prof, g_pipe_prof, sizeof z);
    return occ;
}
