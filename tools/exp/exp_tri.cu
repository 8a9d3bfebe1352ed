// Experiment (not product code): the three-factor pipelined four-step k_tri
// (fft_tri.cuh) at 2^20..2^22 with the ring size / lags given at run time.
#include "fft_tri.cuh"
#include <cudaTypedefs.h>
#include <cmath>
#include <vector>
using namespace bfft;

struct Cfg { const void* fn; int threads; size_t smem; int n1, n2, n3, nkb, ta, tb1, tb2, kb1x; const char* name; int h; };
template <int N1, int N2, int N3, int NST = 3, int NGRP = 4, int CB = 2, int H = 2>
static Cfg mk(const char* name) {
    using CF = TriCfg<N1, N2, N3, NST, NGRP, H>;
    return Cfg{(const void*)&k_tri<N1, N2, N3, false, NST, NGRP, CB, H>, CF::NT, CF::SMEM, N1, N2, N3, CF::NKB, CF::TA,
               CF::TB1, CF::TB2, H * CF::KB1, name, H};
}
static Cfg table(int i) {
    switch (i) {
        case 0: return mk<256, 64, 64>("tri 2^20 256x64x64");
        case 1: return mk<256, 128, 64>("tri 2^21 256x128x64");
        case 2: return mk<256, 128, 128>("tri 2^22 256x128x128");
        case 3: return mk<256, 64, 64, 3, 4, 1>("tri 2^20 cb1");
        case 4: return mk<256, 128, 128, 3, 4, 1>("tri 2^22 cb1");
        case 5: return mk<256, 64, 64, 3, 2, 1, 1>("tri 2^20 h1 s3 g2");
        case 6: return mk<256, 128, 64, 3, 2, 1, 1>("tri 2^21 h1 s3 g2");
        case 7: return mk<256, 128, 128, 3, 2, 1, 1>("tri 2^22 h1 s3 g2");
        case 8: return mk<256, 64, 64, 3, 2, 2, 1>("tri 2^20 h1 s3 g2 cb2");
        case 9: return mk<256, 128, 128, 3, 2, 2, 1>("tri 2^22 h1 s3 g2 cb2");
        default: return Cfg{nullptr};
    }
}
extern "C" int exp_ncfg() { return 10; }
extern "C" const char* exp_name(int i) { return table(i).name; }
extern "C" int exp_logn(int i) { Cfg c = table(i); return (int)std::log2((double)c.n1 * c.n2 * c.n3); }
extern "C" int exp_nctr(int i, int S) { Cfg c = table(i); return 2 + 2 * S + S * c.nkb; }
static void stockham_table(int L, std::vector<float2>& out, int P) {
    out.clear();
    if (L <= P) return;
    const int K = ilog2(L), KP = ilog2(P);
    const int R0 = (K % KP) ? (1 << (K % KP)) : P;
    const int npass = (K % KP) ? 1 + K / KP : K / KP;
    for (int p = 1; p < npass; ++p) {
        const int Ns = R0 * (1 << (KP * (p - 1)));
        const int M = P * Ns;
        for (int q = 1; q < P; ++q)
            for (int jj = 0; jj < Ns; ++jj) {
                const double ang = -2.0 * M_PI * (double)((long long)jj * q) / (double)M;
                out.push_back(make_float2((float)cos(ang), (float)sin(ang)));
            }
    }
}
extern "C" int exp_upload_tw() {
    std::vector<float2> all, one;
    for (int pp = 16; pp <= 32; pp *= 2)
        for (int l = CTW_MIN_L; l <= ctw_max_l(pp); l *= 2) {
            stockham_table(l, one, pp);
            all.insert(all.end(), one.begin(), one.end());
        }
    if ((int)all.size() != CTW_TOTAL) return 1;
    return cudaMemcpyToSymbol(c_tw, all.data(), all.size() * sizeof(float2)) != cudaSuccess;
}
// best of `reps` launch times in ms (negative: error)
extern "C" float exp_run(int i, const void* in, void* out, void* ring, int* ctr, long long nrec, int S, int L1,
                         int L2, const void* hi, const void* lo, int lb, int reps) {
    Cfg c = table(i);
    if (!c.fn) return -1.f;
    cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.fn, c.threads, c.smem);
    if (occ < 1) return -2.f;
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const long long M = (long long)c.n2 * c.n3, N = (long long)c.n1 * M;
    CUtensorMap tm, tr;
    cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)c.n1, (cuuint64_t)nrec};
    cuuint64_t strides[2] = {(cuuint64_t)M * 8, (cuuint64_t)N * 8};
    cuuint32_t box[3] = {(cuuint32_t)(16 * c.h), (cuuint32_t)c.n1, 1}, es[3] = {1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(in), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return -4.f;
    cuuint64_t rd[4] = {(cuuint64_t)c.n3, (cuuint64_t)c.n2, (cuuint64_t)c.n1, (cuuint64_t)S};
    cuuint64_t rsd[3] = {(cuuint64_t)c.n3 * 8, (cuuint64_t)M * 8, (cuuint64_t)N * 8};
    cuuint32_t rb[4] = {16, (cuuint32_t)c.n2, (cuuint32_t)c.kb1x, 1}, res[4] = {1, 1, 1, 1};
    if (enc(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, ring, rd, rsd, rb, res, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) return -5.f;
    using Fn = void (*)(const CUtensorMap, const CUtensorMap, float2*, float2*, int64_t, int*, int, int, int, float,
                        const float2*, const float2*, int);
    Fn fn = (Fn)c.fn;
    float best = 1e9f;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemset(ctr, 0, sizeof(int) * (2 + 2 * S + S * c.nkb));
    for (int it = 0; it < reps; ++it) {
        cudaEventRecord(a);
        fn<<<occ * 148, c.threads, c.smem>>>(tm, tr, (float2*)out, (float2*)ring, nrec, ctr, S, L1, L2, 1.f,
                                             (const float2*)hi, (const float2*)lo, lb);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (cudaGetLastError() != cudaSuccess) return -3.f;
        if (ms < best) best = ms;
    }
    return best;
}
