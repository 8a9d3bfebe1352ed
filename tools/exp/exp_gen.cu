// Experiment (not product code): k_pipe2 factorisations N = N1 x N2 and tile
// shapes at 2^15, 2^17, 2^18 (generalised from exp_wide.cu).
#include "../../paper_1407_6915_b200/csrc/fft_pipe.cuh"
#include <cudaTypedefs.h>
#include <cmath>
#include <vector>
using namespace bfft;

struct Cfg { const void* fn; int threads; size_t smem; int cols, rows, stages, twm, boxr, pp; const char* name; int cb; int h; int n1, n2; };

template <int N1, int N2, int COLS, int ROWS, int NST, int PP, int TWM, int NGRP = 1, int CB = 1>
static Cfg mk(const char* name) {
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NST, PP, NGRP>;
    return Cfg{(const void*)&k_pipe2<N1, N2, COLS, ROWS, false, NST, PP, TWM, NGRP, CB>, CF::NT,
               pipe2_smem<N1, N2, COLS, ROWS, NST, PP, TWM, NGRP>(), COLS, ROWS, NST, TWM, CF::BOXR, PP, name, CB, 1,
               N1, N2};
}
static Cfg table(int i) {
    switch (i) {
        case 0: return mk<256, 128, 16, 32, 3, 32, TW_SPLIT, 2>("2^15 256x128 c16 r32 s3 g2 (default)");
        case 1: return mk<128, 256, 32, 16, 3, 32, TW_SPLIT, 2>("2^15 128x256 c32 r16 s3 g2");
        case 2: return mk<512, 256, 8, 16, 3, 32, TW_SPLIT, 2>("2^17 512x256 c8 r16 s3 g2 (default)");
        case 3: return mk<256, 512, 16, 8, 3, 32, TW_SPLIT, 2>("2^17 256x512 c16 r8 s3 g2");
        case 4: return mk<512, 512, 16, 16, 3, 32, TW_SPLIT, 2>("2^18 512x512 c16 r16 s3 g2 (default, 64K)");
        case 5: return mk<128, 256, 32, 16, 2, 32, TW_SPLIT, 1>("2^15 128x256 c32 r16 s2 g1");
        case 6: return mk<256, 256, 16, 16, 3, 32, TW_SPLIT, 2>("2^16 256x256 c16 r16 s3 g2 (default)");
        case 7: return mk<128, 512, 32, 8, 3, 32, TW_SPLIT, 2>("2^16 128x512 c32 r8 s3 g2");
        case 8: return mk<512, 128, 8, 32, 3, 32, TW_SPLIT, 2>("2^16 512x128 c8 r32 s3 g2");
        case 9: return mk<128, 128, 32, 32, 3, 32, TW_SPLIT, 2>("2^14 128x128 c32 r32 s3 g2");
        case 10: return mk<256, 512, 16, 8, 3, 32, TW_TREE, 2>("2^17 256x512 c16 r8 s3 g2 tree");
        case 11: return mk<256, 512, 16, 8, 3, 32, TW_TABLE, 2>("2^17 256x512 c16 r8 s3 g2 table");
        case 12: return mk<512, 256, 8, 16, 3, 32, TW_TREE, 2>("2^17 512x256 c8 r16 s3 g2 tree");
        case 13: return mk<128, 512, 32, 8, 3, 32, TW_TREE, 2>("2^16 128x512 c32 r8 s3 g2 tree");
        case 14: return mk<512, 512, 8, 8, 3, 32, TW_TABLE, 2>("2^18 512x512 c8 r8 s3 g2 table");
        case 15: return mk<512, 512, 16, 16, 3, 32, TW_TABLE, 2>("2^18 512x512 c16 r16 s3 g2 table");
        case 16: return mk<1024, 512, 8, 16, 3, 32, TW_TABLE, 2>("2^19 1024x512 c8 r16 s3 g2 table");
        case 17: return mk<1024, 512, 8, 16, 3, 32, TW_SPLIT, 2>("2^19 1024x512 c8 r16 s3 g2 (default)");
        case 18: return mk<1024, 1024, 8, 8, 3, 32, TW_TABLE, 2>("2^20 1024x1024 c8 r8 s3 g2 table");
        case 19: return mk<1024, 1024, 8, 8, 3, 32, TW_SPLIT, 2>("2^20 1024x1024 c8 r8 s3 g2 (default)");
        case 20: return mk<512, 512, 8, 8, 3, 32, TW_TREE, 2>("2^18 512x512 c8 r8 s3 g2 tree");
        case 21: return mk<512, 1024, 16, 8, 3, 32, TW_TABLE, 2>("2^19 512x1024 c16 r8 s3 g2 table");
        case 22: return mk<256, 256, 16, 16, 3, 32, TW_TABLE, 2>("2^16 256x256 c16 r16 s3 g2 table");
        case 23: return mk<128, 256, 32, 16, 3, 32, TW_TABLE, 2>("2^15 128x256 c32 r16 s3 g2 table");
        case 24: return mk<1024, 1024, 8, 8, 3, 32, TW_TREE, 2>("2^20 1024x1024 c8 r8 s3 g2 tree");
        case 25: return mk<1024, 1024, 8, 8, 3, 32, TW_SPLIT, 2, 2>("2^20 1024x1024 c8 r8 s3 g2 cb2");
        case 26: return mk<1024, 1024, 8, 8, 2, 32, TW_SPLIT, 1>("2^20 1024x1024 c8 r8 s2 g1");
        case 27: return mk<1024, 512, 8, 16, 3, 32, TW_TREE, 2>("2^19 1024x512 c8 r16 s3 g2 tree");
        case 28: return mk<1024, 512, 8, 16, 3, 32, TW_SPLIT, 2, 2>("2^19 1024x512 c8 r16 s3 g2 cb2");
        case 29: return mk<512, 1024, 16, 8, 3, 32, TW_SPLIT, 2>("2^19 512x1024 c16 r8 s3 g2");
        case 30: return mk<512, 1024, 16, 8, 3, 32, TW_TREE, 2>("2^19 512x1024 c16 r8 s3 g2 tree");
        case 31: return mk<512, 512, 16, 16, 3, 32, TW_TREE, 2>("2^18 512x512 c16 r16 s3 g2 tree");
        case 32: return mk<512, 512, 16, 16, 3, 32, TW_SPLIT, 2, 2>("2^18 512x512 c16 r16 s3 g2 cb2");
        case 33: return mk<256, 1024, 16, 4, 3, 32, TW_TABLE, 2>("2^18 256x1024 c16 r4 s3 g2 table");
        case 34: return mk<512, 1024, 16, 8, 3, 32, TW_SPLIT, 2, 2>("2^19 512x1024 c16 r8 s3 g2 cb2");
        case 35: return mk<512, 512, 16, 16, 3, 32, TW_SPLIT, 2, 4>("2^18 512x512 c16 r16 s3 g2 cb4");
        case 36: return mk<256, 512, 16, 8, 3, 32, TW_TABLE, 2, 2>("2^17 256x512 c16 r8 s3 g2 table cb2");
        case 37: return mk<128, 256, 32, 16, 3, 32, TW_SPLIT, 2, 2>("2^15 128x256 c32 r16 s3 g2 cb2");
        case 38: return mk<512, 1024, 16, 8, 3, 32, TW_SPLIT, 2, 4>("2^19 512x1024 c16 r8 s3 g2 cb4");
        case 39: return mk<2048, 1024, 4, 8, 2, 16, TW_SPLIT, 1>("2^21 2048x1024 c4 r8 s2 g1 (default)");
        case 40: return mk<2048, 1024, 4, 8, 3, 16, TW_SPLIT, 1>("2^21 2048x1024 c4 r8 s3 g1");
        case 41: return mk<2048, 1024, 4, 8, 2, 16, TW_SPLIT, 1, 2>("2^21 2048x1024 c4 r8 s2 g1 cb2");
        case 42: return mk<2048, 1024, 4, 8, 3, 16, TW_SPLIT, 1, 2>("2^21 2048x1024 c4 r8 s3 g1 cb2");
        case 43: return mk<2048, 2048, 4, 4, 2, 16, TW_SPLIT, 1>("2^22 2048x2048 c4 r4 s2 g1 (default)");
        case 44: return mk<2048, 2048, 4, 4, 3, 16, TW_SPLIT, 1, 2>("2^22 2048x2048 c4 r4 s3 g1 cb2");
        case 45: return mk<2048, 1024, 2, 4, 3, 16, TW_SPLIT, 2>("2^21 2048x1024 c2 r4 s3 g2");
        default: return Cfg{nullptr};
    }
}
extern "C" int exp_ncfg() { return 46; }
extern "C" int exp_n1(int i) { return table(i).n1; }
extern "C" int exp_n2(int i) { return table(i).n2; }
// the constant-memory Stockham twiddles of this translation unit (same table as plan.cu builds)
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
extern "C" const char* exp_name(int i) { return table(i).name; }
extern "C" int exp_twm(int i) { return table(i).twm; }
extern "C" int exp_pp(int i) { return table(i).pp; }
// returns the best of `reps` launch times in ms (or -1); S/LAG as the plan sizes them
extern "C" float exp_run(int i, const void* in, void* out, void* ring, int* ctr, long long nrec, int maxS,
                         const void* hi, const void* lo, int lb, int reps, int* sOut, int* occOut) {
    Cfg c = table(i);
    if (!c.fn) return -1.f;
    cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.fn, c.threads, c.smem);
    if (occ < 1) return -2.f;
    const int resident = occ * 148, per_round = c.n2 / (c.cols * c.h) + c.n1 / (c.rows * c.h);
    const long long inflight = (long long)resident * (c.stages + c.cb);
    const long long rounds = (inflight + per_round - 1) / per_round;
    int LAG = (int)(3 * rounds / 2 + 1);
    int S = (int)(LAG + 2 * rounds + 1);
    if (S > maxS) S = maxS;
    *sOut = S; *occOut = occ;
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)c.n2, (cuuint64_t)c.n1, (cuuint64_t)nrec};
    cuuint64_t strides[2] = {(cuuint64_t)c.n2 * 8, (cuuint64_t)c.n1 * c.n2 * 8};
    cuuint32_t box[3] = {(cuuint32_t)(c.cols * c.h), (cuuint32_t)c.boxr, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(in), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    using Fn = void (*)(const CUtensorMap, float2*, float2*, int64_t, int*, int, int, float, const float2*,
                        const float2*, int, const float*, RealTw);
    Fn fn = (Fn)c.fn;
    float best = 1e9f;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < reps; ++it) {
        cudaMemsetAsync(ctr, 0, sizeof(int) * (1 + 2 * S));
        cudaEventRecord(a);
        fn<<<occ * 148, c.threads, c.smem>>>(tm, (float2*)out, (float2*)ring, nrec, ctr, S, LAG, 1.f,
                                             (const float2*)hi, (const float2*)lo, lb, nullptr, RealTw{});
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (cudaGetLastError() != cudaSuccess) return -3.f;
        if (ms < best) best = ms;
    }
    return best;
}
