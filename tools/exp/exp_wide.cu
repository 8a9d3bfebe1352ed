// Experiment (not product code): k_pipe2 tile shapes at 2^16 — 128-byte
// (16-wide) vs 256-byte (32-wide) DRAM runs, radix-16 vs radix-32 engines,
// 2 vs 3 stages, four-step twiddles from a full table (TWT) or two-level.
#include "../../paper_1407_6915_b200/csrc/fft_pipe.cuh"
#include <cudaTypedefs.h>
#include <cmath>
#include <vector>
using namespace bfft;

struct Cfg { const void* fn; int threads; size_t smem; int cols, rows, stages, twm, boxr, pp; const char* name; int cb; int h; };

template <int COLS, int ROWS, int NST, int PP, int TWM, int NGRP = 1, int CB = 1, bool PF = false, int H = 1>
static Cfg mk(const char* name) {
    using CF = Pipe2Cfg<256, 256, COLS, ROWS, NST, PP, NGRP, H>;
    return Cfg{(const void*)&k_pipe2<256, 256, COLS, ROWS, false, NST, PP, TWM, NGRP, CB, PF, H>, CF::NT,
               pipe2_smem<256, 256, COLS, ROWS, NST, PP, TWM, NGRP, H>(), COLS, ROWS, NST, TWM, CF::BOXR, PP, name, CB,
               H};
}
static Cfg table(int i) {
    switch (i) {
        case 0: return mk<16, 16, 2, 32, TW_SPLIT>("c16 s2 g1");
        case 1: return mk<16, 16, 3, 32, TW_SPLIT, 2>("c16 s3 g2 (default)");
        case 2: return mk<8, 8, 6, 32, TW_SPLIT, 4>("c8 s6 g4");
        case 3: return mk<8, 8, 4, 32, TW_SPLIT, 3>("c8 s4 g3");
        case 4: return mk<8, 8, 3, 32, TW_SPLIT, 2>("c8 s3 g2");
        case 5: return mk<16, 16, 4, 32, TW_SPLIT, 3>("c16 s4 g3");
        case 6: return mk<16, 16, 5, 32, TW_SPLIT, 4>("c16 s5 g4");
        case 7: return mk<32, 32, 3, 32, TW_SPLIT, 2>("c32 s3 g2");
        case 8: return mk<16, 16, 3, 32, TW_SPLIT, 4, 1, false, 2>("c16 h2 s3 g4");
        case 9: return mk<16, 16, 3, 32, TW_SPLIT, 4, 2, false, 2>("c16 h2 s3 g4 cb2");
        case 10: return mk<16, 16, 2, 32, TW_SPLIT, 2, 1, false, 2>("c16 h2 s2 g2");
        case 11: return mk<16, 16, 4, 32, TW_SPLIT, 4, 1, false, 2>("c16 h2 s4 g4");
        case 12: return mk<8, 8, 3, 32, TW_SPLIT, 4, 1, false, 2>("c8 h2 s3 g4");
        case 13: return mk<8, 8, 3, 32, TW_SPLIT, 8, 1, false, 4>("c8 h4 s3 g8");
        case 14: return mk<16, 16, 5, 32, TW_SPLIT, 4, 4>("c16 s5 g4 cb4");
        case 15: return mk<16, 16, 6, 32, TW_SPLIT, 4, 4>("c16 s6 g4 cb4");
        case 16: return mk<16, 16, 6, 32, TW_SPLIT, 4, 2>("c16 s6 g4 cb2");
        case 17: return mk<16, 16, 6, 32, TW_SPLIT, 3, 4>("c16 s6 g3 cb4");
        case 18: return mk<16, 16, 3, 32, TW_SPLIT, 2, 2>("c16 s3 g2 cb2");
        case 19: return mk<16, 16, 3, 32, TW_SPLIT, 2, 1, true>("c16 s3 g2 pf");
        case 20: return mk<16, 16, 3, 32, TW_SPLIT, 2, 2, true>("c16 s3 g2 cb2 pf");
        default: return Cfg{nullptr, 0, 0, 0, 0, 0, 0, 0, 0, nullptr, 1, 1};
    }
}
extern "C" int exp_ncfg() { return 21; }
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
    const int resident = occ * 148, per_round = 256 / (c.cols * c.h) + 256 / (c.rows * c.h);
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
    cuuint64_t dims[3] = {256, 256, (cuuint64_t)nrec};
    cuuint64_t strides[2] = {256 * 8, 65536 * 8};
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
