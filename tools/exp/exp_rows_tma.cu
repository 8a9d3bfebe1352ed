// Experiment: k_rows_tma (fft_rows_tma.cuh) vs k_rows at 2^11..2^13
#include "../../paper_1407_6915_b200/csrc/fft_rows_tma.cuh"
#include <cmath>
#include <vector>
using namespace bfft;
struct Cfg { const void* fn; int threads; size_t smem; int L, pp; const char* name; int kind; };
template <int L, int PP, int YL> static Cfg mk2(const char* name) {
    using CF = RowsTma2Cfg<L, PP, YL>;
    return Cfg{(const void*)&k_rows_tma2<L, false, PP, YL>, CF::NT, CF::SMEM, L, PP, name, 1};
}
template <int L, int PP, int NGRP, int NST> static Cfg mk(const char* name) {
    using CF = RowsTmaCfg<L, PP, NGRP, NST>;
    return Cfg{(const void*)&k_rows_tma<L, false, PP, NGRP, NST>, CF::NT, CF::SMEM, L, PP, name, 1};
}
template <int L, int PP, int B, int MINB = 0> static Cfg mkr(const char* name) {
    return Cfg{(const void*)&k_rows<L, B, false, PP, MINB>, B * Sched<L, PP>::T, sizeof(float2) * RowLayout::size(B * L), L, PP, name, 0};
}
static Cfg table(int i) {
    switch (i) {
        case 0: return mkr<8192, 32, 1>("k_rows 2^13 (default)");
        case 1: return mk<8192, 32, 2, 3>("tma 2^13 g2 s3");
        case 2: return mk<8192, 32, 1, 2>("tma 2^13 g1 s2");
        case 3: return mk<8192, 32, 1, 3>("tma 2^13 g1 s3");
        case 4: return mkr<4096, 16, 1>("k_rows 2^12 (default)");
        case 5: return mk<4096, 32, 2, 3>("tma 2^12 p32 g2 s3");
        case 6: return mk<4096, 16, 1, 2>("tma 2^12 p16 g1 s2");
        case 7: return mk<4096, 32, 1, 2>("tma 2^12 p32 g1 s2");
        case 8: return mk<8192, 16, 1, 3>("tma 2^13 p16 g1 s3");
        case 9: return mkr<16384, 32, 1>("k_rows 2^14");
        case 10: return mk2<16384, 32, 10240>("tma2 2^14 head 10240");
        case 11: return mk2<16384, 32, 8192>("tma2 2^14 head 8192");
        case 12: return mk2<16384, 32, 11264>("tma2 2^14 head 11264");
        case 13: return mkr<512, 16, 8>("k_rows 2^9 p16 (default)");
        case 14: return mkr<512, 32, 16>("k_rows 2^9 p32");
        case 15: return mkr<1024, 16, 4>("k_rows 2^10 p16 (default)");
        case 16: return mkr<1024, 32, 8>("k_rows 2^10 p32");
        case 17: return mkr<2048, 16, 2>("k_rows 2^11 p16 (default)");
        case 18: return mkr<2048, 32, 4>("k_rows 2^11 p32");
        case 19: return mkr<4096, 32, 2>("k_rows 2^12 p32");
        case 20: return mkr<256, 16, 16>("k_rows 2^8 p16 (default)");
        case 21: return mk<4096, 32, 2, 3>("tma 2^12 p32 g2 s3");
        case 22: return mk<4096, 16, 1, 3>("tma 2^12 p16 g1 s3");
        case 23: return mk2<16384, 16, 10240>("tma2 2^14 p16 head 10240");
        case 24: return mk2<8192, 32, 4096>("tma2 2^13 p32 head 4096");
        case 25: return mk2<8192, 16, 4096>("tma2 2^13 p16 head 4096");
        case 26: return mkr<512, 16, 8, 4>("k_rows 2^9 minb4");
        case 27: return mkr<1024, 16, 4, 4>("k_rows 2^10 minb4");
        case 28: return mkr<2048, 16, 2, 4>("k_rows 2^11 minb4");
        case 29: return mkr<4096, 16, 1, 4>("k_rows 2^12 minb4");
        case 30: return mkr<1024, 16, 4, 5>("k_rows 2^10 minb5");
        case 31: return mkr<512, 16, 8, 3>("k_rows 2^9 minb3");
        case 32: return mkr<1024, 16, 4, 3>("k_rows 2^10 minb3");
        case 33: return mkr<2048, 16, 2, 3>("k_rows 2^11 minb3");
        case 34: return mkr<4096, 16, 1, 3>("k_rows 2^12 minb3");
        case 35: return mkr<256, 16, 16, 3>("k_rows 2^8 minb3");
        case 36: return mkr<256, 16, 16, 4>("k_rows 2^8 minb4");
        default: return Cfg{nullptr};
    }
}
extern "C" int exp_ncfg() { return 37; }
extern "C" const char* exp_name(int i) { return table(i).name; }
extern "C" int exp_L(int i) { return table(i).L; }
extern "C" int exp_pp(int i) { return table(i).pp; }
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
extern "C" float exp_run(int i, const void* in, void* out, long long nrec, int reps, int* occOut) {
    Cfg c = table(i);
    if (!c.fn) return -1.f;
    std::vector<float2> tw;
    stockham_table(c.L, tw, c.pp);
    float2* dtw = nullptr;
    cudaMalloc(&dtw, (tw.size() + 1) * sizeof(float2));
    cudaMemcpy(dtw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.fn, c.threads, c.smem);
    *occOut = occ;
    if (occ < 1) return -2.f;
    float best = 1e9f;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < reps; ++it) {
        cudaEventRecord(a);
        if (c.kind == 1) {
            using Fn = void (*)(const float2*, float2*, int64_t, const float2*, float, RealTw, int64_t, const float*);
            ((Fn)c.fn)<<<occ * 148, c.threads, c.smem>>>((const float2*)in, (float2*)out, nrec, dtw, 1.f, RealTw{}, c.L,
                                                        nullptr);
        } else {
            using Fn = void (*)(const float2*, float2*, int64_t, const float2*, float, int64_t, const float*, RealTw);
            const int grid = (int)std::min<long long>(nrec, (long long)occ * 148 * 8);
            ((Fn)c.fn)<<<grid, c.threads, c.smem>>>((const float2*)in, (float2*)out, nrec, dtw, 1.f, c.L, nullptr, RealTw{});
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (cudaGetLastError() != cudaSuccess) return -3.f;
        if (ms < best) best = ms;
    }
    cudaFree(dtw);
    return best;
}
