// Experiments (not product code): skeletons of the cluster kernel to locate
// the time — the full k_cluster1 structure with pieces switched off.
//   MODE 0: full kernel (same as product k_cluster1)
//   MODE 1: no FFT arithmetic (engines skipped): load -> barrier -> push -> wait -> store
//   MODE 2: no exchange: load -> engines -> store (no cluster sync)
//   MODE 3: load -> store only (HBM skeleton, same access pattern)
#include "../../paper_1407_6915_b200/csrc/fft_cluster.cuh"

namespace bfft {
template <int N1, int N2, int C, int PP, int MINB_, int MODE>
__global__ void __launch_bounds__(Cluster1Cfg<N1, N2, C, PP, MINB_>::NT, Cluster1Cfg<N1, N2, C, PP, MINB_>::MINB)
kexp(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec) {
    using CF = Cluster1Cfg<N1, N2, C, PP, MINB_>;
    constexpr int N = CF::N, CA = CF::CA, CB = CF::CB, TA = CF::TA, TB = CF::TB, SLICE = CF::SLICE;
    constexpr uint32_t SLICE_BYTES = SLICE * sizeof(float2);
    constexpr int RSTRIDE = CF::RSTRIDE;
    extern __shared__ __align__(128) float2 sm[];
    float2* buf = sm;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + CF::BUF);
    const uint32_t bar_recv = smem_addr(&bars[0]);
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    const int colA = tid % CA, tA = tid / CA;
    const int n2 = (int)rank * CA + colA;
    const int colB = tid % CB, tB = tid / CB;
    const int k1b = (int)rank * CB + colB;
    if (tid == 0) {
        mbar_init(bar_recv, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_arrive_release();
    cluster_wait();
    const uint32_t buf_local = smem_addr(buf);
    const ConstTw<N1, PP> tabA{};
    const ConstTw<N2, PP> tabB{};
    auto addrA = [&](int e) { return ColLayout<CA>::at(e, colA); };
    auto addrB = [&](int e) { return ColLayout<CB>::at(e, colB); };
    uint32_t it = 0;
    for (int64_t r = cid; r < nrec; r += ncl, ++it) {
        if (MODE <= 1 && tid == 0) mbar_expect_tx(bar_recv, SLICE_BYTES);
        const float2* src = in + r * N + n2 + (int64_t)tA * N2;
        float2 v[PP];
#pragma unroll
        for (int s = 0; s < PP; ++s) v[s] = ld_stream(src + (int64_t)s * TA * N2);
        if (MODE == 0 || MODE == 2) fft_engine<N1, PP>(v, tA, buf, addrA, tabA);
        if (MODE <= 1) {
            cluster_arrive_relaxed();
            cluster_wait();
            const uint32_t my_base = buf_local + (uint32_t)((tA * RSTRIDE + n2) * sizeof(float2));
#pragma unroll
            for (int d = 0; d < C; ++d) {
                constexpr int QPD = CB / TA;
                const uint32_t rb = map_rank(my_base, (uint32_t)d);
                const uint32_t rbar = map_rank(bar_recv, (uint32_t)d);
#pragma unroll
                for (int i = 0; i < QPD; ++i) {
                    const int q = d * QPD + i;
                    st_async(rb + (uint32_t)(((q * TA) % CB) * RSTRIDE * sizeof(float2)), v[q], rbar);
                }
            }
            mbar_wait(bar_recv, it & 1);
#pragma unroll
            for (int s = 0; s < PP; ++s) v[s] = buf[colB * RSTRIDE + tB + s * TB];
        }
        if (MODE == 0 || MODE == 2) fft_engine<N2, PP>(v, tB, buf, addrB, tabB);
        float2* dst = out + r * N + k1b + (int64_t)tB * N1;
#pragma unroll
        for (int q = 0; q < PP; ++q) st_stream(dst + (int64_t)q * TB * N1, v[q]);
        __syncthreads();
    }
}
}  // namespace bfft

using namespace bfft;
template <int C, int MINB, int MODE>
static int launch(const float2* in, float2* out, long long nrec, int reps, float* ms) {
    using CF = Cluster1Cfg<256, 256, C, 32, MINB>;
    auto fn = kexp<256, 256, C, 32, MINB, MODE>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    if (C > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C * 148); cfg.blockDim = dim3(CF::NT); cfg.dynamicSmemBytes = CF::SMEM;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void*)fn, &cfg);
    cfg.gridDim = dim3(C * ncl);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) cudaLaunchKernelEx(&cfg, fn, in, out, (int64_t)nrec);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, fn, in, out, (int64_t)nrec);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b); *ms /= reps;
    return cudaGetLastError() == cudaSuccess ? ncl : -1;
}

extern "C" int exp_run(int c, int minb, int mode, const void* in, void* out, long long nrec, int reps, float* ms) {
#define CASE(CC, MB, MD) if (c == CC && minb == MB && mode == MD) return launch<CC, MB, MD>((const float2*)in, (float2*)out, nrec, reps, ms);
#define MODES(CC, MB) CASE(CC, MB, 0) CASE(CC, MB, 1) CASE(CC, MB, 2) CASE(CC, MB, 3)
    MODES(8, 2) MODES(16, 4) MODES(16, 3)
    return -2;
}
