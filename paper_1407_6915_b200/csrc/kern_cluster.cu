// kern_cluster.cu — thread-block-cluster kernels (k_cluster, k_cluster1, k_cluster2): instantiations and picker, compiled as its own translation unit
// (kernel instantiations dominate build time; plan.cu only dispatches).
#include "fft_cluster.cuh"
#include "plan_internal.h"

using namespace bfft;

template <int N1, int N2, int C> static ClusterChoice cluster_kernel(bool inv) {
    using CF = ClusterCfg<N1, N2, C>;
    ClusterChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.c = C;
    ch.impl = 3;
    // exchange by coalesced st.async (measured at least as fast as bulk copies)
    ch.k.fn = inv ? (const void*)&k_cluster<N1, N2, C, true, XCH_STAS> : (const void*)&k_cluster<N1, N2, C, false, XCH_STAS>;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}
template <int N1, int N2, int C, int MINB = 0> static ClusterChoice cluster1_kernel(bool inv) {
    using CF = Cluster1Cfg<N1, N2, C, 32, MINB>;
    ClusterChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.c = C;
    ch.pp = 32;
    ch.impl = 1;
    ch.k.fn = inv ? (const void*)&k_cluster1<N1, N2, C, true, 32, MINB> : (const void*)&k_cluster1<N1, N2, C, false, 32, MINB>;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}
template <int N1, int N2, int C, int PP = 16> static ClusterChoice cluster2_kernel(bool inv) {
    using CF = Cluster2Cfg<N1, N2, C, PP>;
    ClusterChoice ch;
    ch.n1 = N1;
    ch.n2 = N2;
    ch.c = C;
    ch.pp = PP;
    ch.impl = 2;
    ch.k.fn = inv ? (const void*)&k_cluster2<N1, N2, C, true, PP> : (const void*)&k_cluster2<N1, N2, C, false, PP>;
    ch.k.threads = CF::NT;
    ch.k.smem = CF::SMEM;
    return ch;
}
// Cluster configurations: N = N1*N2 over C CTAs.
// impl (fft_plan_opts::impl): 1 = single-buffer k_cluster1, 2 = pipelined
// k_cluster2, 3 = TMA-staged k_cluster; 0 = the fastest measured per size on
// B200 (profiles/r01_variants_*): k_cluster1 for 2^13..2^15 and 2^18,
// k_cluster with C = 16 for 2^16..2^17.  want_c = requested cluster size or 0.
ClusterChoice pick_cluster(int log2n, int want_c, bool inv, int impl) {
    if (impl == 0) impl = (log2n <= 15 || log2n >= 18) ? 1 : 3;
    if (impl == 3 && want_c == 0) want_c = 16;
    if (impl == 2) {
        switch (log2n) {
            case 13: return cluster2_kernel<64, 128, 4>(inv);
            case 14:
                if (want_c == 2) return cluster2_kernel<128, 128, 2>(inv);
                return cluster2_kernel<128, 128, 4>(inv);
            case 15: return cluster2_kernel<128, 256, 8>(inv);
            case 16:
                if (want_c == 8) return cluster2_kernel<256, 256, 8>(inv);
                return cluster2_kernel<256, 256, 16>(inv);
            case 17: return cluster2_kernel<256, 512, 16>(inv);
            default: return ClusterChoice{};
        }
    }
    if (impl == 1) {
        // register budgets (MINB = CTAs per SM) as measured best per size
        switch (log2n) {
            case 13: return cluster1_kernel<64, 128, 4, 6>(inv);
            case 14:
                if (want_c == 2) return cluster1_kernel<128, 128, 2, 2>(inv);
                return cluster1_kernel<128, 128, 4, 3>(inv);
            case 15: return cluster1_kernel<128, 256, 8, 3>(inv);
            case 16:
                if (want_c == 16) return cluster1_kernel<256, 256, 16, 4>(inv);
                return cluster1_kernel<256, 256, 8, 1>(inv);
            case 17:
                if (want_c == 8) return cluster1_kernel<256, 512, 8, 1>(inv);
                return cluster1_kernel<256, 512, 16, 1>(inv);
            case 18: return cluster1_kernel<512, 512, 16, 1>(inv);
            default: return ClusterChoice{};
        }
    }
    if (impl != 3) return ClusterChoice{};
    switch (log2n) {
        case 13: return cluster_kernel<64, 128, 4>(inv);
        case 14:
            if (want_c == 2) return cluster_kernel<128, 128, 2>(inv);
            return cluster_kernel<128, 128, 4>(inv);
        case 15: return cluster_kernel<128, 256, 8>(inv);
        case 16:
            if (want_c == 16) return cluster_kernel<256, 256, 16>(inv);
            return cluster_kernel<256, 256, 8>(inv);
        case 17: return cluster_kernel<256, 512, 16>(inv);
        default: return ClusterChoice{};
    }
}


int cluster_upload_const(const float2* host, size_t count) {
    if (count != (size_t)CTW_TOTAL) return 1;
    return cudaMemcpyToSymbol(c_tw, host, count * sizeof(float2)) == cudaSuccess ? 0 : 1;
}
