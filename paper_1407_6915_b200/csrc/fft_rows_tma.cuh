// fft_rows_tma.cuh — engine E1 (single pass) for the
// longest records that still fit one CTA, with the record loads taken off the
// compute warps: a producer warp streams whole records into an NSTAGE-deep
// ring of shared-memory stages with bulk copies (TMA), and NGRP compute groups
// of T = L / PP threads each FFT one staged record in place (the engine's
// exchanges reuse the stage) and store the result straight from registers.
//
// Why: k_rows holds a record's loads in registers, so at 2^13 (64 KiB records,
// 96 registers x 256 threads) only two records per SM are in flight and HBM
// idles while both compute (71 % of the roofline, profiles/r01_rows_2p13_minb.txt).
// Here the next record is already in shared memory when a group finishes.
//
// Records are dealt statically: CTA c takes records c, c + grid, ...; task k
// of a CTA is its k-th record, staged in stage k mod NSTAGE and computed by
// group k mod NGRP.  full[s] completes when the copy lands; empty[s] when every
// warp of the computing group has read the stage for the last time.
#pragma once

#include "fft_pipe.cuh"

namespace bfft {

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

template <int L, int PP, int NGRP, int NSTAGE>
struct RowsTmaCfg {
    using S = Sched<L, PP>;
    static constexpr int T = S::T;                                     // threads per record (one group)
    static constexpr int NT = NGRP * T + 32;                           // + producer warp
    static constexpr int STAGE = (RowLayout::size(L) + 15) / 16 * 16;  // entries per stage (padded exchanges)
    static constexpr int CHUNKS = L * 8 >= 4 * 16384 ? 4 : 1;          // bulk copies per record
    static constexpr size_t SMEM = sizeof(float2) * (size_t)STAGE * NSTAGE + 16 * NSTAGE;
    static constexpr int MINB = SMEM * 2 <= 227 * 1024 ? 2 : 1;
    static_assert(T % 32 == 0 && NGRP <= NSTAGE && (L / CHUNKS) % 2 == 0, "stage geometry");
};

template <int L, bool INV, int PP, int NGRP, int NSTAGE>
__global__ void __launch_bounds__(RowsTmaCfg<L, PP, NGRP, NSTAGE>::NT, RowsTmaCfg<L, PP, NGRP, NSTAGE>::MINB)
k_rows_tma(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec, const float2* __restrict__ tw,
           float scale) {
    using CF = RowsTmaCfg<L, PP, NGRP, NSTAGE>;
    constexpr int T = CF::T, P = CF::S::P, STAGE = CF::STAGE;
    extern __shared__ __align__(128) float2 sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)STAGE * NSTAGE);   // full | empty
    const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + NSTAGE);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, T / 32);   // one arrival per warp of the computing group
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t G = gridDim.x;
    if (warp == NGRP * T / 32) {
        // ============================================== producer
        const uint64_t pol = policy_evict_first();
        uint32_t k = 0;
        for (int64_t r = blockIdx.x; r < nrec; r += G, ++k) {
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            if (lane == 0) {
                if (u > 0) mbar_wait(empty0 + 8 * s, (u - 1) & 1);
                mbar_expect_tx(full0 + 8 * s, (uint32_t)(L * sizeof(float2)));
            }
            __syncwarp();
            constexpr int CH = L / CF::CHUNKS;
            if (lane < CF::CHUNKS)
                bulk_g2s_hint(smem_addr(sm + (size_t)s * STAGE + lane * CH), in + r * L + lane * CH,
                              CH * sizeof(float2), full0 + 8 * s, pol);
        }
    } else {
        // ============================================== compute groups
        const int grp = warp / (T / 32);
        const int t = tid - grp * T;
        const NamedBarrier bar{1 + grp, T};
        const TableTw<L, PP> tab{tw};
        uint32_t k = grp;
        for (int64_t r = blockIdx.x + (int64_t)grp * G; r < nrec; r += NGRP * G, k += NGRP) {
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            float2* stage = sm + (size_t)s * STAGE;
            mbar_wait(full0 + 8 * s, u & 1);
            float2 v[P];
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const float2 x = stage[t + j * T];
                v[j] = INV ? conjf2(x) : x;
            }
            fft_engine<L, PP>(v, t, stage, [](int e) { return RowLayout::at(e); }, tab, bar);
            fence_proxy_async_smem();   // last generic access of the stage: before its next bulk refill
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * s);
            float2* dst = out + r * L + t;
#pragma unroll
            for (int q = 0; q < P; ++q) st_stream(dst + q * T, INV ? scale_conj(v[q], scale) : v[q]);
        }
    }
}

}  // namespace bfft
