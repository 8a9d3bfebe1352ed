// fft_cluster.cuh — the cluster variant: one record per thread-block cluster,
// the four-step transpose done as an all-to-all through distributed shared
// memory (SURVEY.md §8(a) rows a3', a4), so each record is read from HBM once
// and written once (16 N bytes, the algorithmic minimum).
//
// N = N1 * N2, cluster of C CTAs, n = N2 n1 + n2, k = k1 + N1 k2.
//   phase A (CTA `rank`): columns n2 in [rank*CA, (rank+1)*CA), CA = N2/C:
//       Y[k1][n2] = W_N^{n2 k1} * sum_n1 x[N2 n1 + n2] W_N1^{n1 k1}
//   exchange: Y[k1][n2] goes to CTA k1 / CB (CB = N1/C), into its `recv`
//   phase B (CTA `rank`): rows k1 in [rank*CB, (rank+1)*CB):
//       X[k1 + N1 k2] = sum_n2 Y[k1][n2] W_N2^{n2 k2}
//
// Blackwell mechanics:
//   * phase-A input tile (N1 rows x CA columns of one record) is fetched by a
//     TMA tensor copy (cp.async.bulk.tensor) into `stage`, one record ahead;
//   * the exchange: each CTA lays its Y out destination-major in `work`
//     (one contiguous CA x CB block per destination) and pushes each block
//     with one bulk shared->distributed-shared copy (cp.async.bulk
//     .shared::cluster.shared::cta) that complete_tx's on the destination's
//     mbarrier — no cluster-scope release fence (which would wait for every
//     outstanding global store), few large DSMEM transactions;
//   * the destination, once its slice has landed, arrives remotely on every
//     source's `send_free` mbarrier, which gates the source's next write of
//     `work`;
//   * `recv` reuse is protected by a relaxed split cluster barrier (arrive
//     after the last read of recv, wait before the next pushes).
#pragma once

#include <cuda.h>

#include "fft_kernels.cuh"

namespace bfft {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
// Remote 8-byte store into another CTA's shared memory that counts 8 bytes
// against that CTA's mbarrier `rbar` (both shared::cluster addresses).
__device__ __forceinline__ void st_async(uint32_t raddr, float2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "f"(v.x), "f"(v.y), "r"(rbar)
                 : "memory");
}
// Bulk copy of `bytes` (multiple of 16) from this CTA's shared memory to
// another CTA's (shared::cluster address), completing on that CTA's mbarrier.
__device__ __forceinline__ void bulk_s2s(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
                 "r"(src), "r"(bytes), "r"(rbar)
                 : "memory");
}
// Arrive (count 1) on a possibly remote mbarrier (shared::cluster address).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
// Order this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy / TMA) accesses.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA: 3-D tile {c0, c1, c2} of `tmap` into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tmap, int c0, int c1, int c2,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

template <int N1, int N2, int C>
struct ClusterCfg {
    static constexpr int N = N1 * N2;
    static constexpr int CA = N2 / C;   // phase-A columns per CTA
    static constexpr int CB = N1 / C;   // phase-B columns (rows k1) per CTA
    static constexpr int NT = N / (16 * C);
    static constexpr int TA = Sched<N1>::T, TB = Sched<N2>::T;
    static constexpr int SLICE = N / C;  // complex entries per CTA buffer
    static_assert(Sched<N1>::P == 16 && Sched<N2>::P == 16, "cluster variant needs N1, N2 >= 16");
    static_assert(CA * TA == NT && CB * TB == NT, "thread mapping");
    static_assert(CA >= 16 && CB >= 16, "column tiles of >= 16 keep shared accesses conflict-free");
    static_assert(N1 <= 256 && CA <= 256, "TMA box dimensions are <= 256");
    static constexpr int BLK = CA * CB;  // complex entries sent to each destination
    // stage (TMA landing) + work (phase-A exchange, then send blocks) + recv
    // (phase-B input/exchange) + 3 mbarriers
    static constexpr size_t SMEM = 3 * sizeof(float2) * SLICE + 64;
    // CTAs per SM that fit the shared memory (227 KiB opt-in per SM): the
    // register budget is capped accordingly through __launch_bounds__.
    static constexpr int MINB_RAW = (int)((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB = MINB_RAW < 1 ? 1 : (MINB_RAW > 4 ? 4 : MINB_RAW);
};

// Exchange modes: XCH_BULK stages destination-major blocks in `work` and
// pushes each with one bulk DSMEM copy; XCH_STAS pushes every value with an
// st.async whose warp footprint is a contiguous 256 B run of the
// destination's recv, laid out [k1 mod CB][n2] (n2 fastest, XOR-swizzled in
// 16-element groups so phase B's column reads stay conflict-free).
enum { XCH_BULK = 0, XCH_STAS = 1 };

template <int N1, int N2, int C, bool INV, int XCH>
__global__ void __launch_bounds__(ClusterCfg<N1, N2, C>::NT, ClusterCfg<N1, N2, C>::MINB)
k_cluster(const __grid_constant__ CUtensorMap tmap, float2* __restrict__ out, int64_t nrec,
          const float2* __restrict__ tw1, const float2* __restrict__ tw2, float scale) {
    using CF = ClusterCfg<N1, N2, C>;
    constexpr int N = CF::N, CA = CF::CA, CB = CF::CB, TA = CF::TA, TB = CF::TB, SLICE = CF::SLICE;
    constexpr uint32_t SLICE_BYTES = SLICE * sizeof(float2);
    extern __shared__ __align__(128) float2 sm[];
    float2* stage = sm;              // TMA landing buffer: [n1][CA]
    float2* work = sm + SLICE;       // phase-A exchange
    float2* recv = sm + 2 * SLICE;   // phase-B input (written by every rank) and exchange
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 3 * SLICE);
    const uint32_t bar_stage = smem_addr(&bars[0]);   // TMA tile landed
    const uint32_t bar_recv = smem_addr(&bars[1]);    // all C incoming blocks landed
    const uint32_t bar_free = smem_addr(&bars[2]);    // all C destinations received my blocks
    constexpr int BLK = CF::BLK;
    constexpr uint32_t BLK_BYTES = BLK * sizeof(float2);
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();

    const int colA = tid % CA, tA = tid / CA;
    const int n2 = (int)rank * CA + colA;
    const int colB = tid % CB, tB = tid / CB;
    const int k1b = (int)rank * CB + colB;

    if (tid == 0) {
        mbar_init(bar_stage, 1);
        mbar_init(bar_recv, 1);
        mbar_init(bar_free, C);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // every rank's mbarriers are initialised before anyone pushes
    cluster_arrive_release();
    cluster_wait();

    // W_N^{n2 k1} for this thread's k1 = tA + q*TA: fixed for the whole kernel.
    float2 w4[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
        w4[q] = twiddle_exact(((uint32_t)n2 * (uint32_t)(tA + q * TA)) & (N - 1), N);
    // Send layout in `work`: block d (destination rank) holds Y[k1][n2] for
    // k1 in [d*CB, (d+1)*CB), n2 in [rank*CA, (rank+1)*CA), stored exactly as
    // the destination's recv rows n2: recv[ColLayout<CB>(n2, k1 mod CB)].
    // (XCH_STAS: remote address of Y[k1][n2] in rank k1/CB's recv.)
    uint32_t send_off[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int k1 = tA + q * TA;
        if constexpr (XCH == XCH_BULK)
            send_off[q] = (uint32_t)((k1 / CB) * BLK + (ColLayout<CB>::at(n2, k1 % CB) - rank * BLK));
        else
            send_off[q] = map_rank(smem_addr(recv), (uint32_t)(k1 / CB)) +
                          (uint32_t)(((k1 % CB) * N2 + (n2 ^ ((k1 % CB) & 15))) * sizeof(float2));
    }
    const TableTw<N1> tabA{tw1};
    const TableTw<N2> tabB{tw2};
    auto addrA = [&](int e) { return ColLayout<CA>::at(e, colA); };
    auto addrB = [&](int e) { return ColLayout<CB>::at(e, colB); };

    if (tid == 0 && cid < nrec) {
        mbar_expect_tx(bar_stage, SLICE_BYTES);
        tma_load_3d(smem_addr(stage), &tmap, (int)rank * CA, 0, (int)cid, bar_stage);
    }
    cluster_arrive_relaxed();  // "my recv is free" for the first record
    uint32_t it = 0;
    for (int64_t r = cid; r < nrec; r += ncl, ++it) {
        const uint32_t par = it & 1;
        if (tid == 0) mbar_expect_tx(bar_recv, SLICE_BYTES);  // this record's incoming slice
        // ---- phase A: column FFTs of length N1, times W_N^{n2 k1}
        mbar_wait(bar_stage, par);
        float2 v[16];
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            const float2 x = stage[(tA + s * TA) * CA + colA];
            v[s] = INV ? conjf2(x) : x;
        }
        __syncthreads();  // stage fully consumed: prefetch the next record
        if (tid == 0 && r + ncl < nrec) {
            mbar_expect_tx(bar_stage, SLICE_BYTES);
            tma_load_3d(smem_addr(stage), &tmap, (int)rank * CA, 0, (int)(r + ncl), bar_stage);
        }
        if constexpr (XCH == XCH_BULK) {
            if (it > 0) mbar_wait(bar_free, par ^ 1);  // my previous send blocks were delivered
        }
        fft_engine<N1>(v, tA, work, addrA, tabA);
        if constexpr (XCH == XCH_BULK) {
            __syncthreads();  // every thread finished reading `work`
#pragma unroll
            for (int q = 0; q < 16; ++q) work[send_off[q]] = cmul(v[q], w4[q]);
            fence_proxy_async();
            __syncthreads();
            // ---- exchange: one bulk DSMEM copy per destination rank
            cluster_wait();  // every rank has finished with its recv (previous record)
            if (tid < C) {
                const uint32_t d = (uint32_t)tid;
                bulk_s2s(map_rank(smem_addr(recv), d) + rank * BLK_BYTES, smem_addr(work) + d * BLK_BYTES,
                         BLK_BYTES, map_rank(bar_recv, d));
            }
        } else {
            // ---- exchange: coalesced st.async pushes, counted on the destination's mbarrier
            cluster_wait();  // every rank has finished with its recv (previous record)
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t dr = TA <= CB ? (uint32_t)((q * TA) / CB) : (uint32_t)((tA + q * TA) / CB);
                st_async(send_off[q], cmul(v[q], w4[q]), map_rank(bar_recv, dr));
            }
        }
        // ---- phase B: row FFTs of length N2, stored to X[k1 + N1 k2]
        mbar_wait(bar_recv, par);
        if constexpr (XCH == XCH_BULK) {
            if (tid < C) mbar_arrive_remote(map_rank(bar_free, (uint32_t)tid));  // source tid's block arrived
#pragma unroll
            for (int s = 0; s < 16; ++s) v[s] = recv[addrB(tB + s * TB)];
        } else {
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const int e = tB + s * TB;  // n2
                v[s] = recv[colB * N2 + (e ^ (colB & 15))];
            }
        }
        fft_engine<N2>(v, tB, recv, addrB, tabB);
        fence_proxy_async();
        cluster_arrive_relaxed();  // done with recv for this record
        float2* dst = out + r * N + k1b + (int64_t)tB * N1;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            st_stream(dst + (int64_t)q * TB * N1, INV ? scale_conj(v[q], scale) : v[q]);
    }
    cluster_wait();
    if constexpr (XCH == XCH_BULK) {
        if (it > 0) mbar_wait(bar_free, (it - 1) & 1);  // no bulk copy still reading `work` at exit
    }
}

}  // namespace bfft
