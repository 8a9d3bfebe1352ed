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
            send_off[q] = (uint32_t)((k1 / CB) * BLK + (SwzColLayout<CB>::at(n2, k1 % CB) - rank * BLK));
        else
            send_off[q] = map_rank(smem_addr(recv), (uint32_t)(k1 / CB)) +
                          (uint32_t)(((k1 % CB) * N2 + (n2 ^ ((k1 % CB) & 15))) * sizeof(float2));
    }
    const ConstTw<N1> tabA{};
    const ConstTw<N2> tabB{};
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
            for (int s = 0; s < 16; ++s) v[s] = recv[SwzColLayout<CB>::at(tB + s * TB, colB)];
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

namespace bfft {

// ======================================================================
// Cluster variant, single-buffer form (k_cluster1).
//
// Same four-step split as k_cluster, tuned for shared-memory bandwidth
// (the binding on-chip resource: DESIGN.md "cluster variant"):
//   * phase A loads straight from HBM into registers (lanes = adjacent
//     columns n2, 256-byte coalesced rows) — no staging copy;
//   * each thread holds PP = 32 points (radix-32 passes), so a length-256
//     FFT is one radix-8 pass + one radix-32 pass with one exchange;
//   * the exchange is coalesced st.async into the destination's buffer,
//     laid out [k1 mod CB][n2] with rows padded to N2+1 entries (phase B's
//     column reads hit 16 distinct bank pairs), completing on its mbarrier;
//   * ONE shared buffer per CTA (N/C entries) serves phase A's exchange, the
//     incoming slice and phase B's exchange, so two CTAs fit per SM and the
//     second CTA's work hides the first one's cluster barrier and latency.
//     Ordering per record: phase A exchange -> cluster barrier (every rank's
//     buffer is free) -> pushes -> mbarrier (slice complete) -> phase B.
// ======================================================================
template <int N1, int N2, int C, int PP, int MINB_ = 0>
struct Cluster1Cfg {
    static constexpr int N = N1 * N2;
    static constexpr int CA = N2 / C, CB = N1 / C;
    static constexpr int TA = Sched<N1, PP>::T, TB = Sched<N2, PP>::T;
    static constexpr int NT = CA * TA;
    static constexpr int SLICE = N / C;
    static constexpr int RSTRIDE = N2 + 1;              // padded recv row [k1 mod CB][n2]
    static constexpr int BUF = CB * RSTRIDE;            // >= SLICE entries
    static_assert(Sched<N1, PP>::P == PP && Sched<N2, PP>::P == PP, "N1, N2 >= PP");
    static_assert(CB * TB == NT, "thread mapping");
    static_assert(CA >= 16 && CB >= 16, "column tiles of >= 16 keep shared accesses conflict-free");
    static constexpr size_t SMEM = sizeof(float2) * BUF + 16;
    static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB_REG = 65536 / (NT * 128);  // keep >= 128 registers per thread
    static constexpr int MINB0 = MINB_SMEM < MINB_REG ? MINB_SMEM : MINB_REG;
    // CTAs per SM the register budget is sized for (MINB_ = 0: as many as fit)
    static constexpr int MINB = MINB_ > 0 ? MINB_ : (MINB0 < 1 ? 1 : MINB0);
    static_assert(MINB <= MINB_SMEM, "shared memory does not fit MINB CTAs per SM");
};

template <int N1, int N2, int C, bool INV, int PP, int MINB_>
__global__ void __launch_bounds__(Cluster1Cfg<N1, N2, C, PP, MINB_>::NT, Cluster1Cfg<N1, N2, C, PP, MINB_>::MINB)
k_cluster1(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec,
           const float2* __restrict__ tw1, const float2* __restrict__ tw2, float scale) {
    using CF = Cluster1Cfg<N1, N2, C, PP, MINB_>;
    constexpr int N = CF::N, CA = CF::CA, CB = CF::CB, TA = CF::TA, TB = CF::TB, SLICE = CF::SLICE;
    constexpr uint32_t SLICE_BYTES = SLICE * sizeof(float2);
    extern __shared__ __align__(128) float2 sm[];
    constexpr int RSTRIDE = CF::RSTRIDE;
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

    // W_N^{n2 k1}, k1 = tA + q*TA, from fp64-accurate factors (<= 5 products)
    const uint32_t nmask = N - 1;
    const uint32_t m0 = ((uint32_t)n2 * (uint32_t)tA) & nmask, dm = ((uint32_t)n2 * (uint32_t)TA) & nmask;
    const float2 wb = twiddle_exact(m0, N);
    float2 ws[5];  // W^{dm * 2^i}
#pragma unroll
    for (int i = 0; i < 5; ++i) ws[i] = twiddle_exact((dm << i) & nmask, N);
    const uint32_t buf_local = smem_addr(buf);
    // remote bases: rank d's buffer and mbarrier
    const ConstTw<N1, PP> tabA{};
    const ConstTw<N2, PP> tabB{};
    auto addrA = [&](int e) { return ColLayout<CA>::at(e, colA); };
    auto addrB = [&](int e) { return ColLayout<CB>::at(e, colB); };

    uint32_t it = 0;
    for (int64_t r = cid; r < nrec; r += ncl, ++it) {
        if (tid == 0) mbar_expect_tx(bar_recv, SLICE_BYTES);
        // ---- phase A: column FFTs of length N1 (lanes = adjacent columns)
        const float2* src = in + r * N + n2 + (int64_t)tA * N2;
        float2 v[PP];
#pragma unroll
        for (int s = 0; s < PP; ++s) {
            const float2 x = ld_stream(src + (int64_t)s * TA * N2);
            v[s] = INV ? conjf2(x) : x;
        }
        fft_engine<N1, PP>(v, tA, buf, addrA, tabA);
        // ---- twiddle W_N^{n2 k1} and exchange
        cluster_arrive_relaxed();  // my reads of buf (phase A exchange) are done
        // w[q] = W^{m0 + q dm} = w[q with its lowest set bit cleared] * ws[that bit]
        // (one product per q, depth <= 5; indices are compile-time)
        float2 w[PP];
        w[0] = wb;
        v[0] = cmul(v[0], wb);
#pragma unroll
        for (int q = 1; q < PP; ++q) {
            const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;  // lowest set bit
            w[q] = cmul(w[q & (q - 1)], ws[lb]);
            v[q] = cmul(v[q], w[q]);
        }
        cluster_wait();  // every rank's buf is free
        static_assert(CB % TA == 0, "k1 = tA + q*TA: destination rank and row are compile-time offsets");
        // k1 = tA + q TA -> rank d = (q TA) / CB, row kl = tA + (q TA) mod CB.
        // mapa once per destination, then compile-time byte offsets (keeps the
        // 32 remote addresses out of registers).
        const uint32_t my_base = buf_local + (uint32_t)((tA * RSTRIDE + n2) * sizeof(float2));
#pragma unroll
        for (int d = 0; d < C; ++d) {
            constexpr int QPD = CB / TA;  // values per destination
            const uint32_t rb = map_rank(my_base, (uint32_t)d);
            const uint32_t rbar = map_rank(bar_recv, (uint32_t)d);
#pragma unroll
            for (int i = 0; i < QPD; ++i) {
                const int q = d * QPD + i;
                st_async(rb + (uint32_t)(((q * TA) % CB) * RSTRIDE * sizeof(float2)), v[q], rbar);
            }
        }
        // ---- phase B: row FFTs of length N2, stored to X[k1 + N1 k2]
        mbar_wait(bar_recv, it & 1);
#pragma unroll
        for (int s = 0; s < PP; ++s) {
            v[s] = buf[colB * RSTRIDE + tB + s * TB];  // Y[k1][n2 = tB + s TB]
        }
        fft_engine<N2, PP>(v, tB, buf, addrB, tabB);
        float2* dst = out + r * N + k1b + (int64_t)tB * N1;
#pragma unroll
        for (int q = 0; q < PP; ++q)
            st_stream(dst + (int64_t)q * TB * N1, INV ? scale_conj(v[q], scale) : v[q]);
        __syncthreads();  // phase B's last reads of buf precede the next record's phase-A writes
    }
}

}  // namespace bfft

namespace bfft {

// ======================================================================
// Cluster variant, software-pipelined form (k_cluster2) — the default.
//
// As k_cluster1 (LDG phase A, coalesced st.async exchange into padded
// [k1 mod CB][n2] rows, mbarrier completion), but the incoming slice is
// double-buffered so that iteration k runs phase A of record k and then
// phase B of record k-1:
//     A(k):   load, column FFTs (exchange in `work`), twiddle,
//             cluster-wait (every rank has finished B(k-2) = recv[k&1] free),
//             push into recv[k&1] of the destinations;
//     B(k-1): wait recv[(k-1)&1] complete, row FFTs (exchange in place), store;
//             cluster-arrive (my recv[(k-1)&1] is free again).
// The cluster barrier and the DSMEM transfer of record k are hidden behind
// a whole phase of compute instead of stalling every CTA of the cluster.
// Shared memory: work + 2 x recv.
// ======================================================================
template <int N1, int N2, int C, int PP>
struct Cluster2Cfg {
    static constexpr int N = N1 * N2;
    static constexpr int CA = N2 / C, CB = N1 / C;
    static constexpr int TA = Sched<N1, PP>::T, TB = Sched<N2, PP>::T;
    static constexpr int NT = CA * TA;
    static constexpr int SLICE = N / C;
    static constexpr int RSTRIDE = N2 + 1;   // padded recv row [k1 mod CB][n2]
    static constexpr int RBUF = CB * RSTRIDE;
    static_assert(Sched<N1, PP>::P == PP && Sched<N2, PP>::P == PP, "N1, N2 >= PP");
    static_assert(CB * TB == NT, "thread mapping");
    static_assert(CA >= 16 && CB >= 16, "column tiles of >= 16 keep shared accesses conflict-free");
    static_assert(CB % TA == 0, "destination rank/row of k1 = tA + q*TA are compile-time offsets");
    static constexpr size_t SMEM = sizeof(float2) * (SLICE + 2 * RBUF) + 32;
    static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB_REG = 65536 / (NT * 128);
    static constexpr int MINB0 = MINB_SMEM < MINB_REG ? MINB_SMEM : MINB_REG;
    static constexpr int MINB = MINB0 < 1 ? 1 : MINB0;
};

template <int N1, int N2, int C, bool INV, int PP>
__global__ void __launch_bounds__(Cluster2Cfg<N1, N2, C, PP>::NT, Cluster2Cfg<N1, N2, C, PP>::MINB)
k_cluster2(const float2* __restrict__ in, float2* __restrict__ out, int64_t nrec, float scale) {
    using CF = Cluster2Cfg<N1, N2, C, PP>;
    constexpr int N = CF::N, CA = CF::CA, CB = CF::CB, TA = CF::TA, TB = CF::TB, SLICE = CF::SLICE;
    constexpr int RSTRIDE = CF::RSTRIDE, RBUF = CF::RBUF;
    constexpr uint32_t SLICE_BYTES = SLICE * sizeof(float2);
    extern __shared__ __align__(128) float2 sm[];
    float2* work = sm;
    float2* recv0 = sm + SLICE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + SLICE + 2 * RBUF);
    const uint32_t bar0 = smem_addr(&bars[0]);   // bars[b]: slice of recv[b] complete
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    // records of this cluster: r_k = cid + k * ncl, k < K (cluster-uniform)
    const int64_t K = cid < nrec ? (nrec - cid + ncl - 1) / ncl : 0;

    const int colA = tid % CA, tA = tid / CA;
    const int n2 = (int)rank * CA + colA;
    const int colB = tid % CB, tB = tid / CB;
    const int k1b = (int)rank * CB + colB;

    if (tid == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_arrive_release();
    cluster_wait();

    // W_N^{n2 k1}, k1 = tA + q TA, from fp64-accurate factors (depth <= log2 PP)
    constexpr int LPP = ilog2(PP);
    const uint32_t nmask = N - 1;
    const float2 wb = twiddle_exact(((uint32_t)n2 * (uint32_t)tA) & nmask, N);
    float2 ws[LPP];
#pragma unroll
    for (int i = 0; i < LPP; ++i) ws[i] = twiddle_exact(((uint32_t)n2 * (uint32_t)(TA << i)) & nmask, N);
    const uint32_t recv_local = smem_addr(recv0);
    const uint32_t my_off = (uint32_t)((tA * RSTRIDE + n2) * sizeof(float2));
    const ConstTw<N1, PP> tabA{};
    const ConstTw<N2, PP> tabB{};
    auto addrA = [&](int e) { return ColLayout<CA>::at(e, colA); };

    if (K > 1 || K == 1) cluster_arrive_relaxed();  // recv[0] is free for A(0)
    for (int64_t k = 0; k <= K; ++k) {
        if (k < K) {
            // ================= phase A of record r_k
            const int64_t r = cid + k * ncl;
            const uint32_t b = (uint32_t)(k & 1);
            if (tid == 0) mbar_expect_tx(bar0 + 8 * b, SLICE_BYTES);
            const float2* src = in + r * N + n2 + (int64_t)tA * N2;
            float2 v[PP];
#pragma unroll
            for (int s = 0; s < PP; ++s) {
                const float2 x = ld_stream(src + (int64_t)s * TA * N2);
                v[s] = INV ? conjf2(x) : x;
            }
            fft_engine<N1, PP>(v, tA, work, addrA, tabA);
            {
                float2 w[PP];
                w[0] = wb;
                v[0] = cmul(v[0], wb);
#pragma unroll
                for (int q = 1; q < PP; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                    w[q] = cmul(w[q & (q - 1)], ws[lb]);
                    v[q] = cmul(v[q], w[q]);
                }
            }
            cluster_wait();  // every rank finished B(k-2): recv[b] is free everywhere
            const uint32_t base = recv_local + b * (uint32_t)(RBUF * sizeof(float2)) + my_off;
            const uint32_t bar = bar0 + 8 * b;
#pragma unroll
            for (int d = 0; d < C; ++d) {
                constexpr int QPD = CB / TA;
                const uint32_t rb = map_rank(base, (uint32_t)d);
                const uint32_t rbar = map_rank(bar, (uint32_t)d);
#pragma unroll
                for (int i = 0; i < QPD; ++i) {
                    const int q = d * QPD + i;
                    st_async(rb + (uint32_t)(((q * TA) % CB) * RSTRIDE * sizeof(float2)), v[q], rbar);
                }
            }
        }
        if (k >= 1) {
            // ================= phase B of record r_{k-1}
            const int64_t r = cid + (k - 1) * ncl;
            const uint32_t b = (uint32_t)((k - 1) & 1);
            float2* recv = recv0 + b * RBUF;
            mbar_wait(bar0 + 8 * b, (uint32_t)(((k - 1) >> 1) & 1));
            float2 v[PP];
#pragma unroll
            for (int s = 0; s < PP; ++s) v[s] = recv[colB * RSTRIDE + tB + s * TB];
            fft_engine<N2, PP>(v, tB, recv, [&](int e) { return ColLayout<CB>::at(e, colB); }, tabB);
            float2* dst = out + r * N + k1b + (int64_t)tB * N1;
#pragma unroll
            for (int q = 0; q < PP; ++q)
                st_stream(dst + (int64_t)q * TB * N1, INV ? scale_conj(v[q], scale) : v[q]);
        }
        if (k + 1 < K) cluster_arrive_relaxed();  // my recv[(k-1)&1] = recv[(k+1)&1] is free
    }
}

}  // namespace bfft
