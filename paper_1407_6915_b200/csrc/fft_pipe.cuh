// fft_pipe.cuh — the four-step as ONE persistent,
// dependency-driven kernel whose intermediate stays in L2.
//
// N = N1 * N2, n = N2 n1 + n2, k = k1 + N1 k2:
//   A-task (record r, column tile c0..c0+COLS):
//       Y[k1][n2] = W_N^{n2 k1} * FFT_N1 over n1 of x[N2 n1 + n2]   -> ring slot r mod S
//   B-task (record r, row tile k0..k0+ROWS):
//       X[k1 + N1 k2] = FFT_N2 over n2 of Y[k1][n2]                  -> output
// Tasks are handed out in rounds by one global atomic counter: round s holds
// the A-tasks of record s and then the B-tasks of record s - LAG.  A B-task
// waits (acquire) until every A-task of its record has published; an A-task
// waits until the B-tasks of the record that last used its ring slot have
// read it.  Every dependency points to an earlier-issued task held by a
// running CTA, so the schedule cannot deadlock, and CTAs never idle at a
// grid-wide barrier.  The ring is S records (S N 8 bytes, sized to stay in
// the 126 MB L2): HBM sees x once and X once (16 N bytes per record, the
// algorithmic minimum) while the transpose traffic stays on chip.
#pragma once

#include <type_traits>

#include "fft_cluster.cuh"
#include "fft_kernels.cuh"

namespace bfft {

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Wait until *p >= target, with acquire semantics.  An acquire load compiles
// to LDG.STRONG.GPU + CCTL.IVALL (L1 invalidation), so only the first probe
// and the final load acquire: the polls in between are relaxed (invalidating
// L1 on every poll evicts the other warps' L1-cached data).  The writer
// publishes with a release (fence + red), so acquiring any later value
// synchronises with it.  Returns the value seen.
__device__ __forceinline__ int wait_geq_v(const int* p, int target) {
    int v = ld_acquire_gpu(p);
    if (v >= target) return v;
    int ns = 32;
    do {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : ns;
        v = ld_relaxed_gpu(p);
    } while (v < target);
    return ld_acquire_gpu(p);
}
__device__ __forceinline__ void wait_geq(const int* p, int target) { (void)wait_geq_v(p, target); }
// Cross-proxy fences (PTX memory model, "proxies"): data written by generic
// st.global in other CTAs and acquired by this thread must be made visible to
// this thread's later async-proxy (cp.async.bulk / TMA) reads of global
// memory; generic shared-memory accesses of a stage must be ordered before the
// TMA / bulk copy that later overwrites it.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ float2 ld_l2(const float2* p) { return __ldcg(p); }
// Drop a dead 128-byte line of the ring from L2 without writing it back: once
// a B-task holds its rows in shared memory the intermediate is dead, and
// discarding it keeps the ring's dirty lines from ever reaching HBM.
__device__ __forceinline__ void l2_discard128(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
// L2 eviction-priority policy for streaming data read exactly once.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// L2 prefetch of one TMA box (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* tmap, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* tmap, int c0, int c1, int c2,
                                                 uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
}

// The last CTA out resets the task and dependency counters ctr[0 .. 2S] and
// the exit counter ctr[2S + 1] to zero, so the next launch on the stream
// starts clean without a memset: fft_exec enqueues exactly one kernel.  Every
// CTA has finished with the counters before it counts itself out (CTA barrier,
// then a gpu-scope fence before the exit atomic), so the reset cannot race.
__device__ __forceinline__ void pipe_exit_reset(int* ctr, int S) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(ctr + 1 + 2 * S, 1);
        if (prev == (int)gridDim.x - 1) {
            __threadfence();
            for (int i = 0; i <= 2 * S + 1; ++i) ctr[i] = 0;
        }
    }
}
// W_N^m from the plan's two-level table (fp64-computed, fp32-rounded):
// W^m = hi[m >> LB] * lo[m & (2^LB - 1)], one extra rounding.
struct TwoLevel {
    const float2* __restrict__ hi;
    const float2* __restrict__ lo;
    int lb;
    uint32_t nmask;
    __device__ __forceinline__ float2 operator()(uint32_t m) const {
        m &= nmask;
        return cmul(__ldg(hi + (m >> lb)), __ldg(lo + (m & ((1u << lb) - 1))));
    }
};

template <int N1, int N2, int COLS, int ROWS>
struct PipeCfg {
    static constexpr int N = N1 * N2;
    static constexpr int NT = COLS * Sched<N1>::T;
    static_assert(ROWS * Sched<N2>::T == NT, "A and B tasks use the same block");
    static_assert(Sched<N1>::P == 16 && Sched<N2>::P == 16, "N1, N2 >= 16");
    static constexpr int TA = N2 / COLS;  // A-tasks per record
    static constexpr int TB = N1 / ROWS;  // B-tasks per record
    static constexpr int SM_ENTRIES = (COLS * N1 > ROWS * N2 ? COLS * N1 : ROWS * N2);
    static constexpr size_t SMEM = sizeof(float2) * SM_ENTRIES + 16;
    static constexpr int MINB_RAW = 65536 / (NT * 64);  // registers per thread >= 64
    static constexpr int MINB = MINB_RAW < 1 ? 1 : (MINB_RAW > 8 ? 8 : MINB_RAW);
};

// Optional phase timing (experiments only: tools/exp/exp_pipe.cu defines
// BFFT_PIPE_PROF; the product library never does).
#ifdef BFFT_PIPE_PROF
static __device__ unsigned long long g_pipe_prof[32];
#define P2_T(v) unsigned long long v = clock64();
#define P2_ACC(slot, a, b) atomicAdd(&g_pipe_prof[slot], (b) - (a));
#else
#define P2_T(v)
#define P2_ACC(slot, a, b)
#endif
#ifdef BFFT_PIPE_PROF
#define PIPE_T(i) unsigned long long _t##i = 0; if (tid == 0) _t##i = clock64();
#define PIPE_ACC(slot, a, b) if (tid == 0) atomicAdd(&g_pipe_prof[slot], _t##b - _t##a);
#else
#define PIPE_T(i)
#define PIPE_ACC(slot, a, b)
#endif

// Stress build (tests only: tools/stress_build.py compiles the pipelined units
// with -DBFFT_STRESS into libblockfft_stress.so): pseudo-random sleeps of up to
// ~2 us at the protocol's synchronisation points perturb the interleaving of
// producers, compute warps, release warps and CTAs, so a missing wait or an
// unordered publication shows up as a result that differs from the product
// build's (tests/test_gpu_stress.py; compute-sanitizer is closed on this pool,
// profiles/r02_compute_sanitizer_closed.txt).
#ifdef BFFT_STRESS
__device__ __forceinline__ void stress_delay(unsigned salt) {
    const unsigned long long c = clock64();
    unsigned h = (unsigned)(c ^ (c >> 13)) * 2654435761u ^ (blockIdx.x * 97u + salt * 131u + (threadIdx.x >> 5) * 7u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    if ((h & 3u) == 0) __nanosleep((h >> 20) & 2047u);
}
#define BFFT_STRESS_DELAY(salt) stress_delay(salt)
#else
#define BFFT_STRESS_DELAY(salt)
#endif

// ctr layout (int32): [0] task counter, [1 .. S] A-tasks published per slot,
// [S+1 .. 2S] B-tasks finished reading per slot (cumulative across reuses),
// [2S+1] CTAs finished (pipe_exit_reset).
template <int N1, int N2, int COLS, int ROWS, bool INV>
__global__ void __launch_bounds__(PipeCfg<N1, N2, COLS, ROWS>::NT, PipeCfg<N1, N2, COLS, ROWS>::MINB)
k_pipe(const float2* __restrict__ in, float2* __restrict__ out, float2* __restrict__ ring, int64_t nrec,
       int* __restrict__ ctr, int S, int LAG, float scale, const float2* __restrict__ w_hi,
       const float2* __restrict__ w_lo, int w_lb) {
    using CF = PipeCfg<N1, N2, COLS, ROWS>;
    constexpr int N = CF::N, TA = CF::TA, TB = CF::TB;
    constexpr int TA1 = Sched<N1>::T, TB2 = Sched<N2>::T;
    constexpr int NT = CF::NT;
    extern __shared__ __align__(128) float2 sm[];
    __shared__ int s_task;
    const int tid = threadIdx.x;
    int* doneA = ctr + 1;
    int* doneB = ctr + 1 + S;
    const int64_t per_round = TA + TB;
    const int64_t total = (nrec + LAG) * per_round;
    const ConstTw<N1> tabA{};
    const ConstTw<N2> tabB{};
    const TwoLevel W{w_hi, w_lo, w_lb, (uint32_t)(N - 1)};

    // The next task index is claimed while the current task runs (its atomic
    // round trip to L2 is off the critical path).
    int next = 0;
    if (tid == 0) next = atomicAdd(ctr, 1);
    for (;;) {
        __syncthreads();  // s_task and shared memory of the previous task are free
        if (tid == 0) {
            s_task = next;
            if (next < total) next = atomicAdd(ctr, 1);
        }
        __syncthreads();
        const int64_t task = s_task;
        if (task >= total) break;
        PIPE_T(0)
        const int64_t round = task / per_round;
        const int o = (int)(task - round * per_round);
        if (o < TA) {
            // ================================================ A-task
            const int64_t r = round;
            if (r >= nrec) continue;
            const int slot = (int)(r % S);
            const int gen = (int)(r / S);
            const int col = tid % COLS, t = tid / COLS;
            const int n2 = o * COLS + col;
            const float2* src = in + r * N + n2 + (int64_t)t * N2;
            float2 v[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const float2 x = ld_stream(src + (int64_t)s * TA1 * N2);
                v[s] = INV ? conjf2(x) : x;
            }
            // W_N^{n2 k1} factors, fetched before the engine so their latency hides behind it
            float2 f[4], w0;
#pragma unroll
            for (int i = 0; i < 4; ++i) f[i] = W((uint32_t)n2 * (uint32_t)(TA1 << i));
            w0 = W((uint32_t)n2 * (uint32_t)t);
            fft_engine<N1>(v, t, sm, [&](int e) { return ColLayout<COLS>::at(e, col); }, tabA);
            PIPE_T(1)
            // k1 = t + q TA1: w[q] = w[q without its lowest bit] * f[lowbit]
            {
                float2 w[16];
                w[0] = w0;
                v[0] = cmul(v[0], w[0]);
#pragma unroll
                for (int q = 1; q < 16; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : 3;
                    w[q] = cmul(w[q & (q - 1)], f[lb]);
                    v[q] = cmul(v[q], w[q]);
                }
            }
            PIPE_T(2)
            BFFT_STRESS_DELAY(1);
            // the slot's previous record must have been read by all its B-tasks
            if (gen > 0) {
                if (tid == 0) wait_geq(doneB + slot, gen * TB);
                __syncthreads();
            }
            PIPE_T(3)
            BFFT_STRESS_DELAY(2);
            float2* dst = ring + (int64_t)slot * N + n2 + (int64_t)t * N2;
#pragma unroll
            for (int q = 0; q < 16; ++q) dst[(int64_t)q * TA1 * N2] = v[q];
            __syncthreads();
            if (tid == 0) red_release_gpu(doneA + slot, 1);
            PIPE_T(4)
            PIPE_ACC(0, 0, 1) PIPE_ACC(1, 1, 2) PIPE_ACC(2, 2, 3) PIPE_ACC(3, 3, 4)
            if (tid == 0) { PIPE_ACC(4, 0, 4) }
#ifdef BFFT_PIPE_PROF
            if (tid == 0) atomicAdd(&g_pipe_prof[10], 1ull);
#endif
        } else {
            // ================================================ B-task
            const int64_t r = round - LAG;
            if (r < 0 || r >= nrec) continue;
            const int b = o - TA;
            const int slot = (int)(r % S);
            const int gen = (int)(r / S);
            const int k0 = b * ROWS;
            if (tid == 0) wait_geq(doneA + slot, (gen + 1) * TA);
            __syncthreads();
            PIPE_T(5)
            BFFT_STRESS_DELAY(3);
            const float2* src = ring + (int64_t)slot * N + (int64_t)k0 * N2;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int i = tid + u * NT;  // linear index in the ROWS x N2 tile
                const int row = i / N2, e = i - (i / N2) * N2;
                sm[SwzColLayout<ROWS>::at(e, row)] = ld_l2(src + i);
            }
            __syncthreads();
            for (int i = tid; i < ROWS * N2 * 8 / 128; i += NT)
                l2_discard128(reinterpret_cast<const char*>(src) + 128 * i);  // dead intermediate: no write-back
            if (tid == 0) red_release_gpu(doneB + slot, 1);  // slot rows read: A-tasks may reuse
            PIPE_T(6)
            BFFT_STRESS_DELAY(4);
            const int col = tid % ROWS, t = tid / ROWS;
            float2 v[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) v[s] = sm[SwzColLayout<ROWS>::at(t + s * TB2, col)];
            fft_engine<N2>(v, t, sm, [&](int e) { return ColLayout<ROWS>::at(e, col); }, tabB);
            float2* dst = out + r * N + k0 + col + (int64_t)t * N1;
#pragma unroll
            for (int q = 0; q < 16; ++q)
                st_stream(dst + (int64_t)q * TB2 * N1, INV ? scale_conj(v[q], scale) : v[q]);
            PIPE_T(7)
            PIPE_ACC(5, 0, 5) PIPE_ACC(6, 5, 6) PIPE_ACC(7, 6, 7) PIPE_ACC(8, 0, 7)
#ifdef BFFT_PIPE_PROF
            if (tid == 0) atomicAdd(&g_pipe_prof[11], 1ull);
#endif
        }
    }
    pipe_exit_reset(ctr, S);
}

}  // namespace bfft

namespace bfft {

// ======================================================================
// k_pipe2: the same task graph as k_pipe, warp-specialised so that no
// memory latency sits on the compute warps' critical path.
//   producer warp : claims tasks, waits for their dependencies, and loads
//                   each task's tile into an NSTAGE-deep shared-memory ring
//                   with TMA (A-tile: one tensor box per 256 rows of the
//                   record's column tile; B-tile: one bulk copy per ring row
//                   into a padded row) completing on full[stage];
//   compute warps : FFT the staged tile (exchanges inside the same stage
//                   buffer, consumer-only named barrier), apply twiddles,
//                   store, arrive done[stage];
//   release warp  : once a task's stores are issued, publishes it with
//                   fence.acq_rel.gpu + red (the ~us fence latency stays off
//                   the compute warps), then frees the stage.
// ======================================================================
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_gpu(int* p, int v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int N1, int N2, int COLS, int ROWS, int NSTAGE, int PP = 16, int NGRP = 1, int H = 1>
struct Pipe2Cfg {
    static constexpr int N = N1 * N2;
    static constexpr int NTC = COLS * Sched<N1, PP>::T;        // compute threads per group
    static_assert(ROWS * Sched<N2, PP>::T == NTC, "A and B tasks use the same compute warps");
    static_assert(Sched<N1, PP>::P == PP && Sched<N2, PP>::P == PP, "N1, N2 >= PP");
    static_assert(NTC % 32 == 0, "whole compute warps");
    static_assert(NGRP >= 1 && NGRP % H == 0 && NGRP / H <= NSTAGE,
                  "every group sequence's end marker needs a stage of its own");
    static constexpr int NSEQ = NGRP / H;                        // task sequences (H groups share a task)
    static constexpr int NT = NTC * NGRP + 64;                   // + producer warp + release warp
    static constexpr int TA = N2 / (H * COLS), TB = N1 / (H * ROWS);   // tasks per record
    static constexpr int RSTRIDE = N2 + 2;                       // padded B-tile row (16-B multiple)
    using LayA = PadColLayout<COLS, Sched<N1, PP>::R0>;           // exchange layouts (fft_device.cuh)
    using LayB = PadColLayout<ROWS, Sched<N2, PP>::R0>;
    // a task's H halves exchange in disjoint regions of its stage (16-entry aligned)
    static constexpr int REG_A = (LayA::size(N1) + 15) / 16 * 16, REG_B = (LayB::size(N2) + 15) / 16 * 16;
    static constexpr int TILE_A0 = H * REG_A > H * COLS * N1 ? H * REG_A : H * COLS * N1;
    static constexpr int TILE_B0 = H * ROWS * RSTRIDE > H * REG_B ? H * ROWS * RSTRIDE : H * REG_B;
    static constexpr int TILE_A = H * COLS * N1, TILE_B = H * ROWS * RSTRIDE;   // entries the copies bring
    // stage stride rounded to 128 bytes: TMA writes shared memory at 128-byte aligned addresses
    static constexpr int TILE = ((TILE_A0 > TILE_B0 ? TILE_A0 : TILE_B0) + 15) / 16 * 16;
    static constexpr int BOXR = N1 < 256 ? N1 : 256;             // TMA box rows
    static constexpr int TB2 = Sched<N2, PP>::T;
    // split four-step twiddles (TW_SPLIT): B-side tables in shared memory,
    // T[q][s] = W_{PP^2}^{q s} (rows padded to PP + 1) and WB0[t][q] = W_{N2 PP}^{t q}
    static constexpr int TW_T = PP * (PP + 1), TW_B0 = TB2 * PP;
    static constexpr size_t OFF_TW = sizeof(float2) * (size_t)TILE * NSTAGE + 64 * NSTAGE + 128;
    static constexpr size_t SMEM_TW = sizeof(float2) * (size_t)(TW_T + TW_B0);
    static constexpr size_t SMEM = OFF_TW;   // + SMEM_TW with TW_SPLIT (pipe2_smem)
    static constexpr int MINB_RAW = 65536 / (NT * (PP == 16 ? 64 : 96));
    static constexpr int MINB = MINB_RAW < 1 ? 1 : (MINB_RAW > 8 ? 8 : MINB_RAW);
};

// How k_pipe2 applies the four-step twiddle W_N^{n2 k1}:
//   TW_TREE  : A-side, products of log2 PP factors from the plan's two-level table;
//   TW_TABLE : A-side, one load per element from a full [k1][n2] table (N entries);
//   TW_SPLIT : W_N^{n2 k1} = W_N^{n2 t} * W_{N2 PP}^{n2 q} with k1 = t + TA1 q
//              (t = the A thread's index, q = its register index).  A multiplies
//              by its one per-thread factor W_N^{n2 t}, loaded before its column
//              FFT; B (which holds n2 = t' + TB2 s) multiplies by
//              W_{N2 PP}^{t' q} * W_{PP^2}^{q s} from two small shared-memory
//              tables — no global load on either task's critical path.
enum { TW_TREE = 0, TW_TABLE = 1, TW_SPLIT = 2 };
template <int N1, int N2, int COLS, int ROWS, int NSTAGE, int PP, int TWM, int NGRP = 1, int H = 1>
constexpr size_t pipe2_smem() {
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP, H>;
    return CF::SMEM + (TWM == TW_SPLIT ? CF::SMEM_TW : 0);
}

struct PipeTask {
    long long rec;  // record index
    int kind;       // 0 = A, 1 = B, 2 = end
    int tile;       // column tile (A) or row tile (B)
};

// NGRP compute groups (NTC threads each, own named barrier) take tasks
// k = g, g + NGRP, ... of the CTA's claimed sequence, each computing in the
// stage its task was loaded into: NGRP tasks compute concurrently per CTA
// while the producer stages the next (NSTAGE >= NGRP + 1 to overlap).
// With H > 1 a task is H adjacent tiles (an A-task H*COLS columns — one
// H*COLS*8-byte DRAM run per row; a B-task H*ROWS ring rows) staged together
// and computed by H groups, one tile each: groups g = H j .. H j + H - 1 take
// tasks k = j, j + NGRP / H, ...
// RS = 1 (real records of n = 2N samples, forward; H = 2): the real split
// X[k] = E + W_n^k O (E = (Z[k] + conj Z[N-k])/2, O = (Z[k] - conj Z[N-k])/(2i),
// SURVEY.md §8(f) NEXT-1) is fused into the B-task.  The partner of k = k1 + N1 k2
// is N - k = (N1 - k1) + N1 (N2 - 1 - k2), so a B-task takes rows k1 = tile*ROWS + c
// (half 0) and their mirrors N1 - k1 (half 1; the mirror of row 0 is row 0 itself,
// and row N1/2 — its own mirror — takes that slot), exchanges the transformed rows
// through the stage and stores the packed half spectrum (X[0] slot = (X[0], X[N])).
// RS = 2 (inverse): the C2R merge is fused into the A-task's read (rt.src holds
// the packed half spectra for the partner reads).
template <int N1, int N2, int COLS, int ROWS, bool INV, int NSTAGE, int PP = 16, int TWM = TW_TREE, int NGRP = 1,
          int CB = 1, bool PF = false, int H = 1, int RS = 0>
__global__ void __launch_bounds__(Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP, H>::NT,
                                  Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP, H>::MINB)
k_pipe2(const __grid_constant__ CUtensorMap tmap_in, float2* __restrict__ out, float2* __restrict__ ring,
        int64_t nrec, int* __restrict__ ctr, int S, int LAG, float scale, const float2* __restrict__ w_hi,
        const float2* __restrict__ w_lo, int w_lb, const float* __restrict__ window, RealTw rt) {
    // window: optional per-sample weights w[0..N) applied as the A-tile is read
    // (STFT frames: tmap_in then strides records by the hop)
    // rt: W_n^k (n = 2N) for RS = 1, else unused
    static_assert(RS == 0 || (RS == 1 && H == 2 && !INV) || (RS == 2 && INV),
                  "fused real split: forward over mirrored half tiles (1), merge on load: inverse (2)");
    using CF = Pipe2Cfg<N1, N2, COLS, ROWS, NSTAGE, PP, NGRP, H>;
    constexpr int LPP = ilog2(PP);
    constexpr int N = CF::N, TA = CF::TA, TB = CF::TB, NTC = CF::NTC, TILE = CF::TILE, RSTRIDE = CF::RSTRIDE;
    constexpr int TA1 = Sched<N1, PP>::T, TB2 = Sched<N2, PP>::T;
    // B-task row of half h, slot c (RS: half 1 holds the mirrors, see above)
    auto brow = [](int tile, int h, int c) -> int {
        if constexpr (RS == 1) {
            if (h == 0) return tile * ROWS + c;
            const int m = N1 - tile * ROWS - c;
            return m == N1 ? N1 / 2 : m;
        } else {
            return (tile * H + h) * ROWS + c;
        }
    };
    extern __shared__ __align__(128) float2 sm[];
    PipeTask* info = reinterpret_cast<PipeTask*>(sm + (size_t)TILE * NSTAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(info + NSTAGE);   // full | empty | done | sfree
    const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + NSTAGE), done0 = smem_addr(bars + 2 * NSTAGE);
    const uint32_t sfree0 = smem_addr(bars + 3 * NSTAGE);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int WP = NGRP * NTC / 32, WR = WP + 1;  // producer, release warps
    int* doneA = ctr + 1;
    int* doneB = ctr + 1 + S;
    const int64_t per_round = TA + TB;
    const int64_t total = (nrec + LAG) * per_round;

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);       // the release warp frees a stage
            mbar_init(done0 + 8 * i, H * NTC / 32); // one arrival per compute warp: stores issued
            mbar_init(sfree0 + 8 * i, H * NTC / 32);// one arrival per compute warp: stage read for the last time
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == WP) {
        // ============================================== producer
        // lane 0 claims, waits and arms the stage; the B-tile's ROWS row copies
        // are spread over the warp's lanes
        uint32_t k = 0;
        int ends = 0;   // end markers staged (one per compute group)
        const uint64_t pol_stream = policy_evict_first();
        // Tasks are claimed CB at a time (one atomic per batch, the next batch's
        // claim in flight while this one is staged); consecutive tasks mostly
        // share a record, so a dependency already seen satisfied is not waited
        // for again (the last (counter, value) acquired is cached).
        long long base = 0, nextb = 0;
        int sub = 0;
        const int* dep_ptr = nullptr;
        int dep_seen = 0;
        auto decode = [&](long long task, PipeTask& t) -> bool {   // false: not a task of this launch
            if (task >= total) {
                t.kind = 2;
                t.rec = 0;
                t.tile = 0;
                return true;
            }
            const long long round = task / per_round;
            const int o = (int)(task - round * per_round);
            if (o < TA) {
                t.kind = 0;
                t.rec = round;
                t.tile = o;
                return round < nrec;
            }
            t.kind = 1;
            t.rec = round - LAG;
            t.tile = o - TA;
            return t.rec >= 0 && t.rec < nrec;
        };
        if (lane == 0) {
            base = atomicAdd(ctr, CB);
            if (base < total) nextb = atomicAdd(ctr, CB);
        }
        for (;;) {
            PipeTask d;
            bool valid = true;
            if (lane == 0) {
                const long long task = base + sub;
                if (++sub == CB) {
                    sub = 0;
                    base = nextb;
                    if (base < total) nextb = atomicAdd(ctr, CB);
                }
                valid = decode(task, d);
                if constexpr (PF) {
                    // pull the next A-tile from HBM into L2 while this task waits for its stage
                    PipeTask nx;
                    if (valid && d.kind != 2 && decode(base + sub, nx) && nx.kind == 0) {
#pragma unroll 1
                        for (int r0 = 0; r0 < N1; r0 += CF::BOXR)
                            tma_prefetch_3d(&tmap_in, nx.tile * H * COLS, r0, (int)nx.rec);
                    }
                }
            }
            valid = __shfl_sync(0xffffffffu, valid, 0);
            if (!valid) continue;
            d.kind = __shfl_sync(0xffffffffu, d.kind, 0);
            d.rec = __shfl_sync(0xffffffffu, d.rec, 0);
            d.tile = __shfl_sync(0xffffffffu, d.tile, 0);
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            const uint32_t fb = full0 + 8 * s;
            if (lane == 0) {
                BFFT_STRESS_DELAY(10);
                if (u > 0) mbar_wait(empty0 + 8 * s, (u - 1) & 1);
                if (d.kind == 2) {
                    info[s] = d;
                    mbar_arrive(fb);
                } else {
                    const int slot = (int)(d.rec % S), gen = (int)(d.rec / S);
#ifndef BFFT_PIPE_NODEPS  // (experiments only: tools/exp measures the kernel without its waits)
                    const int* dp = nullptr;
                    int target = 0;
                    if (d.kind == 0) {
#ifndef BFFT_PIPE_NOWAR   // (mutation experiment only: tools/exp/stress_mutant.py)
                        if (gen > 0) dp = doneB + slot, target = gen * TB;   // ring slot free (WAR)
#endif
                    } else {
                        dp = doneA + slot, target = (gen + 1) * TA;          // column FFTs published
                    }
                    if (dp && !(dp == dep_ptr && target <= dep_seen)) {
                        dep_seen = wait_geq_v(dp, target);
                        dep_ptr = dp;
                        // generic ring stores acquired here -> this thread's later bulk-copy reads
                        if (d.kind == 1) fence_proxy_async_global();
                    }
#endif
                    info[s] = d;
                    mbar_expect_tx(fb, (uint32_t)((d.kind == 0 ? CF::TILE_A : H * ROWS * N2) * sizeof(float2)));
                }
            }
            if (d.kind == 2) {
                if (++ends == CF::NSEQ) break;
                ++k;
                continue;
            }
            __syncwarp();
            float2* stage = sm + (size_t)s * TILE;
            if (d.kind == 0) {
                if (lane == 0) {
#pragma unroll 1
                    for (int r0 = 0; r0 < N1; r0 += CF::BOXR)
                        tma_load_3d_hint(smem_addr(stage + r0 * H * COLS), &tmap_in, d.tile * H * COLS, r0,
                                         (int)d.rec, fb, pol_stream);
                }
            } else {
                const int slot = (int)(d.rec % S);
                const float2* src = ring + (int64_t)slot * N;
                for (int j = lane; j < H * ROWS; j += 32)
                    bulk_g2s(smem_addr(stage + j * RSTRIDE), src + (int64_t)brow(d.tile, j / ROWS, j % ROWS) * N2,
                             N2 * sizeof(float2), fb);
            }
            ++k;
        }
    } else if (warp == WR) {
        // ============================================== release
        if (lane == 0) {
            for (uint32_t k = 0;; ++k) {
                const uint32_t s = k % NSTAGE, u = k / NSTAGE;
                mbar_wait(full0 + 8 * s, u & 1);
                const PipeTask d = info[s];
                if (d.kind == 2) break;
                P2_T(rt0)
                BFFT_STRESS_DELAY(11);
                mbar_wait(sfree0 + 8 * s, u & 1);
                mbar_arrive(empty0 + 8 * s);   // stage reusable: its last exchange has been read
                mbar_wait(done0 + 8 * s, u & 1);
                P2_T(rt1)
                BFFT_STRESS_DELAY(12);
#ifndef BFFT_PIPE_NODEPS
#ifndef BFFT_PIPE_REDREL
                fence_acq_rel_gpu();            // their stores, observed through done[s], become visible
#endif
#endif
                const int slot = (int)(d.rec % S);
#ifdef BFFT_PIPE_REDREL
                red_release_gpu((d.kind == 0 ? doneA : doneB) + slot, 1);
#else
                red_relaxed_gpu((d.kind == 0 ? doneA : doneB) + slot, 1);
#endif
                P2_T(rt2)
                P2_ACC(16, rt0, rt1)
                P2_ACC(17, rt1, rt2)
            }
        }
    } else {
        // ============================================== compute warps
        const TwoLevel W{w_hi, w_lo, w_lb, (uint32_t)(N - 1)};
        const ConstTw<N1, PP> tabA{};
        const ConstTw<N2, PP> tabB{};
        const int grp = warp / (NTC / 32);
        const int gtid = tid - grp * NTC;   // thread index within the group
        const NamedBarrier bar{1 + grp, NTC};
        const int half = grp % H;           // which of its task's H tiles the group computes
        const NamedBarrier pair{2 + NGRP + grp / H, H * NTC};   // the task's H groups: inputs read
        float2* tw_t = reinterpret_cast<float2*>(reinterpret_cast<char*>(sm) + CF::OFF_TW);   // T[q][s]
        float2* tw_b0 = tw_t + CF::TW_T;                                                       // WB0[t][q]
        if constexpr (TWM == TW_SPLIT) {
            // w_lo = WB0 [TB2][PP] then T [PP][PP]: copy into shared memory (T rows padded)
            for (int i = tid; i < CF::TW_B0; i += NGRP * NTC) tw_b0[i] = w_lo[i];
            for (int i = tid; i < PP * PP; i += NGRP * NTC) tw_t[(i / PP) * (PP + 1) + i % PP] = w_lo[CF::TW_B0 + i];
            const NamedBarrier all{1 + NGRP, NGRP * NTC};
            all();
        }
        for (uint32_t k = grp / H;; k += CF::NSEQ) {
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            P2_T(ct0)
            mbar_wait(full0 + 8 * s, u & 1);
            P2_T(ct1)
            BFFT_STRESS_DELAY(13);
            const PipeTask d = info[s];
            if (d.kind == 2) break;
            float2* stage = sm + (size_t)s * TILE;
            const int64_t r = d.rec;
            const int slot = (int)(r % S);
            float2 v[PP];
            if (d.kind == 0) {
                // ---------------- A: columns n2 of record r, FFT over n1, twiddle, -> ring
                const int col = gtid % COLS, t = gtid / COLS;
                const int n2 = (d.tile * H + half) * COLS + col;
                float2 f[LPP], w0;
                if constexpr (TWM == TW_TREE) {
#pragma unroll
                    for (int i = 0; i < LPP; ++i) f[i] = W((uint32_t)n2 * (uint32_t)(TA1 << i));
                    w0 = W((uint32_t)n2 * (uint32_t)t);
                } else if constexpr (TWM == TW_SPLIT) {
                    w0 = __ldg(w_hi + t * N2 + n2);   // W_N^{n2 t}: in flight during the column FFT
                }
                if constexpr (RS == 2) {
                    // C2R merge on load: Z[k] = E + i O, E = (X[k] + conj X[N-k]) / 2,
                    // O = (X[k] - conj X[N-k]) conj(W_n^k) / 2 for k = n1 N2 + n2; the
                    // partner N - k = (N1 - 1 - n1) N2 + (N2 - n2) (n2 > 0) or
                    // (N1 - n1) N2 (n2 = 0) is read from L2 / HBM (the mirrored
                    // column tile's own A-task stages it too).  W_n^k = W_n^{n2 + N2 t}
                    // W_{2PP}^q for n1 = t + TA1 q.
                    const float2* xr = rt.src + r * N;
                    const float2 a = rt((int)n2 + N2 * t);
#pragma unroll
                    for (int q = 0; q < PP; ++q) {
                        const int n1 = t + q * TA1;
                        const float2 x = stage[n1 * (H * COLS) + half * COLS + col];
                        const int pk = n2 ? (N1 - 1 - n1) * N2 + (N2 - n2) : ((N1 - n1) & (N1 - 1)) * N2;
                        float2 z;
                        if (n2 == 0 && n1 == 0) {
                            z = make_float2(0.5f * (x.x + x.y), 0.5f * (x.x - x.y));   // (E[0], O[0])
                        } else {
                            const float2 y = __ldg(xr + pk);
                            const float2 e = __fmul2_rn(cadd(x, conjf2(y)), make_float2(0.5f, 0.5f));
                            const float2 o = cmul(__fmul2_rn(csub(x, conjf2(y)), make_float2(0.5f, 0.5f)),
                                                  conjf2(cmul(a, c_rw64[q * (32 / PP)])));
                            z = cadd(e, mul_pi(o));
                        }
                        v[q] = conjf2(z);   // INV
                    }
                } else if (window) {
#pragma unroll
                    for (int q = 0; q < PP; ++q) {
                        const float w = __ldg(window + (t + q * TA1) * N2 + n2);
                        const float2 x = stage[(t + q * TA1) * (H * COLS) + half * COLS + col];
                        v[q] = INV ? make_float2(x.x * w, -x.y * w) : make_float2(x.x * w, x.y * w);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PP; ++q) {
                        const float2 x = stage[(t + q * TA1) * (H * COLS) + half * COLS + col];
                        v[q] = INV ? conjf2(x) : x;
                    }
                }
                if constexpr (H > 1) pair();   // the halves' exchange regions overlap both halves' inputs
                float2* xch = stage + half * CF::REG_A;
#ifndef BFFT_PIPE_NOCOMPUTE  // (experiments only: data movement without the FFT)
                fft_engine<N1, PP>(v, t, xch, [&](int e) { return CF::LayA::at(e, col); }, tabA, bar);
#endif
#ifndef BFFT_PIPE_NOFENCE
                fence_proxy_async_smem();   // last generic access of the stage: before its next TMA refill
#endif
                __syncwarp();
                if (lane == 0) mbar_arrive(sfree0 + 8 * s);   // the producer may refill the stage now
#ifdef BFFT_PIPE_NOTW   // (experiments only: the kernel without its four-step twiddle; results wrong)
                if constexpr (true) {
                } else
#endif
                if constexpr (TWM == TW_SPLIT) {
#pragma unroll
                    for (int q = 0; q < PP; ++q) v[q] = cmul(v[q], w0);   // the W_N^{n2 t} part
                } else if constexpr (TWM == TW_TABLE) {
                    // W_N^{n2 k1} from the full [k1][n2] table (w_hi): one coalesced load per element
                    const float2* wt = w_hi + (int64_t)t * N2 + n2;
#pragma unroll
                    for (int q = 0; q < PP; ++q) v[q] = cmul(v[q], __ldg(wt + (int64_t)q * TA1 * N2));
                } else {
                    float2 w[PP];
                    w[0] = w0;
                    v[0] = cmul(v[0], w0);
#pragma unroll
                    for (int q = 1; q < PP; ++q) {
                        const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                        w[q] = cmul(w[q & (q - 1)], f[lb]);
                        v[q] = cmul(v[q], w[q]);
                    }
                }
                BFFT_STRESS_DELAY(14);
                float2* dst = ring + (int64_t)slot * N + n2 + (int64_t)t * N2;
#pragma unroll
                for (int q = 0; q < PP; ++q) dst[(int64_t)q * TA1 * N2] = v[q];
            } else {
                // ---------------- B: rows k1 of record r, FFT over n2, -> X[k1 + N1 k2]
                const int col = gtid % ROWS, t = gtid / ROWS;
                const int k1 = brow(d.tile, half, col);
                const float2* srow = stage + (half * ROWS + col) * RSTRIDE;
                {   // the tile's ring rows are staged: drop them from L2 (no write-back)
                    constexpr int LPR = N2 * 8 / 128;   // 128-byte lines per row
                    const char* base = reinterpret_cast<const char*>(ring + (int64_t)slot * N);
                    for (int i = gtid; i < ROWS * LPR; i += NTC)
                        l2_discard128(base + ((int64_t)brow(d.tile, half, i / LPR) * N2) * 8 + 128 * (i % LPR));
                }
                if constexpr (TWM == TW_SPLIT) {
                    // the W_{N2 PP}^{n2 qa} part, n2 = t + TB2 s, qa = k1 / TA1, applied
                    // as the elements arrive, 8 at a time (a compiler barrier keeps the
                    // loads from all being hoisted: v plus every factor would spill)
                    const int qa = k1 / TA1;
                    const float2 wb = tw_b0[t * PP + qa];
                    const float2* trow = tw_t + qa * (PP + 1);
#pragma unroll
                    for (int q0 = 0; q0 < PP; q0 += 8) {
#pragma unroll
                        for (int q = q0; q < q0 + 8; ++q)
                            v[q] = cmul(srow[t + q * TB2], cmul(wb, trow[q]));
                        asm volatile("" ::: "memory");
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PP; ++q) v[q] = srow[t + q * TB2];
                }
                if constexpr (H > 1) pair();
                float2* xch = stage + half * CF::REG_B;
#ifndef BFFT_PIPE_NOCOMPUTE
                fft_engine<N2, PP>(v, t, xch, [&](int e) { return CF::LayB::at(e, col); }, tabB, bar);
#endif
                float2* dst = out + r * N + k1 + (int64_t)t * N1;
                if constexpr (RS == 1) {
                    // the real split: both halves' rows through the stage, then X[k] = E + W_n^k O
                    pair();   // both groups are done with their exchange regions
                    float2* zrow = stage + (half * ROWS + col) * RSTRIDE;
#pragma unroll
                    for (int q = 0; q < PP; ++q) zrow[t + q * TB2] = v[q];
                    pair();
                    const bool self = d.tile == 0 && col == 0;   // rows 0 and N1/2: their own mirrors
                    const float2* prow = self ? zrow : stage + ((1 - half) * ROWS + col) * RSTRIDE;
                    const float2 a = rt(k1 + N1 * t);            // W_n^{k1 + N1 t}; W_n^{N1 TB2 q} = W_{2PP}^q
#pragma unroll
                    for (int q = 0; q < PP; ++q) {
                        const int k2 = t + q * TB2;
                        const int pk2 = (self && half == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
                        const float2 z = v[q], c = prow[pk2];
                        float2 x;
                        if (self && half == 0 && k2 == 0) {
                            x = make_float2(z.x + z.y, z.x - z.y);                     // (X[0], X[N])
                        } else {
                            const float2 e = __fmul2_rn(cadd(z, conjf2(c)), make_float2(0.5f, 0.5f));
                            const float2 o = mul_mi(__fmul2_rn(csub(z, conjf2(c)), make_float2(0.5f, 0.5f)));
                            x = cadd(e, cmul(o, cmul(a, c_rw64[q * (32 / PP)])));
                        }
                        st_stream(dst + (int64_t)q * TB2 * N1, x);
                    }
#ifndef BFFT_PIPE_NOFENCE
                    fence_proxy_async_smem();
#endif
                    __syncwarp();
                    if (lane == 0) mbar_arrive(sfree0 + 8 * s);
                } else {
#ifndef BFFT_PIPE_NOFENCE
                fence_proxy_async_smem();   // last generic access of the stage: before its next bulk refill
#endif
                __syncwarp();
                if (lane == 0) mbar_arrive(sfree0 + 8 * s);   // the producer may refill the stage now
#pragma unroll
                for (int q = 0; q < PP; ++q)
                    st_stream(dst + (int64_t)q * TB2 * N1, INV ? scale_conj(v[q], scale) : v[q]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(done0 + 8 * s);
            P2_T(ct2)
            if (tid == 0) {
                P2_ACC(18 + d.kind * 2, ct0, ct1)
                P2_ACC(19 + d.kind * 2, ct1, ct2)
#ifdef BFFT_PIPE_PROF
                atomicAdd(&g_pipe_prof[22 + d.kind], 1ull);
#endif
            }
        }
    }
    pipe_exit_reset(ctr, S);
}

}  // namespace bfft
