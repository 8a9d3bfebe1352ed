// fft_pipe3.cuh — k_pipe3: the pipelined four-step task graph of k_pipe /
// k_pipe2 (fft_pipe.cuh: same A/B tasks, rounds, LAG, ring and dependency
// counters) with more compute warps per SM.
//
// k_pipe2 holds a staged tile for the whole life of its task (the column/row
// FFT exchanges in place), so shared memory (six 32 KiB tiles per SM at 2^16)
// caps an SM at ~12 compute warps and the FFT engine is latency-bound
// (profiles/r01_final_pipe2_bench_ncu.md: 36 % issue, 43 % FMA pipe).  Here a
// stage is held only until its task's elements are in registers:
//   producer warp : claims task k, waits until stage k % NS is empty and the
//                   task's dependencies are met, publishes the descriptor
//                   (seq = k) and loads the tile (TMA / bulk) onto full[s];
//   G compute groups (NTC threads each, own exchange buffer and named
//                   barrier): group g runs tasks k = g, g + G, ...: waits for
//                   the descriptor, then full[s]; reads its elements into
//                   registers and frees the stage at once (empty[s]); FFTs in
//                   its private exchange buffer; stores; then pushes the
//                   completed task onto its completion FIFO;
//   release warp  : drains the FIFOs — one fence.acq_rel.gpu per batch, then
//                   red.relaxed.gpu on each task's doneA / doneB counter.
// Shared memory = NS staging tiles + G exchange buffers, e.g. 2^16: 3 x 33 KiB
// + 4 x 32 KiB (16 compute warps per SM instead of 12); 2^20: 1 x 64 KiB +
// 2 x 64 KiB (16 instead of 8).
//
// Memory model: the stage is only read by the groups (generic loads) before
// the producer refills it with TMA / bulk copies; the mbarrier arrive (empty)
// -> wait -> copy chain orders that write-after-read, as in CUTLASS's TMA
// pipelines (no proxy fence needed).  Ring data written with generic stores by
// other CTAs is read with bulk copies: the producer issues
// fence.proxy.async.global after acquiring the dependency counter.
//
// Deadlock freedom is k_pipe's argument unchanged: the producer blocks on a
// task's dependencies only while the tasks its CTA already holds are staged
// or computing, and those finish without waiting on anything outside the
// CTA; the release warp never waits on a group, and a group waits for FIFO
// space only on the release warp.
#pragma once

#include "fft_pipe.cuh"

namespace bfft {

template <int N1, int N2, int COLS, int ROWS, int NS, int G, int PP = 32>
struct Pipe3Cfg {
    static constexpr int N = N1 * N2;
    static constexpr int NTC = COLS * Sched<N1, PP>::T;        // threads per compute group
    static_assert(ROWS * Sched<N2, PP>::T == NTC, "A and B tasks use the same group size");
    static_assert(Sched<N1, PP>::P == PP && Sched<N2, PP>::P == PP, "N1, N2 >= PP");
    static_assert(NTC % 32 == 0, "whole compute warps");
    static_assert(G >= 1 && G <= 14 && NS >= 1, "named barriers 1..G");
    static constexpr int NT = NTC * G + 64;                      // + producer warp + release warp
    static constexpr int TA = N2 / COLS, TB = N1 / ROWS;
    static constexpr int RSTRIDE = N2 + 2;                       // padded B-tile row (16-B multiple)
    static constexpr int TILE_A = COLS * N1, TILE_B = ROWS * RSTRIDE;
    // stage stride rounded to 128 bytes: TMA writes shared memory at 128-byte aligned addresses
    static constexpr int TILE = ((TILE_A > TILE_B ? TILE_A : TILE_B) + 15) / 16 * 16;
    static constexpr int XA = COLS * N1, XB = ROWS * N2;         // ColLayout exchange buffers
    static constexpr int XTILE = XA > XB ? XA : XB;
    static constexpr int BOXR = N1 < 256 ? N1 : 256;             // TMA box rows
    static constexpr int FIFO = 32;                              // completions per group
    static constexpr size_t TILES_BYTES = sizeof(float2) * ((size_t)TILE * NS + (size_t)XTILE * G);
    // control block: info[NS] (32 B) | full[NS] | empty[NS] | end_k | cnt[G] | rel[G] | exited[G] | fifo[G][FIFO]
    static constexpr size_t CTRL_BYTES = 32 * NS + 16 * NS + 16 + 12 * G + 4 * G * FIFO + 64;
    static constexpr size_t SMEM = TILES_BYTES + CTRL_BYTES;
    static constexpr int MINB = 2 * SMEM <= 227 * 1024 ? 2 : 1;   // two CTAs per SM when they fit
};

struct PipeTask3 {
    long long rec;  // record index
    int kind;       // 0 = A, 1 = B, 2 = end
    int tile;       // column tile (A) or row tile (B)
    int seq;        // task index k this descriptor belongs to
    int pad[3];
};

__device__ __forceinline__ int ld_acquire_cta_s(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_s(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_s(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

template <int N1, int N2, int COLS, int ROWS, bool INV, int NS, int G, int PP = 32, int CB = 4, bool PF = false>
__global__ void __launch_bounds__(Pipe3Cfg<N1, N2, COLS, ROWS, NS, G, PP>::NT, Pipe3Cfg<N1, N2, COLS, ROWS, NS, G, PP>::MINB)
k_pipe3(const __grid_constant__ CUtensorMap tmap_in, float2* __restrict__ out, float2* __restrict__ ring,
        int64_t nrec, int* __restrict__ ctr, int S, int LAG, float scale, const float2* __restrict__ w_hi,
        const float2* __restrict__ w_lo, int w_lb, const float* __restrict__ /*window: k_pipe2 only, pass null*/,
        RealTw /*k_pipe2 only*/) {
    using CF = Pipe3Cfg<N1, N2, COLS, ROWS, NS, G, PP>;
    constexpr int LPP = ilog2(PP);
    constexpr int N = CF::N, TA = CF::TA, TB = CF::TB, NTC = CF::NTC, TILE = CF::TILE, RSTRIDE = CF::RSTRIDE;
    constexpr int TA1 = Sched<N1, PP>::T, TB2 = Sched<N2, PP>::T, FIFO = CF::FIFO;
    extern __shared__ __align__(128) float2 sm[];
    float2* xbuf0 = sm + (size_t)TILE * NS;
    PipeTask3* info = reinterpret_cast<PipeTask3*>(xbuf0 + (size_t)CF::XTILE * G);
    uint64_t* bars = reinterpret_cast<uint64_t*>(info + NS);    // full[NS] | empty[NS]
    int* end_k = reinterpret_cast<int*>(bars + 2 * NS);
    int* cnt = end_k + 4;        // completions pushed, per group
    int* rel = cnt + G;          // completions released, per group
    int* exited = rel + G;       // group finished, per group
    int* fifo = exited + G;      // [G][FIFO] completed (kind << 30 | slot)
    const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + NS);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int WP = G * NTC / 32, WR = WP + 1;  // producer, release warps
    int* doneA = ctr + 1;
    int* doneB = ctr + 1 + S;
    const int64_t per_round = TA + TB;
    const int64_t total = (nrec + LAG) * per_round;

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, NTC / 32);  // one arrival per warp of the consuming group
            info[i].seq = -1;
        }
        *end_k = 0x7fffffff;
        for (int g = 0; g < G; ++g) cnt[g] = rel[g] = exited[g] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == WP) {
        // ============================================== producer
        // Tasks are claimed CB at a time (one atomic per batch; consecutive tasks
        // usually share a record, so its dependency is checked once: the last
        // satisfied (counter, value) pair is cached).
        uint32_t k = 0;
        const uint64_t pol_stream = policy_evict_first();
        long long base = 0, nextb = 0;
        int sub = 0;
        const int* dep_ptr = nullptr;
        int dep_seen = 0;
        if (lane == 0) {
            base = atomicAdd(ctr, CB);
            if (base < total) nextb = atomicAdd(ctr, CB);  // the next batch is claimed while this one is staged
        }
        for (;;) {
            PipeTask3 d;
            bool valid = true;
            if (lane == 0) {
                const long long task = base + sub;
                if (++sub == CB) {
                    sub = 0;
                    base = nextb;
                    if (base < total) nextb = atomicAdd(ctr, CB);
                }
                if (task >= total) {
                    d.kind = 2;
                    d.rec = 0;
                    d.tile = 0;
                } else {
                    const long long round = task / per_round;
                    const int o = (int)(task - round * per_round);
                    if (o < TA) {
                        d.kind = 0;
                        d.rec = round;
                        d.tile = o;
                        valid = round < nrec;
                    } else {
                        d.kind = 1;
                        d.rec = round - LAG;
                        d.tile = o - TA;
                        valid = d.rec >= 0 && d.rec < nrec;
                    }
                }
            }
            valid = __shfl_sync(0xffffffffu, valid, 0);
            if (!valid) continue;
            d.kind = __shfl_sync(0xffffffffu, d.kind, 0);
            if (d.kind == 2) {
                if (lane == 0) st_release_cta_s(end_k, (int)k);  // groups waiting for k' >= k leave
                break;
            }
            d.rec = __shfl_sync(0xffffffffu, d.rec, 0);
            d.tile = __shfl_sync(0xffffffffu, d.tile, 0);
            const uint32_t s = k % NS, u = k / NS;
            const uint32_t fb = full0 + 8 * s;
            if (lane == 0) {
                if (PF && d.kind == 0) {
                    // pull the A-tile from HBM into L2 while the stage is still busy
#pragma unroll 1
                    for (int r0 = 0; r0 < N1; r0 += CF::BOXR) tma_prefetch_3d(&tmap_in, d.tile * COLS, r0, (int)d.rec);
                }
                BFFT_STRESS_DELAY(20);
                if (u > 0) mbar_wait(empty0 + 8 * s, (u - 1) & 1);   // task k - NS read out of the stage
                const int slot = (int)(d.rec % S), gen = (int)(d.rec / S);
                const int* dp = nullptr;
                int target = 0;
                if (d.kind == 0) {
                    if (gen > 0) dp = doneB + slot, target = gen * TB;   // ring slot free (WAR)
                } else {
                    dp = doneA + slot, target = (gen + 1) * TA;          // column FFTs published
                }
                if (dp && !(dp == dep_ptr && target <= dep_seen)) {
                    dep_seen = wait_geq_v(dp, target);
                    dep_ptr = dp;
                    // generic ring stores acquired here -> this thread's later bulk-copy reads
                    if (d.kind == 1) fence_proxy_async_global();
                }
                info[s].rec = d.rec;
                info[s].kind = d.kind;
                info[s].tile = d.tile;
                st_release_cta_s(&info[s].seq, (int)k);
                mbar_expect_tx(fb, (uint32_t)((d.kind == 0 ? CF::TILE_A : ROWS * N2) * sizeof(float2)));
            }
            __syncwarp();
            float2* stage = sm + (size_t)s * TILE;
            if (d.kind == 0) {
                if (lane == 0) {
#pragma unroll 1
                    for (int r0 = 0; r0 < N1; r0 += CF::BOXR)
                        tma_load_3d_hint(smem_addr(stage + r0 * COLS), &tmap_in, d.tile * COLS, r0, (int)d.rec, fb,
                                         pol_stream);
                }
            } else {
                const int slot = (int)(d.rec % S);
                const float2* src = ring + (int64_t)slot * N + (int64_t)d.tile * ROWS * N2;
                for (int j = lane; j < ROWS; j += 32)
                    bulk_g2s(smem_addr(stage + j * RSTRIDE), src + (int64_t)j * N2, N2 * sizeof(float2), fb);
            }
            ++k;
        }
    } else if (warp == WR) {
        // ============================================== release
        if (lane == 0) {
            int done_g[G];
#pragma unroll
            for (int g = 0; g < G; ++g) done_g[g] = 0;
            int ns = 32;
            for (;;) {
                int c[G];
                bool any = false, all_exited = true;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int ex = ld_acquire_cta_s(exited + g);   // read before cnt: a group exits after its last push
                    c[g] = ld_acquire_cta_s(cnt + g);
                    any |= c[g] > done_g[g];
                    all_exited &= ex != 0;
                }
                if (!any) {
                    if (all_exited) break;
                    __nanosleep(ns);
                    ns = ns < 256 ? 2 * ns : ns;
                    continue;
                }
                ns = 32;
                BFFT_STRESS_DELAY(22);
                fence_acq_rel_gpu();   // the groups' stores, observed through cnt[], become visible
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    for (int i = done_g[g]; i < c[g]; ++i) {
                        const int e = ld_volatile_s(fifo + g * FIFO + i % FIFO);
                        red_relaxed_gpu(((e >> 30) == 0 ? doneA : doneB) + (e & 0x3fffffff), 1);
                    }
                    if (c[g] > done_g[g]) {
                        done_g[g] = c[g];
                        st_release_cta_s(rel + g, c[g]);   // FIFO entries reusable
                    }
                }
            }
        }
    } else {
        // ============================================== compute groups
        const int grp = warp / (NTC / 32);
        const int gt = tid - grp * NTC;   // thread index within the group
        float2* xbuf = xbuf0 + (size_t)grp * CF::XTILE;
        const TwoLevel W{w_hi, w_lo, w_lb, (uint32_t)(N - 1)};
        const ConstTw<N1, PP> tabA{};
        const ConstTw<N2, PP> tabB{};
        const NamedBarrier bar{1 + grp, NTC};
        int pushed = 0;
        for (uint32_t k = grp;; k += G) {
            const uint32_t s = k % NS, u = k / NS;
            // the descriptor for task k (its seq) or the end of the task stream
            bool end = false;
            for (;;) {
                if (ld_acquire_cta_s(&info[s].seq) == (int)k) break;
                if (ld_acquire_cta_s(end_k) <= (int)k) {
                    end = true;
                    break;
                }
                __nanosleep(20);
            }
            if (end) break;
            const long long r = info[s].rec;
            const int kind = info[s].kind, tile = info[s].tile;
            mbar_wait(full0 + 8 * s, u & 1);
            BFFT_STRESS_DELAY(21);
            float2* stage = sm + (size_t)s * TILE;
            const int slot = (int)(r % S);
            float2 v[PP];
            if (kind == 0) {
                // ---------------- A: columns n2 of record r, FFT over n1, twiddle, -> ring
                const int col = gt % COLS, t = gt / COLS;
                const int n2 = tile * COLS + col;
#pragma unroll
                for (int q = 0; q < PP; ++q) {
                    const float2 x = stage[(t + q * TA1) * COLS + col];
                    v[q] = INV ? conjf2(x) : x;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty0 + 8 * s);   // stage free: the producer refills it
                float2 f[LPP], w0;
#pragma unroll
                for (int i = 0; i < LPP; ++i) f[i] = W((uint32_t)n2 * (uint32_t)(TA1 << i));
                w0 = W((uint32_t)n2 * (uint32_t)t);
                fft_engine<N1, PP>(v, t, xbuf, [&](int e) { return ColLayout<COLS>::at(e, col); }, tabA, bar);
                float2 w[PP];
                w[0] = w0;
                v[0] = cmul(v[0], w0);
#pragma unroll
                for (int q = 1; q < PP; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                    w[q] = cmul(w[q & (q - 1)], f[lb]);
                    v[q] = cmul(v[q], w[q]);
                }
                float2* dst = ring + (int64_t)slot * N + n2 + (int64_t)t * N2;
#pragma unroll
                for (int q = 0; q < PP; ++q) dst[(int64_t)q * TA1 * N2] = v[q];
            } else {
                // ---------------- B: rows k1 of record r, FFT over n2, -> X[k1 + N1 k2]
                const int col = gt % ROWS, t = gt / ROWS;
                const int k0 = tile * ROWS;
#pragma unroll
                for (int q = 0; q < PP; ++q) v[q] = stage[col * RSTRIDE + t + q * TB2];
                __syncwarp();
                if (lane == 0) mbar_arrive(empty0 + 8 * s);
                {   // the tile's ring rows are staged: drop them from L2 (no write-back)
                    const char* rows = reinterpret_cast<const char*>(ring + (int64_t)slot * N + (int64_t)k0 * N2);
                    for (int i = gt; i < ROWS * N2 * 8 / 128; i += NTC) l2_discard128(rows + 128 * i);
                }
                fft_engine<N2, PP>(v, t, xbuf, [&](int e) { return ColLayout<ROWS>::at(e, col); }, tabB, bar);
                float2* dst = out + r * N + k0 + col + (int64_t)t * N1;
#pragma unroll
                for (int q = 0; q < PP; ++q)
                    st_stream(dst + (int64_t)q * TB2 * N1, INV ? scale_conj(v[q], scale) : v[q]);
            }
            bar();   // every store of the group's task is issued
            if (gt == 0) {
                if (pushed - ld_acquire_cta_s(rel + grp) >= FIFO) {
                    while (pushed - ld_acquire_cta_s(rel + grp) >= FIFO) __nanosleep(32);
                }
                fifo[grp * FIFO + pushed % FIFO] = (kind << 30) | slot;
                ++pushed;
                st_release_cta_s(cnt + grp, pushed);
            }
        }
        if (gt == 0) st_release_cta_s(exited + grp, 1);
    }
    pipe_exit_reset(ctr, S);
}

}  // namespace bfft
