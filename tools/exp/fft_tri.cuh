// fft_tri.cuh (experiment, not product code: tools/exp/exp_tri.cu) — the four-step of SURVEY.md §8(a) row a4 for long records,
// with the row transform itself split once more (three factors), as ONE
// persistent dependency-driven kernel whose intermediates stay in L2.
//
// Why: with two factors a 2^21..2^22 record needs N1 = 2048-point columns, so
// a 64 KiB tile is only 4 columns wide and both HBM legs move 32-byte runs
// (k_pipe2 at 28-33 % of the roofline, profiles/r02_pipe2_2p2[12]_ncu.md).
// With N = N1 * N2 * N3, N1 = 256, every HBM access is a 256-byte run and
// every transform is 64..256 points.
//
// n = n1 M + m, m = n2 N3 + n3 (M = N2 N3);  k = k1 + N1 (k2 + N2 k3):
//   A  (record r, 32 columns m):   y[k1][m]     = W_N^{m k1} FFT_N1 over n1 of x[n1 M + m]      HBM -> ring
//   B1 (r, k1 group, 16 n3):       u[k1][k2][n3] = W_M^{n3 k2} FFT_N2 over n2 of y[k1][n2 N3 + n3]  ring -> ring (in place)
//   B2 (r, 32 k1, K2 k2):          X[k1 + N1 (k2 + N2 k3)] = FFT_N3 over n3 of u[k1][k2][n3]      ring -> HBM
// (X[k1 + N1 k'] = sum_m W_M^{m k'} y[k1][m], and the length-M DFT over m is
// itself the four-step of M = N2 N3 — the decomposition of PAPER.md P:41 /
// the paper's Cooley-Tukey recursion applied twice.)
//
// Scheduling is k_pipe2's: one global atomic hands out tasks in rounds; round
// j holds the A-tasks of record j, the B1-tasks of record j - L1 and the
// B2-tasks of record j - L2 (1 <= L1 <= L2 < S; B1- and B2-tasks in k1-block
// order, so with L1 = L2 a B2-task follows the B1-tasks it needs by a whole
// block of tasks and a record's intermediate is live for about one round —
// 2^22-point records are 32 MiB, and the L2 holds little more than two).
// Dependencies (acquire / release counters):
//   A(r)  : the B2-tasks of record r - S have read slot r mod S (WAR);
//   B1(r) : every A-task of record r has published;
//   B2(r) : the B1-tasks of record r covering its 32 k1 rows have published.
// Every dependency points to an earlier-issued task, so the schedule cannot
// deadlock.  Warp roles as in k_pipe2: a producer warp (claims, waits, stages
// each task's 64 KiB tile: A by a 3-D TMA box of the input, B1 by a 4-D TMA
// box of the ring, B2 by one bulk copy per ring row into padded rows), NGRP
// compute groups of 4 warps, two per task (each FFTs half of the tile in its
// own exchange region), and a release warp that publishes finished tasks.
#pragma once

#include "../../paper_1407_6915_b200/csrc/fft_pipe.cuh"

namespace bfft {

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* tmap, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

template <int N1, int N2, int N3, int NSTAGE = 3, int NGRP = 4, int H = 2>
struct TriCfg {
    static constexpr int PP = 32;                              // points per thread
    static constexpr int M = N2 * N3, N = N1 * M;
    static constexpr int T1 = N1 / PP, T2 = N2 / PP, T3 = N3 / PP;   // threads per transform
    static constexpr int NTC = 128;                            // threads per compute group
    static constexpr int CA = NTC / T1;                        // A: columns m per group
    static constexpr int CB1 = NTC / T2;                       // B1: (k1, n3) columns per group
    static constexpr int KB1 = CB1 / 16;                       //     k1 per group (16 n3 each)
    static constexpr int R3 = NTC / T3;                        // B2: rows (k1, k2) per group
    static constexpr int K2 = R3 / 16;                         //     k2 per group (16 k1 each)
    static constexpr int NKB = N1 / (H * 16);                  // B2 k1 blocks (32 rows each)
    static constexpr int TA = M / (H * CA);                    // tasks per record, by kind
    static constexpr int TB1 = (N1 / (H * KB1)) * (N3 / 16);
    static constexpr int TB2 = NKB * (N2 / K2);
    static constexpr int TB1_PER_KB = TB1 / NKB;               // B1 tasks per B2 k1 block
    static constexpr int RS3 = N3 + 2;                         // padded B2 row
    static_assert(N1 == 256 && N2 >= 64 && N3 >= 64 && N2 <= 256 && N3 <= 256, "three-factor shapes");
    static_assert(CA == 16 && CB1 % 16 == 0 && R3 % 16 == 0, "16-wide lanes");
    static_assert(NGRP % H == 0 && NGRP / H <= NSTAGE, "every sequence's end marker needs a stage");
    static constexpr int NSEQ = NGRP / H;
    static constexpr int NT = NTC * NGRP + 64;
    using LayA = PadColLayout<CA, Sched<N1, PP>::R0>;
    using LayB1 = PadColLayout<CB1, Sched<N2, PP>::R0>;
    using LayB2 = PadColLayout<R3, Sched<N3, PP>::R0>;
    static constexpr int r16(int x) { return (x + 15) / 16 * 16; }
    static constexpr int mx(int a, int b) { return a > b ? a : b; }
    static constexpr int REG_A = r16(LayA::size(N1)), REG_B1 = r16(LayB1::size(N2)), REG_B2 = r16(LayB2::size(N3));
    static constexpr int TILE_A = H * CA * N1, TILE_B1 = H * CB1 * N2, TILE_B2 = H * R3 * RS3;
    static constexpr int TILE =
        r16(mx(mx(mx(TILE_A, H * REG_A), mx(TILE_B1, H * REG_B1)), mx(TILE_B2, H * REG_B2)));
    static constexpr size_t SMEM = sizeof(float2) * (size_t)TILE * NSTAGE + 64 * NSTAGE + 128;
    static constexpr int MINB = SMEM * 2 <= 227 * 1024 ? 2 : 1;
};

// ctr layout (int32): [0] task counter, [1 .. S] A-tasks published per slot,
// [S+1 .. 2S] B2-tasks finished per slot, [2S+1 .. 2S+S*NKB] B1-tasks
// published per (slot, k1 block), [2S+1+S*NKB] CTAs finished.
template <int N1, int N2, int N3, bool INV, int NSTAGE = 3, int NGRP = 4, int CB = 2, int H = 2>
__global__ void __launch_bounds__(TriCfg<N1, N2, N3, NSTAGE, NGRP, H>::NT, (TriCfg<N1, N2, N3, NSTAGE, NGRP, H>::MINB))
k_tri(const __grid_constant__ CUtensorMap tmap_in, const __grid_constant__ CUtensorMap tmap_ring,
      float2* __restrict__ out, float2* __restrict__ ring, int64_t nrec, int* __restrict__ ctr, int S, int L1,
      int L2, float scale, const float2* __restrict__ w_hi, const float2* __restrict__ w_lo, int w_lb) {
    using CF = TriCfg<N1, N2, N3, NSTAGE, NGRP, H>;
    constexpr int PP = CF::PP, M = CF::M, N = CF::N, NTC = CF::NTC, TILE = CF::TILE;
    constexpr int T1 = CF::T1, T2 = CF::T2, T3 = CF::T3, CB1 = CF::CB1, KB1 = CF::KB1, R3 = CF::R3, K2 = CF::K2;
    constexpr int TA = CF::TA, TB1 = CF::TB1, TB2 = CF::TB2, NKB = CF::NKB, RS3 = CF::RS3;
    extern __shared__ __align__(128) float2 sm[];
    PipeTask* info = reinterpret_cast<PipeTask*>(sm + (size_t)TILE * NSTAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(info + NSTAGE);   // full | empty | done | sfree
    const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + NSTAGE), done0 = smem_addr(bars + 2 * NSTAGE);
    const uint32_t sfree0 = smem_addr(bars + 3 * NSTAGE);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int WP = NGRP * NTC / 32, WR = WP + 1;   // producer, release warps
    int* doneA = ctr + 1;
    int* doneB2 = ctr + 1 + S;
    int* doneB1 = ctr + 1 + 2 * S;
    const int64_t per_round = TA + TB1 + TB2;
    const int64_t total = (nrec + L2) * per_round;

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
            mbar_init(done0 + 8 * i, H * NTC / 32);
            mbar_init(sfree0 + 8 * i, H * NTC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // kind 0 = A, 1 = B1, 2 = B2, 3 = end
    auto decode = [&](long long task, PipeTask& t) -> bool {
        if (task >= total) {
            t.kind = 3;
            t.rec = 0;
            t.tile = 0;
            return true;
        }
        const long long round = task / per_round;
        int o = (int)(task - round * per_round);
        if (o < TA) {
            t.kind = 0;
            t.rec = round;
            t.tile = o;
        } else if ((o -= TA) < TB1) {
            t.kind = 1;
            t.rec = round - L1;
            t.tile = o;
        } else {
            t.kind = 2;
            t.rec = round - L2;
            t.tile = o - TB1;
        }
        return t.rec >= 0 && t.rec < nrec;
    };

    if (warp == WP) {
        // ============================================== producer
        uint32_t k = 0;
        int ends = 0;
        const uint64_t pol_stream = policy_evict_first();
        long long base = 0, nextb = 0;
        int sub = 0;
        const int* dep_ptr = nullptr;
        int dep_seen = 0;
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
            }
            valid = __shfl_sync(0xffffffffu, valid, 0);
            if (!valid) continue;
            d.kind = __shfl_sync(0xffffffffu, d.kind, 0);
            d.rec = __shfl_sync(0xffffffffu, d.rec, 0);
            d.tile = __shfl_sync(0xffffffffu, d.tile, 0);
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            const uint32_t fb = full0 + 8 * s;
            if (lane == 0) {
                BFFT_STRESS_DELAY(20);
                if (u > 0) mbar_wait(empty0 + 8 * s, (u - 1) & 1);
                if (d.kind == 3) {
                    info[s] = d;
                    mbar_arrive(fb);
                } else {
                    const int slot = (int)(d.rec % S), gen = (int)(d.rec / S);
                    const int* dp = nullptr;
                    int target = 0;
                    if (d.kind == 0) {
                        if (gen > 0) dp = doneB2 + slot, target = gen * TB2;                 // slot free (WAR)
                    } else if (d.kind == 1) {
                        dp = doneA + slot, target = (gen + 1) * TA;                           // y published
                    } else {
                        const int kb = d.tile / (N2 / K2);
                        dp = doneB1 + slot * NKB + kb, target = (gen + 1) * CF::TB1_PER_KB;   // u rows published
                    }
#ifdef BFFT_PIPE_NODEPS   // (experiments only: the kernel without its waits; results wrong)
                    dp = nullptr;
#endif
                    if (dp && !(dp == dep_ptr && target <= dep_seen)) {
                        dep_seen = wait_geq_v(dp, target);
                        dep_ptr = dp;
                        // generic ring stores acquired here -> this thread's later async-proxy reads
                        if (d.kind != 0) fence_proxy_async_global();
                    }
                    info[s] = d;
                    mbar_expect_tx(fb, (uint32_t)((d.kind == 0 ? CF::TILE_A : d.kind == 1 ? CF::TILE_B1
                                                                                          : H * R3 * N3) *
                                                  sizeof(float2)));
                }
            }
            if (d.kind == 3) {
                if (++ends == CF::NSEQ) break;
                ++k;
                continue;
            }
            __syncwarp();
            float2* stage = sm + (size_t)s * TILE;
            const int slot = (int)(d.rec % S);
            if (d.kind == 0) {
                if (lane == 0)
                    tma_load_3d_hint(smem_addr(stage), &tmap_in, d.tile * (H * CF::CA), 0, (int)d.rec, fb,
                                     pol_stream);
            } else if (d.kind == 1) {
                if (lane == 0) {
                    const int kb = d.tile / CF::TB1_PER_KB, jj = d.tile % CF::TB1_PER_KB;
                    const int k10 = kb * (H * 16) + (jj / (N3 / 16)) * (H * KB1), n30 = (jj % (N3 / 16)) * 16;
                    tma_load_4d(smem_addr(stage), &tmap_ring, n30, 0, k10, slot, fb);
                }
            } else {
                const int kb = d.tile / (N2 / K2), k2b = d.tile % (N2 / K2);
                for (int j = lane; j < H * R3; j += 32) {
                    const int h = j / R3, rho = j % R3;
                    const int k1 = kb * (H * 16) + 16 * h + (rho & 15), k2 = k2b * K2 + (rho >> 4);
                    bulk_g2s(smem_addr(stage + j * RS3), ring + (int64_t)slot * N + (int64_t)k1 * M + k2 * N3,
                             N3 * sizeof(float2), fb);
                }
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
                if (d.kind == 3) break;
                BFFT_STRESS_DELAY(21);
                mbar_wait(sfree0 + 8 * s, u & 1);
                mbar_arrive(empty0 + 8 * s);
                mbar_wait(done0 + 8 * s, u & 1);
                BFFT_STRESS_DELAY(22);
                fence_acq_rel_gpu();   // the group's stores, observed through done[s], become visible
                const int slot = (int)(d.rec % S);
                int* c = d.kind == 0 ? doneA + slot
                       : d.kind == 1 ? doneB1 + slot * NKB + d.tile / CF::TB1_PER_KB
                                     : doneB2 + slot;
                red_relaxed_gpu(c, 1);
            }
        }
    } else {
        // ============================================== compute warps
        const TwoLevel W{w_hi, w_lo, w_lb, (uint32_t)(N - 1)};
        const ConstTw<N1, PP> tabA{};
        const ConstTw<N2, PP> tabB1{};
        const ConstTw<N3, PP> tabB2{};
        const int grp = warp / (NTC / 32);
        const int gtid = tid - grp * NTC;
        const int half = grp % H;
        const NamedBarrier bar{1 + grp, NTC};
        const NamedBarrier pair{1 + NGRP + grp / H, H * NTC};   // the task's two groups: inputs read
        for (uint32_t k = grp / H;; k += CF::NSEQ) {
            const uint32_t s = k % NSTAGE, u = k / NSTAGE;
            mbar_wait(full0 + 8 * s, u & 1);
            BFFT_STRESS_DELAY(23);
            const PipeTask d = info[s];
            if (d.kind == 3) break;
            float2* stage = sm + (size_t)s * TILE;
            const int64_t r = d.rec;
            const int slot = (int)(r % S);
            float2* rs = ring + (int64_t)slot * N;
            float2 v[PP];
            if (d.kind == 0) {
                // ---------------- A: 16 columns m, FFT over n1, W_N^{m k1}, -> y[k1][m]
                const int c = gtid % 16, t = gtid / 16;
                const uint32_t m = (uint32_t)(d.tile * (H * 16) + 16 * half + c);
                float2 f[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) f[i] = W(m * (uint32_t)(T1 << i));
                const float2 w0 = W(m * (uint32_t)t);
#pragma unroll
                for (int q = 0; q < PP; ++q) {
                    const float2 x = stage[(t + q * T1) * (H * 16) + 16 * half + c];
                    v[q] = INV ? conjf2(x) : x;
                }
                if constexpr (H > 1) pair();
                fft_engine<N1, PP>(v, t, stage + half * CF::REG_A, [&](int e) { return CF::LayA::at(e, c); }, tabA,
                                   bar);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(sfree0 + 8 * s);
                float2 w[PP];
                w[0] = w0;
                v[0] = cmul(v[0], w0);
#pragma unroll
                for (int q = 1; q < PP; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                    w[q] = cmul(w[q & (q - 1)], f[lb]);
                    v[q] = cmul(v[q], w[q]);
                }
                float2* dst = rs + (int64_t)t * M + m;
#pragma unroll
                for (int q = 0; q < PP; ++q) dst[(int64_t)q * T1 * M] = v[q];
            } else if (d.kind == 1) {
                // ---------------- B1: columns (k1, n3), FFT over n2, W_M^{n3 k2}, -> u in place
                const int kb = d.tile / CF::TB1_PER_KB, jj = d.tile % CF::TB1_PER_KB;
                const int c = gtid % CB1, t = gtid / CB1;
                const int k1l = half * KB1 + c / 16;
                const int k1 = kb * (H * 16) + (jj / (N3 / 16)) * (H * KB1) + k1l;
                const int n3 = (jj % (N3 / 16)) * 16 + (c & 15);
                // W_M^{n3 k2} = W_N^{N1 n3 k2}, k2 = t + T2 q
                float2 f[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) f[i] = W((uint32_t)(N1 * n3) * (uint32_t)(T2 << i));
                const float2 w0 = W((uint32_t)(N1 * n3) * (uint32_t)t);
                const float2* src = stage + (size_t)k1l * N2 * 16 + (c & 15);
#pragma unroll
                for (int q = 0; q < PP; ++q) v[q] = src[(t + q * T2) * 16];
                if constexpr (H > 1) pair();
                fft_engine<N2, PP>(v, t, stage + half * CF::REG_B1, [&](int e) { return CF::LayB1::at(e, c); },
                                   tabB1, bar);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(sfree0 + 8 * s);
                float2 w[PP];
                w[0] = w0;
                v[0] = cmul(v[0], w0);
#pragma unroll
                for (int q = 1; q < PP; ++q) {
                    const int lb = (q & 1) ? 0 : (q & 2) ? 1 : (q & 4) ? 2 : (q & 8) ? 3 : 4;
                    w[q] = cmul(w[q & (q - 1)], f[lb]);
                    v[q] = cmul(v[q], w[q]);
                }
                float2* dst = rs + (int64_t)k1 * M + (int64_t)t * N3 + n3;
#pragma unroll
                for (int q = 0; q < PP; ++q) dst[(int64_t)q * T2 * N3] = v[q];
            } else {
                // ---------------- B2: rows (k1, k2), FFT over n3, -> X[k1 + N1 (k2 + N2 k3)]
                const int kb = d.tile / (N2 / K2), k2b = d.tile % (N2 / K2);
                const int rho = gtid % R3, t = gtid / R3;
                const int k1 = kb * (H * 16) + 16 * half + (rho & 15), k2 = k2b * K2 + (rho >> 4);
                {   // the rows are staged: drop them from L2 (no write-back)
                    const char* row0 = reinterpret_cast<const char*>(rs);
                    constexpr int LPR = N3 * 8 / 128;   // 128-byte lines per row
                    for (int i = gtid; i < R3 * LPR; i += NTC) {
                        const int rr = i / LPR, ln = i % LPR;
                        const int kk1 = kb * (H * 16) + 16 * half + (rr & 15), kk2 = k2b * K2 + (rr >> 4);
                        l2_discard128(row0 + ((int64_t)kk1 * M + (int64_t)kk2 * N3) * 8 + 128 * ln);
                    }
                }
                const float2* src = stage + (size_t)(half * R3 + rho) * RS3;
#pragma unroll
                for (int q = 0; q < PP; ++q) v[q] = src[t + q * T3];
                if constexpr (H > 1) pair();
                fft_engine<N3, PP>(v, t, stage + half * CF::REG_B2, [&](int e) { return CF::LayB2::at(e, rho); },
                                   tabB2, bar);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(sfree0 + 8 * s);
                float2* dst = out + r * N + k1 + (int64_t)N1 * k2 + (int64_t)t * N1 * N2;
#pragma unroll
                for (int q = 0; q < PP; ++q)
                    st_stream(dst + (int64_t)q * T3 * N1 * N2, INV ? scale_conj(v[q], scale) : v[q]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(done0 + 8 * s);
        }
    }
    // the last CTA out resets every counter (one launch per exec)
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nctr = 1 + 2 * S + S * NKB;
        __threadfence();
        const int prev = atomicAdd(ctr + nctr, 1);
        if (prev == (int)gridDim.x - 1) {
            __threadfence();
            for (int i = 0; i <= nctr; ++i) ctr[i] = 0;
        }
    }
}

}  // namespace bfft
