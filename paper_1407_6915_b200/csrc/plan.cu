// plan.cu — the C ABI's plan layer: fft_plan_create / fft_exec / fft_plan_destroy
// (include/blockfft.h).
//
// PAPER.md:53 §III moves each block to the GPU and runs "CUFFT's batched FFT
// plan" over it; here the batched plan is our own: validation, variant choice
// by N, fp64-computed twiddle tables rounded once to fp32 and uploaded, launch
// geometry, and (four-step) an HBM scratch wave.  fft_exec only enqueues.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/blockfft.h"
#include "common.h"
#include <cuda.h>
#include <cudaTypedefs.h>

#include "fft_kernels.cuh"
#include "plan_internal.h"

enum { TW_TREE = 0, TW_TABLE = 1, TW_SPLIT = 2 };   // fft_pipe.cuh

using namespace bfft;

// ------------------------------------------------------------ error state
static thread_local std::string g_err;
static thread_local int g_code = 0;

int bfft_set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    g_code = code;
    return code;
}
void bfft_clear_error() {
    g_err.clear();
    g_code = 0;
}
int bfft_last_code() { return g_code ? g_code : FFT_E_CUDA; }

extern "C" const char* fft_last_error(void) { return g_err.c_str(); }
extern "C" int fft_last_status(void) { return g_code; }
extern "C" int fft_version(void) { return BLOCKFFT_VERSION; }

#define CUDA_TRY(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return bfft_set_error(FFT_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------ kernel tables: kern_*.cu (plan_internal.h)

// ------------------------------------------------------------ TMA tensor maps
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    // function-local static: initialised once, thread-safe (several streamer
    // threads make their first TMA launch concurrently)
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000)p;
        cudaGetLastError();
        return nullptr;
    }();
    return fn;
}

// Records viewed as a 3-D tensor of 8-byte elements [count][n1][n2] (n2
// fastest), consecutive records rec_stride elements apart (n1 n2 for records,
// the hop for STFT frames; a multiple of 2: TMA strides are 16-byte multiples);
// box = {box_cols, box_rows, 1}: one record's column tile.
static int make_record_tmap(CUtensorMap* m, const void* base, int64_t count, int n1, int n2, int box_cols,
                            int box_rows, int64_t rec_stride = 0) {
    auto fn = encode_fn();
    if (!fn) return bfft_set_error(FFT_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    if (rec_stride == 0) rec_stride = (int64_t)n1 * n2;
    cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)count};
    cuuint64_t strides[2] = {(cuuint64_t)n2 * 8, (cuuint64_t)rec_stride * 8};
    cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    // L2 promotion 256 B (measured no different from none or 128 B: profiles/r01_tmap_promotion.txt)
    const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return bfft_set_error(FFT_E_CUDA, "cuTensorMapEncodeTiled failed: CUresult %d", (int)r);
    return FFT_OK;
}

// ------------------------------------------------------------ twiddle tables
// Stockham per-pass table for length L (same schedule as Sched<L, P>): for each
// pass p >= 1 with sub-length Ns, entries [(q-1)*Ns + jj] = W_{P Ns}^{jj q},
// computed in fp64 and rounded once to fp32.
static void stockham_table(int L, std::vector<float2>& out, int P = 16) {
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
                const long long m = (long long)jj * q;  // < M
                const double ang = -2.0 * M_PI * (double)m / (double)M;
                out.push_back(make_float2((float)cos(ang), (float)sin(ang)));
            }
    }
}

// Fill c_tw (the constant-memory twiddles of the column engines) once per
// device, in const_tw_base order.
#include <mutex>
static int upload_const_twiddles(int device) {
    static std::mutex mu;
    static bool done[256] = {};
    std::lock_guard<std::mutex> g(mu);
    if (device < 0 || device >= 256) return bfft_set_error(FFT_E_DEVICE, "device index out of range: %d", device);
    if (done[device]) return FFT_OK;
    std::vector<float2> all, one;
    for (int pp = 16; pp <= 32; pp *= 2)
        for (int l = CTW_MIN_L; l <= ctw_max_l(pp); l *= 2) {
            if (const_tw_base(l, pp) != (int)all.size())
                return bfft_set_error(FFT_E_CUDA, "constant twiddle layout mismatch at L=%d P=%d", l, pp);
            stockham_table(l, one, pp);
            all.insert(all.end(), one.begin(), one.end());
        }
    if ((int)all.size() != CTW_TOTAL) return bfft_set_error(FFT_E_CUDA, "constant twiddle size mismatch");
    CUDA_TRY(cudaMemcpyToSymbol(c_tw, all.data(), all.size() * sizeof(float2)));
    if (pipe3_upload_const(all.data(), all.size()) != 0 || rows_upload_const(all.data(), all.size()) != 0 ||
        cluster_upload_const(all.data(), all.size()) != 0 || pipe_upload_const(all.data(), all.size()) != 0)
        return bfft_set_error(FFT_E_CUDA, "constant twiddle upload failed");
    done[device] = true;
    return FFT_OK;
}

// ------------------------------------------------------------ the plan
struct fft_plan {
    int64_t n = 0, batch = 0;
    int dir = 0, variant = 0, device = 0, log2n = 0, sms = 0;
    int n1 = 0, n2 = 0, cluster = 1, cluster_impl = 0;
    int pipe_S = 0, pipe_LAG = 0;     // pipelined four-step ring depth and lag
    int w_lb = 0;                     // two-level twiddle split (tw_a = hi, tw_b = lo)
    int pipe_impl = 1, pipe_boxr = 0; // k_pipe (1) or warp-specialised k_pipe2 (2)
    int* d_ctr = nullptr;             // pipelined four-step task/dependency counters
    float scale = 1.f;
    float2* d_tab = nullptr;          // all twiddle tables
    size_t tab_bytes = 0;
    const float2* tw_a = nullptr;     // table for the first (or only) length
    const float2* tw_b = nullptr;     // table for the second length
    float2* d_scratch = nullptr;      // four-step wave scratch
    int64_t wave = 0;                 // records per four-step wave
    KernelSet ka, kb;                 // kernels (kb only for four-step)
    KernelSet kt;                     // single pass: k_rows_tma for contiguous records (ka = k_rows
                                      // stays for strided / windowed STFT frames)
    int occ_t = 0;
    int grid_a = 0, grid_b = 0;       // persistent/capped grid sizes (per full batch)
    int occ_a = 0, occ_b = 0;
    int real = 0;                     // 1: real records (fft_plan_create_real), n reals each
    int real_split = 0;               // inner plan of a real plan: k_pipe2 with the split (1) or merge (2) fused
    int64_t hop = 0;                  // > 0: STFT frames every `hop` samples (fft_plan_create_stft)
    float* d_win = nullptr;           // STFT: optional window, n floats
    fft_plan* inner = nullptr;        // real: the n/2-point complex plan; STFT: the frames' plan
    int rt_lb = 0;                    // real: two-level W_n split (tw_a = hi, tw_b = lo)
};

// dir_ok_zero: direction 0 (identity) is accepted only where the identity
// variant is requested explicitly (fft_plan_create_ex / _opts, the streamer)
static int validate(int64_t n, int64_t batch, int dir, bool dir_ok_zero = false) {
    if (n < 2 || n > (1 << 22) || (n & (n - 1)) != 0)
        return bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
    if (batch < 1) return bfft_set_error(FFT_E_BATCH, "batch must be >= 1: %lld", (long long)batch);
    if (dir != FFT_FORWARD && dir != FFT_INVERSE && !(dir == 0 && dir_ok_zero))
        return bfft_set_error(FFT_E_DIR, "direction must be -1 or +1: %d", dir);
    return FFT_OK;
}

// fastest measured per size (profiles/r01_variants_*.txt)
// single pass up to 2^14 (k_rows, k_rows_tma at 2^13, k_rows_tma2 at 2^14), the
// pipelined four-step above (profiles/r02_config5_sweep_final.txt)
static int default_variant(int log2n) { return log2n <= 14 ? FFT_VARIANT_SINGLE : FFT_VARIANT_PIPE; }

static int set_smem(const KernelSet& k) {
    if (k.smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
    return FFT_OK;
}

static int plan_init(fft_plan* p, int64_t n, int64_t batch, int dir, const fft_plan_opts& o) {
    int variant = o.variant;
    int rc = validate(n, batch, dir, variant == FFT_VARIANT_IDENTITY);
    if (rc) return rc;
    if (dir != 0 && variant == FFT_VARIANT_IDENTITY)
        return bfft_set_error(FFT_E_DIR, "identity variant takes direction 0: %d", dir);
    if (variant < 0 || variant > FFT_VARIANT_PIPE)
        return bfft_set_error(FFT_E_ARG, "unknown variant: %d", variant);
    p->n = n;
    p->batch = batch;
    p->dir = dir;
    p->log2n = ilog2((int)n);
    p->scale = 1.0f / (float)n;
    CUDA_TRY(cudaGetDevice(&p->device));
    CUDA_TRY(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, p->device));
    const bool inv = dir == FFT_INVERSE;
    rc = upload_const_twiddles(p->device);
    if (rc) return rc;
    if (variant == FFT_VARIANT_AUTO) variant = default_variant(p->log2n);
    p->variant = variant;

    std::vector<float2> ta, tb;
    if (variant == FFT_VARIANT_IDENTITY) {
        p->n1 = (int)n;
        p->n2 = 1;
    } else if (variant == FFT_VARIANT_SINGLE) {
        if (p->log2n > 14) return bfft_set_error(FFT_E_SIZE, "unsupported transform size for single-pass variant: %lld", (long long)n);
        p->ka = pick_row(p->log2n, inv);
        if (o.impl > 2) return bfft_set_error(FFT_E_ARG, "single-pass impl must be 0, 1 (k_rows) or 2 (k_rows_tma): %d", o.impl);
        if (o.impl != 1) p->kt = pick_row_tma(p->log2n, inv);
        if (o.impl == 2 && !p->kt.fn)
            return bfft_set_error(FFT_E_SIZE, "no k_rows_tma kernel for n = %lld", (long long)n);
        if (p->kt.fn && p->kt.pp != p->ka.pp) p->kt = KernelSet{};   // they share the plan's twiddle table
        p->n1 = (int)n;
        p->n2 = 1;
        stockham_table((int)n, ta, p->ka.pp);
    } else if (variant == FFT_VARIANT_CLUSTER) {
        ClusterChoice ch = pick_cluster(p->log2n, o.cluster_size, inv, o.impl);
        if (!ch.k.fn) return bfft_set_error(FFT_E_SIZE, "unsupported transform size for cluster variant: %lld", (long long)n);
        p->ka = ch.k;
        p->n1 = ch.n1;
        p->n2 = ch.n2;
        p->cluster = ch.c;
        p->cluster_impl = ch.impl;
        stockham_table(ch.n1, ta, ch.pp);
        stockham_table(ch.n2, tb, ch.pp);
    } else if (variant == FFT_VARIANT_PIPE) {
        PipeChoice ch = p->real_split == 1   ? pick_pipe_real(p->log2n)
                         : p->real_split == 2 ? pick_pipe_real_inv(p->log2n)
                                              : pick_pipe(p->log2n, inv, o.impl, o.config);
        if (!ch.k.fn) return bfft_set_error(FFT_E_SIZE, "unsupported transform size for pipelined variant: %lld", (long long)n);
        p->ka = ch.k;
        p->n1 = ch.n1;
        p->n2 = ch.n2;
        p->ka.cols = ch.cols;
        p->kb.cols = ch.rows;
        p->pipe_impl = ch.impl;
        p->pipe_boxr = ch.boxr;
        // four-step twiddle tables (fp64 -> fp32 RN), by the kernel's twiddle mode
        auto w = [](int64_t m, int64_t M) {
            const double ang = -2.0 * M_PI * (double)(m % M) / (double)M;
            return make_float2((float)cos(ang), (float)sin(ang));
        };
        if (ch.twm == TW_SPLIT) {
            // W_N^{n2 k1} = W_N^{n2 t} W_{N2 PP}^{n2 q}, k1 = t + TA1 q (fft_pipe.cuh TW_SPLIT):
            // tw_a = WA[t][n2] = W_N^{n2 t}; tw_b = WB0[t'][q] = W_{N2 PP}^{t' q}, then T[q][s] = W_{PP^2}^{q s}
            const int pp = ch.pp, ta1 = ch.n1 / pp, tb2 = ch.n2 / pp;
            for (int t = 0; t < ta1; ++t)
                for (int n2 = 0; n2 < ch.n2; ++n2) ta.push_back(w((int64_t)n2 * t, n));
            for (int t = 0; t < tb2; ++t)
                for (int q = 0; q < pp; ++q) tb.push_back(w((int64_t)t * q, (int64_t)ch.n2 * pp));
            for (int q = 0; q < pp; ++q)
                for (int s2 = 0; s2 < pp; ++s2) tb.push_back(w((int64_t)q * s2, (int64_t)pp * pp));
        } else if (ch.twm == TW_TABLE) {
            // full four-step twiddle table [k1][n2] = W_N^{n2 k1}
            for (int k1 = 0; k1 < ch.n1; ++k1)
                for (int n2 = 0; n2 < ch.n2; ++n2) ta.push_back(w((int64_t)n2 * k1, n));
            tb.push_back(make_float2(1.f, 0.f));
        } else {
            // two-level W_N table: hi[a] = W_N^{a 2^lb}, lo[b] = W_N^b
            p->w_lb = (p->log2n + 1) / 2;
            const int nhi = 1 << (p->log2n - p->w_lb), nlo = 1 << p->w_lb;
            for (int a = 0; a < nhi; ++a) ta.push_back(w((int64_t)a << p->w_lb, n));
            for (int b = 0; b < nlo; ++b) tb.push_back(w(b, n));
        }
    } else if (variant == FFT_VARIANT_FOURSTEP) {
        if (p->log2n < 8) return bfft_set_error(FFT_E_SIZE, "unsupported transform size for four-step variant: %lld", (long long)n);
        const int k1 = p->log2n / 2, k2 = p->log2n - k1;
        p->n1 = 1 << k1;
        p->n2 = 1 << k2;
        p->ka = pick_fs_col(k1, p->n2, inv);
        p->kb = pick_fs_row(k2, inv);
        if (p->ka.cols > p->n2) p->ka = KernelSet{};
        if (p->kb.cols > p->n1) p->kb = KernelSet{};
        if (!p->ka.fn || !p->kb.fn)
            return bfft_set_error(FFT_E_SIZE, "unsupported transform size for four-step variant: %lld", (long long)n);
        stockham_table(p->n1, ta);
        stockham_table(p->n2, tb);
    } else {
        return bfft_set_error(FFT_E_ARG, "unknown variant: %d", variant);
    }

    // upload tables (one allocation; b after a, 256-byte aligned)
    const size_t a_bytes = ta.size() * sizeof(float2);
    const size_t b_off = (a_bytes + 255) & ~(size_t)255;
    const size_t tot = b_off + tb.size() * sizeof(float2);
    if (tot > 0) {
        cudaError_t e = cudaMalloc(&p->d_tab, tot);
        if (e != cudaSuccess) return bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for twiddle tables failed: %s", tot, cudaGetErrorString(e));
        if (a_bytes) CUDA_TRY(cudaMemcpy(p->d_tab, ta.data(), a_bytes, cudaMemcpyHostToDevice));
        if (!tb.empty()) CUDA_TRY(cudaMemcpy((char*)p->d_tab + b_off, tb.data(), tb.size() * sizeof(float2), cudaMemcpyHostToDevice));
    }
    p->tab_bytes = tot;
    p->tw_a = p->d_tab;
    p->tw_b = (const float2*)((const char*)p->d_tab + b_off);

    // launch geometry
    if (variant == FFT_VARIANT_SINGLE) {
        rc = set_smem(p->ka);
        if (rc) return rc;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_a, p->ka.fn, p->ka.threads, p->ka.smem));
        p->occ_a = std::max(p->occ_a, 1);
        if (p->kt.fn) {
            rc = set_smem(p->kt);
            if (rc) return rc;
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_t, p->kt.fn, p->kt.threads, p->kt.smem));
            if (p->occ_t < 1) return bfft_set_error(FFT_E_CUDA, "k_rows_tma cannot be scheduled (%zu B shared memory)", p->kt.smem);
        }
    } else if (variant == FFT_VARIANT_CLUSTER) {
        rc = set_smem(p->ka);
        if (rc) return rc;
        if (p->cluster > 8)
            CUDA_TRY(cudaFuncSetAttribute(p->ka.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = p->cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(p->cluster * p->sms, 1, 1);
        cfg.blockDim = dim3(p->ka.threads, 1, 1);
        cfg.dynamicSmemBytes = p->ka.smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        CUDA_TRY(cudaOccupancyMaxActiveClusters(&ncl, p->ka.fn, &cfg));
        if (ncl < 1) return bfft_set_error(FFT_E_CUDA, "cluster of %d CTAs x %zu B shared memory cannot be scheduled", p->cluster, p->ka.smem);
        p->occ_a = ncl;  // co-resident clusters
    } else if (variant == FFT_VARIANT_PIPE) {
        rc = set_smem(p->ka);
        if (rc) return rc;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_a, p->ka.fn, p->ka.threads, p->ka.smem));
        p->occ_a = std::max(p->occ_a, 1);
        const int resident = p->occ_a * p->sms;
        const int per_round = p->n2 / p->ka.cols + p->n1 / p->kb.cols;
        PipeChoice ch = p->real_split == 1   ? pick_pipe_real(p->log2n)
                         : p->real_split == 2 ? pick_pipe_real_inv(p->log2n)
                                              : pick_pipe(p->log2n, inv, o.impl, o.config);
        // B-tasks of record r are issued LAG rounds after its A-tasks, and an
        // A-task reuses the ring slot of record r - S, whose B-tasks were
        // issued S - LAG rounds earlier.  Both gaps must exceed the tasks a
        // GPU holds in flight (resident CTAs x tasks each CTA has claimed:
        // 1 for k_pipe, stages + 1 for k_pipe2) or tasks stall on their
        // dependencies; measured best on B200 (profiles/r01_pipe_lag_sweep.txt):
        // LAG ~ 1.5x and S - LAG ~ 2x the in-flight rounds.  The ring is capped
        // at 96 MiB so it stays resident in the 126 MB L2.
        const int stages = ch.impl >= 2 ? ch.stages : 0;   // k_pipe3: stages + groups
        const int64_t inflight = (int64_t)resident * (stages + 1);
        const int64_t rounds = (inflight + per_round - 1) / per_round;
        p->pipe_LAG = (int)(3 * rounds / 2 + 1);
        if (o.ring_lag > 0) p->pipe_LAG = o.ring_lag;
        const int64_t rec_bytes = n * (int64_t)sizeof(float2);
        const int s_cap = (int)std::max<int64_t>(p->pipe_LAG + 2, (96ll << 20) / rec_bytes);
        p->pipe_S = (int)std::min<int64_t>(p->pipe_LAG + 2 * rounds + 1, s_cap);
        if (o.ring_records > 0) p->pipe_S = std::max(p->pipe_LAG + 1, o.ring_records);
        const size_t rb = (size_t)p->pipe_S * (size_t)n * sizeof(float2);
        cudaError_t e = cudaMalloc(&p->d_scratch, rb);
        if (e != cudaSuccess) return bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for the pipelined ring failed: %s", rb, cudaGetErrorString(e));
        // counters: task, doneA[S], doneB[S], CTAs out; zero here, and reset to zero by
        // the last CTA of every launch (pipe_exit_reset), so fft_exec is one launch
        e = cudaMalloc(&p->d_ctr, sizeof(int) * (2 + 2 * p->pipe_S));
        if (e != cudaSuccess) return bfft_set_error(FFT_E_NOMEM, "cudaMalloc for pipelined counters failed: %s", cudaGetErrorString(e));
        CUDA_TRY(cudaMemset(p->d_ctr, 0, sizeof(int) * (2 + 2 * p->pipe_S)));
        p->wave = p->pipe_S;
    } else if (variant == FFT_VARIANT_FOURSTEP) {
        rc = set_smem(p->ka);
        if (rc) return rc;
        rc = set_smem(p->kb);
        if (rc) return rc;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_a, p->ka.fn, p->ka.threads, p->ka.smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_b, p->kb.fn, p->kb.threads, p->kb.smem));
        p->occ_a = std::max(p->occ_a, 1);
        p->occ_b = std::max(p->occ_b, 1);
        const int64_t wave_bytes = 256ll << 20;   // one wave of records through the HBM scratch
        p->wave = std::max<int64_t>(1, std::min<int64_t>(batch, wave_bytes / (8 * n)));
        const size_t sb = (size_t)p->wave * (size_t)n * sizeof(float2);
        cudaError_t e = cudaMalloc(&p->d_scratch, sb);
        if (e != cudaSuccess) return bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for four-step scratch failed: %s", sb, cudaGetErrorString(e));
    }
    return FFT_OK;
}

static void plan_free(fft_plan* p) {
    if (!p) return;
    if (p->inner) plan_free(p->inner);
    if (p->d_win) cudaFree(p->d_win);
    if (p->d_tab) cudaFree(p->d_tab);
    if (p->d_scratch) cudaFree(p->d_scratch);
    if (p->d_ctr) cudaFree(p->d_ctr);
    delete p;
}

extern "C" fft_plan* fft_plan_create_opts(int64_t n, int64_t batch, int dir, const fft_plan_opts* opts) {
    bfft_clear_error();
    fft_plan_opts o{};
    if (opts) o = *opts;
    if (o.variant < 0 || o.variant > FFT_VARIANT_PIPE || o.impl < 0 || o.config < 0 || o.cluster_size < 0 ||
        o.ring_records < 0 || o.ring_lag < 0) {
        bfft_set_error(FFT_E_ARG, "invalid plan options: variant=%d impl=%d config=%d cluster_size=%d "
                       "ring_records=%d ring_lag=%d", o.variant, o.impl, o.config, o.cluster_size, o.ring_records,
                       o.ring_lag);
        return nullptr;
    }
    fft_plan* p = new (std::nothrow) fft_plan();
    if (!p) {
        bfft_set_error(FFT_E_NOMEM, "out of host memory");
        return nullptr;
    }
    if (plan_init(p, n, batch, dir, o) != FFT_OK) {
        std::string keep = g_err;
        int code = g_code;
        plan_free(p);
        g_err = keep;
        g_code = code;
        return nullptr;
    }
    return p;
}

extern "C" fft_plan* fft_plan_create_ex(int64_t n, int64_t batch, int dir, int variant) {
    fft_plan_opts o{};
    o.variant = variant;
    return fft_plan_create_opts(n, batch, dir, &o);
}

extern "C" fft_plan* fft_plan_create(int64_t n, int64_t batch, int dir) {
    return fft_plan_create_opts(n, batch, dir, nullptr);
}

extern "C" fft_plan* fft_plan_create_real(int64_t n, int64_t batch, int dir) {
    bfft_clear_error();
    if (n < 4 || n > (1 << 23) || (n & (n - 1)) != 0) {
        bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
        return nullptr;
    }
    if (batch < 1) {
        bfft_set_error(FFT_E_BATCH, "batch must be >= 1: %lld", (long long)batch);
        return nullptr;
    }
    if (dir != FFT_FORWARD && dir != FFT_INVERSE) {
        bfft_set_error(FFT_E_DIR, "direction must be -1 or +1: %d", dir);
        return nullptr;
    }
    fft_plan* p = new (std::nothrow) fft_plan();
    if (!p) {
        bfft_set_error(FFT_E_NOMEM, "out of host memory");
        return nullptr;
    }
    auto fail = [&]() -> fft_plan* {
        std::string keep = g_err;
        int code = g_code;
        plan_free(p);
        g_err = keep;
        g_code = code;
        return nullptr;
    };
    p->real = 1;
    p->n = n;
    p->batch = batch;
    p->dir = dir;
    p->log2n = ilog2((int)(n >> 1)) + 1;
    // 2^16..2^19 samples: k_pipe2 with the split (forward) or the merge (inverse)
    // fused — one launch (measured: the fused merge loses to two kernels above
    // 2^19, where its partner reads miss L2; profiles/r02_real_bench_shfl.txt);
    // other sizes: the complex n/2-point plan (+ k_real_split above 2^15)
    const bool fuse = n >= (1 << 16) && n <= (1 << 19);
    const int rs = !fuse ? 0 : dir == FFT_FORWARD ? (pick_pipe_real(ilog2((int)(n / 2))).k.fn ? 1 : 0)
                                                  : (pick_pipe_real_inv(ilog2((int)(n / 2))).k.fn ? 2 : 0);
    if (rs) {
        fft_plan* q = new (std::nothrow) fft_plan();
        if (!q) {
            bfft_set_error(FFT_E_NOMEM, "out of host memory");
            return fail();
        }
        q->real_split = rs;
        fft_plan_opts o{};
        o.variant = FFT_VARIANT_PIPE;
        o.impl = 2;
        p->inner = q;
        if (plan_init(q, n / 2, batch, dir, o) != FFT_OK) return fail();
    } else {
        p->inner = fft_plan_create_opts(n / 2, batch, dir, nullptr);
    }
    if (!p->inner) return fail();
    p->device = p->inner->device;
    p->sms = p->inner->sms;
    p->variant = p->inner->variant;
    // W_n^k for k <= n/2 as hi[k >> lb] * lo[k & (2^lb - 1)], fp64 -> fp32 (reading c9)
    p->rt_lb = p->log2n / 2;
    // k up to n/2: the fused single-pass kernel evaluates X[k] for every k < n/2
    const int64_t nhi = ((n / 2) >> p->rt_lb) + 1, nlo = 1ll << p->rt_lb;
    std::vector<float2> t;
    for (int64_t a = 0; a < nhi; ++a) {
        const double ang = -2.0 * M_PI * (double)(a << p->rt_lb) / (double)n;
        t.push_back(make_float2((float)cos(ang), (float)sin(ang)));
    }
    for (int64_t b = 0; b < nlo; ++b) {
        const double ang = -2.0 * M_PI * (double)b / (double)n;
        t.push_back(make_float2((float)cos(ang), (float)sin(ang)));
    }
    p->tab_bytes = t.size() * sizeof(float2);
    cudaError_t e = cudaMalloc(&p->d_tab, p->tab_bytes);
    if (e != cudaSuccess) {
        bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for twiddle tables failed: %s", p->tab_bytes, cudaGetErrorString(e));
        return fail();
    }
    e = cudaMemcpy(p->d_tab, t.data(), p->tab_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        bfft_set_error(FFT_E_CUDA, "cudaMemcpy of twiddle tables failed: %s", cudaGetErrorString(e));
        return fail();
    }
    p->tw_a = p->d_tab;
    p->tw_b = p->d_tab + nhi;
    if (p->inner->variant == FFT_VARIANT_SINGLE) {
        // records of up to 2^14 reals: one kernel, the split / merge fused into the
        // single-pass transform (k_rows<..., REAL>); longer records: two kernels
        // 2^14 / 2^15 reals: the staged kernels (k_rows_tma / k_rows_tma2 <..., REAL>) when the
        // inner plan uses them; else k_rows<..., REAL>
        if (p->inner->kt.fn) p->kt = pick_row_real_tma(ilog2((int)(n / 2)), dir == FFT_INVERSE);
        if (p->kt.fn) {
            if (set_smem(p->kt)) return fail();
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_t, p->kt.fn, p->kt.threads, p->kt.smem);
            if (e != cudaSuccess || p->occ_t < 1) {
                bfft_set_error(FFT_E_CUDA, "k_rows_tma (real) cannot be scheduled");
                return fail();
            }
        } else {
            p->ka = pick_row_real(ilog2((int)(n / 2)), dir == FFT_INVERSE);
            if (!p->ka.fn) {
                bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
                return fail();
            }
            if (set_smem(p->ka)) return fail();
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->occ_a, p->ka.fn, p->ka.threads, p->ka.smem);
            if (e != cudaSuccess) {
                bfft_set_error(FFT_E_CUDA, "occupancy query failed: %s", cudaGetErrorString(e));
                return fail();
            }
            p->occ_a = std::max(p->occ_a, 1);
        }
    }
    return p;
}

extern "C" fft_plan* fft_plan_create_stft(int64_t n, int64_t hop, int64_t frames, int dir, const float* window) {
    bfft_clear_error();
    if (validate(n, frames, dir)) return nullptr;
    if (hop < 1) {
        bfft_set_error(FFT_E_ARG, "hop must be >= 1: %lld", (long long)hop);
        return nullptr;
    }
    fft_plan* p = new (std::nothrow) fft_plan();
    if (!p) {
        bfft_set_error(FFT_E_NOMEM, "out of host memory");
        return nullptr;
    }
    auto fail = [&]() -> fft_plan* {
        std::string keep = g_err;
        int code = g_code;
        plan_free(p);
        g_err = keep;
        g_code = code;
        return nullptr;
    };
    p->n = n;
    p->batch = frames;
    p->dir = dir;
    p->hop = hop;
    p->log2n = ilog2((int)n);
    p->inner = fft_plan_create_opts(n, frames, dir, nullptr);
    if (!p->inner) return fail();
    p->device = p->inner->device;
    p->sms = p->inner->sms;
    p->variant = p->inner->variant;
    if (window) {
        cudaError_t e = cudaMalloc(&p->d_win, sizeof(float) * n);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_win, window, sizeof(float) * n, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            bfft_set_error(FFT_E_CUDA, "window upload failed: %s", cudaGetErrorString(e));
            return fail();
        }
    }
    return p;
}

extern "C" void fft_plan_destroy(fft_plan* p) { plan_free(p); }

// STFT frames longer than the single-pass kernels handle are framed (hop-strided
// tensor map) and windowed as k_pipe2 reads its A-tiles — one launch — when the
// hop keeps TMA's 16-byte stride alignment; otherwise k_frames frames them first.
static bool stft_fused(const fft_plan* p) {
    return p->hop > 0 && p->inner && p->inner->variant == FFT_VARIANT_PIPE && p->inner->pipe_impl == 2 &&
           p->hop % 2 == 0;
}

extern "C" int fft_plan_get_info(const fft_plan* p, fft_plan_info* info) {
    if (!p || !info) return bfft_set_error(FFT_E_ARG, "null plan or info pointer");
    if (p->real) {
        int rc = fft_plan_get_info(p->inner, info);
        info->n = p->n;
        info->dir = p->dir;
        if (!p->ka.fn && !p->kt.fn && !p->inner->real_split)
            info->kernels_per_exec += 1;   // + the split / merge kernel (fused up to 2^15, and forward to 2^19)
        info->table_bytes += (int64_t)p->tab_bytes;
        info->real = 1;
        info->hop = 0;
        return rc;
    }
    info->real = 0;
    if (p->hop) {
        int rc = fft_plan_get_info(p->inner, info);
        info->hop = p->hop;
        if (p->inner->variant != FFT_VARIANT_SINGLE && !stft_fused(p)) info->kernels_per_exec += 1;   // + k_frames
        return rc;
    }
    info->hop = 0;
    info->n = p->n;
    info->batch = p->batch;
    info->dir = p->dir;
    info->variant = p->variant;
    info->device = p->device;
    info->n1 = p->n1;
    info->n2 = p->n2;
    info->cluster = p->cluster;
    info->scratch_bytes = p->d_scratch ? p->wave * p->n * 8 : 0;
    info->table_bytes = (int64_t)p->tab_bytes;
    info->resident = p->kt.fn ? p->occ_t : p->occ_a;   // the kernel a contiguous exec launches
    info->exclusive = (p->variant == FFT_VARIANT_PIPE || p->variant == FFT_VARIANT_FOURSTEP) ? 1 : 0;
    info->ring_records = p->variant == FFT_VARIANT_PIPE ? p->pipe_S : 0;
    info->ring_lag = p->variant == FFT_VARIANT_PIPE ? p->pipe_LAG : 0;
    if (p->variant == FFT_VARIANT_FOURSTEP)
        info->kernels_per_exec = (int)(2 * ((p->batch + p->wave - 1) / p->wave));
    else
        info->kernels_per_exec = 1;
    return FFT_OK;
}

// ------------------------------------------------------------ exec
static int launch(const fft_plan* p, const float2* in, float2* out, int64_t count, cudaStream_t st,
                  int64_t istride = 0, const float* window = nullptr, RealTw rt = RealTw{nullptr, nullptr, 0}) {
    const int64_t n = p->n;
    if (istride == 0) istride = n;
    switch (p->variant) {
        case FFT_VARIANT_IDENTITY: {
            const int64_t n16 = count * n * 8 / 16;
            const int threads = 256;
            const int64_t want = (n16 + threads - 1) / threads;
            const int grid = (int)std::min<int64_t>(want, (int64_t)p->sms * 16);
            k_copy<<<grid, threads, 0, st>>>((const float4*)in, (float4*)out, n16);
            break;
        }
        case FFT_VARIANT_SINGLE: {
            if (p->kt.fn && istride % 2 == 0) {
                // persistent staged kernel (records, or STFT frames at an even hop: 16-byte aligned copies)
                const int grid = (int)std::min<int64_t>(count, (int64_t)p->sms * p->occ_t);
                if (grid > 0)
                    ((RowTmaFn)p->kt.fn)<<<grid, p->kt.threads, p->kt.smem, st>>>(
                        in, out, count, p->tw_a, p->scale, RealTw{nullptr, nullptr, 0}, istride, window);
                break;
            }
            const int64_t groups = (count + p->ka.cols - 1) / p->ka.cols;
            const int grid = (int)std::min<int64_t>(groups, (int64_t)p->sms * p->occ_a * 8);
            auto fn = (RowFn)p->ka.fn;
            fn<<<grid, p->ka.threads, p->ka.smem, st>>>(in, out, count, p->tw_a, p->scale, istride, window,
                                                         RealTw{nullptr, nullptr, 0});
            break;
        }
        case FFT_VARIANT_CLUSTER: {
            const int64_t ncl = std::min<int64_t>(count, p->occ_a);
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = p->cluster;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3((unsigned)(ncl * p->cluster), 1, 1);
            cfg.blockDim = dim3(p->ka.threads, 1, 1);
            cfg.dynamicSmemBytes = p->ka.smem;
            cfg.stream = st;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (p->cluster_impl == 2) {
                CUDA_TRY(cudaLaunchKernelEx(&cfg, (Cluster2Fn)p->ka.fn, in, out, count, p->scale));
            } else if (p->cluster_impl == 1) {
                CUDA_TRY(cudaLaunchKernelEx(&cfg, (Cluster1Fn)p->ka.fn, in, out, count, p->tw_a, p->tw_b, p->scale));
            } else {
                CUtensorMap tm;
                const int ca = p->n2 / p->cluster;
                int rc = make_record_tmap(&tm, in, count, p->n1, p->n2, ca, p->n1);
                if (rc) return rc;
                CUDA_TRY(cudaLaunchKernelEx(&cfg, (ClusterFn)p->ka.fn, tm, out, count, p->tw_a, p->tw_b, p->scale));
            }
            break;
        }
        case FFT_VARIANT_PIPE: {
            const int grid = p->occ_a * p->sms;
            if (p->pipe_impl >= 2) {
                CUtensorMap tm;
                // STFT frames (istride = hop, window): k_pipe2 only (stft_fused)
                int rc = make_record_tmap(&tm, in, count, p->n1, p->n2, p->ka.cols, p->pipe_boxr, istride);
                if (rc) return rc;
                ((Pipe2Fn)p->ka.fn)<<<grid, p->ka.threads, p->ka.smem, st>>>(tm, out, p->d_scratch, count, p->d_ctr,
                                                                            p->pipe_S, p->pipe_LAG, p->scale, p->tw_a,
                                                                            p->tw_b, p->w_lb, window, rt);
            } else {
                ((PipeFn)p->ka.fn)<<<grid, p->ka.threads, p->ka.smem, st>>>(in, out, p->d_scratch, count, p->d_ctr,
                                                                           p->pipe_S, p->pipe_LAG, p->scale, p->tw_a,
                                                                           p->tw_b, p->w_lb);
            }
            break;
        }
        case FFT_VARIANT_FOURSTEP: {
            const int k1 = ilog2(p->n1), k2 = ilog2(p->n2);
            for (int64_t r0 = 0; r0 < count; r0 += p->wave) {
                const int64_t w = std::min<int64_t>(p->wave, count - r0);
                const int64_t ta = w * (p->n2 / p->ka.cols), tb = w * (p->n1 / p->kb.cols);
                const int ga = (int)std::min<int64_t>(ta, (int64_t)p->sms * p->occ_a * 8);
                const int gb = (int)std::min<int64_t>(tb, (int64_t)p->sms * p->occ_b * 8);
                ((ColFn)p->ka.fn)<<<ga, p->ka.threads, p->ka.smem, st>>>(in + r0 * n, p->d_scratch, w, k2, p->tw_a);
                ((RowTFn)p->kb.fn)<<<gb, p->kb.threads, p->kb.smem, st>>>(p->d_scratch, out + r0 * n, w, k1, p->tw_b, p->scale);
            }
            break;
        }
        default:
            return bfft_set_error(FFT_E_ARG, "plan has unknown variant %d", p->variant);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return FFT_OK;
}

extern "C" int fft_exec_range(const fft_plan* p, const void* in, void* out, int64_t count, void* stream) {
    bfft_clear_error();
    if (!p) return bfft_set_error(FFT_E_ARG, "null plan");
    if (!in || !out) return bfft_set_error(FFT_E_ARG, "null data pointer");
    if (((uintptr_t)in & 15) || ((uintptr_t)out & 15))
        return bfft_set_error(FFT_E_ARG, "data pointers must be 16-byte aligned: in=%p out=%p", in, out);
    if (count < 1 || count > p->batch)
        return bfft_set_error(FFT_E_ARG, "record count out of range: expected 1..%lld, got %lld", (long long)p->batch, (long long)count);
    const uintptr_t bytes = (uintptr_t)(count * p->n * (p->real ? 4 : 8));
    const uintptr_t a = (uintptr_t)in, b = (uintptr_t)out;
    if (p->hop) {
        // STFT: frames overlap in the input, so input and output must be disjoint
        const uintptr_t in_bytes = (uintptr_t)(((count - 1) * p->hop + p->n) * 8);
        if (a < b + bytes && b < a + in_bytes)
            return bfft_set_error(FFT_E_ARG, "STFT input and output overlap");
    } else if (a != b && a < b + bytes && b < a + bytes) {
        return bfft_set_error(FFT_E_ARG, "input and output partially overlap");
    }
    int dev = -1;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev != p->device)
        return bfft_set_error(FFT_E_DEVICE, "plan belongs to device %d, current device is %d", p->device, dev);
    if (p->hop) {
        // STFT frames: the single-pass kernel frames and windows on load; longer
        // frames are framed into `out` first and transformed in place
        cudaStream_t st = (cudaStream_t)stream;
        if (p->inner->variant == FFT_VARIANT_SINGLE || stft_fused(p))
            return launch(p->inner, (const float2*)in, (float2*)out, count, st, p->hop, p->d_win);
        const int threads = 256;
        const int grid = (int)std::min<int64_t>((count * p->n + threads - 1) / threads, (int64_t)p->sms * 16);
        k_frames<<<grid, threads, 0, st>>>((const float2*)in, (float2*)out, count, p->n, p->hop, p->d_win);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
        return launch(p->inner, (const float2*)out, (float2*)out, count, st);
    }
    if (p->real) {
        // real records: forward = complex n/2 transform, then the split in place;
        // inverse = the merge into `out`, then the complex inverse in place
        const int64_t h = p->n / 2;
        cudaStream_t st = (cudaStream_t)stream;
        if (p->kt.fn) {   // fused staged kernel
            const int grid = (int)std::min<int64_t>(count, (int64_t)p->sms * p->occ_t);
            if (grid > 0)
                ((RowTmaFn)p->kt.fn)<<<grid, p->kt.threads, p->kt.smem, st>>>(
                    (const float2*)in, (float2*)out, count, p->inner->tw_a, p->inner->scale, RealTw{p->tw_a, p->tw_b, p->rt_lb},
                    h, nullptr);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
            return FFT_OK;
        }
        if (p->ka.fn) {   // fused single-pass kernel
            const int64_t groups = (count + p->ka.cols - 1) / p->ka.cols;
            const int grid = (int)std::min<int64_t>(groups, (int64_t)p->sms * p->occ_a * 8);
            ((RowFn)p->ka.fn)<<<grid, p->ka.threads, p->ka.smem, st>>>(
                (const float2*)in, (float2*)out, count, p->inner->tw_a, p->inner->scale, h, nullptr,
                RealTw{p->tw_a, p->tw_b, p->rt_lb});
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
            return FFT_OK;
        }
        if (p->inner->real_split)   // k_pipe2 with the split / merge fused (merge: partners read from in)
            return launch(p->inner, (const float2*)in, (float2*)out, count, st, 0, nullptr,
                          RealTw{p->tw_a, p->tw_b, p->rt_lb, (const float2*)in});
        if (p->dir == FFT_FORWARD) {
            int rc = launch(p->inner, (const float2*)in, (float2*)out, count, st);
            if (rc) return rc;
            if (real_split_launch(false, out, out, count, h, p->tw_a, p->tw_b, p->rt_lb, p->sms, st))
                return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
            return FFT_OK;
        }
        if (real_split_launch(true, in, out, count, h, p->tw_a, p->tw_b, p->rt_lb, p->sms, st))
            return bfft_set_error(FFT_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        return launch(p->inner, (const float2*)out, (float2*)out, count, st);
    }
    return launch(p, (const float2*)in, (float2*)out, count, (cudaStream_t)stream);
}

extern "C" int fft_exec(const fft_plan* p, const void* in, void* out, void* stream) {
    if (!p) return bfft_set_error(FFT_E_ARG, "null plan");
    return fft_exec_range(p, in, out, p->batch, stream);
}

// ------------------------------------------------------------ partitioner
extern "C" int64_t fft_file_records(int64_t file_bytes, int64_t record_len) {
    bfft_clear_error();
    int rc = validate(record_len, 1, FFT_FORWARD);
    if (rc) return -rc;
    if (file_bytes < 0 || file_bytes % 8)
        return -bfft_set_error(FFT_E_ARG, "file size %lld is not a multiple of 8 bytes", (long long)file_bytes);
    if (file_bytes == 0) return -bfft_set_error(FFT_E_EMPTY, "empty input");
    const int64_t rb = 8 * record_len;
    return (file_bytes + rb - 1) / rb;
}

extern "C" int fft_partition(int64_t total, int nparts, int part, int64_t* first, int64_t* count) {
    bfft_clear_error();
    if (!first || !count || total < 0 || nparts < 1 || part < 0 || part >= nparts)
        return bfft_set_error(FFT_E_ARG, "invalid partition request: total=%lld nparts=%d part=%d",
                              (long long)total, nparts, part);
    // floor(part*R/G) without overflow for R up to 2^62: split R = qG + rem.
    auto bound = [&](int64_t g) {
        const int64_t q = total / nparts, rem = total % nparts;
        return q * g + (rem * g) / nparts;
    };
    *first = bound(part);
    *count = bound(part + 1) - *first;
    return FFT_OK;
}
