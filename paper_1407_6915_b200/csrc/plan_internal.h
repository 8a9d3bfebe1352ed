// plan_internal.h — kernel descriptors shared by the plan layer (plan.cu) and
// the separately compiled kernel units (kern_*.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace bfft {
struct RealTw;   // fft_kernels.cuh
}

struct KernelSet {
    const void* fn = nullptr;
    int threads = 0;
    size_t smem = 0;
    int cols = 0;
    int pp = 16;
};

struct PipeChoice {
    int n1 = 0, n2 = 0, cols = 0, rows = 0, impl = 1, boxr = 0, stages = 0, pp = 16;
    int twm = 0;   // four-step twiddle mode (fft_pipe.cuh TW_TREE / TW_TABLE / TW_SPLIT)
    KernelSet k;
};

struct ClusterChoice {
    int n1 = 0, n2 = 0, c = 0, pp = 16, impl = 0;
    KernelSet k;
};

// kernel signatures, by family (launch casts KernelSet::fn to these)
using RowFn = void (*)(const float2*, float2*, int64_t, const float2*, float, int64_t, const float*, bfft::RealTw);
using RowTmaFn = void (*)(const float2*, float2*, int64_t, const float2*, float, bfft::RealTw, int64_t, const float*);
using ColFn = void (*)(const float2*, float2*, int64_t, int, const float2*);
using RowTFn = void (*)(const float2*, float2*, int64_t, int, const float2*, float);
using ClusterFn = void (*)(const CUtensorMap, float2*, int64_t, const float2*, const float2*, float);
using Cluster1Fn = void (*)(const float2*, float2*, int64_t, const float2*, const float2*, float);
using Cluster2Fn = void (*)(const float2*, float2*, int64_t, float);
using PipeFn = void (*)(const float2*, float2*, float2*, int64_t, int*, int, int, float, const float2*,
                        const float2*, int);

using Pipe2Fn = void (*)(const CUtensorMap, float2*, float2*, int64_t, int*, int, int, float, const float2*,
                         const float2*, int, const float*, bfft::RealTw);

// kern_rows.cu: single-pass row kernel for 2^log2l; four-step column / row kernels
KernelSet pick_row(int log2l, bool inv);
// kern_rows.cu: the staged single-pass kernel (k_rows_tma) for 2^log2l, or an
// empty set where k_rows is the faster kernel (same twiddle table as pick_row)
KernelSet pick_row_tma(int log2l, bool inv);
KernelSet pick_row_real_tma(int log2l, bool inv);
// kern_rows.cu: the single-pass kernel with the real-record split (R2C, !inv)
// or merge (C2R, inv) fused, for real records of n = 2^(log2l+1) points
KernelSet pick_row_real(int log2l, bool inv);
KernelSet pick_fs_col(int log2l, int n2, bool inv);
KernelSet pick_fs_row(int log2l, bool inv);
// kern_cluster.cu: cluster kernel for 2^log2n (want_c = requested cluster size or 0)
ClusterChoice pick_cluster(int log2n, int want_c, bool inv, int impl);
// kern_pipe.cu: pipelined four-step (k_pipe / k_pipe2, or k_pipe3 through pick_pipe3)
PipeChoice pick_pipe(int log2n, bool inv, int impl, int config);
// kern_pipe.cu: k_pipe2 with the forward real split fused (complex length
// 2^log2n; empty choice where none is built)
PipeChoice pick_pipe_real(int log2n);
// kern_pipe.cu: k_pipe2 with the inverse real merge fused into the A-task read
PipeChoice pick_pipe_real_inv(int log2n);
// each kernel unit's copy of the constant twiddles (same contents as plan.cu's); 0 on success
int rows_upload_const(const float2* host, size_t count);
int cluster_upload_const(const float2* host, size_t count);
int pipe_upload_const(const float2* host, size_t count);

// kern_pipe3.cu: k_pipe3 (compute groups with early stage release) for 2^log2n
// (empty choice if that size has no k_pipe3 configuration)
PipeChoice pick_pipe3(int log2n, bool inv, int config);
// the constant-memory twiddles of kern_pipe3.cu's translation unit (same
// contents and layout as plan.cu's c_tw); 0 on success
int pipe3_upload_const(const float2* host, size_t count);

// real.cu: the real-record split (forward, in place on the n/2-point complex
// spectrum) or merge (inverse, packed half spectrum -> Z) of h = n/2 points per
// record; 0 on success
int real_split_launch(bool inv, const void* in, void* out, int64_t nrec, int64_t h, const void* hi, const void* lo,
                      int lb, int sms, cudaStream_t st);
