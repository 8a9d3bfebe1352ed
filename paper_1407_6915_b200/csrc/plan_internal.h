// plan_internal.h — kernel descriptors shared by the plan layer (plan.cu) and
// the separately compiled kernel units (kern_*.cu).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

struct KernelSet {
    const void* fn = nullptr;
    int threads = 0;
    size_t smem = 0;
    int cols = 0;
    int pp = 16;
};

struct PipeChoice {
    int n1 = 0, n2 = 0, cols = 0, rows = 0, impl = 1, boxr = 0, stages = 0, pp = 16;
    KernelSet k;
};

// kern_pipe3.cu: k_pipe3 (compute groups with early stage release) for 2^log2n
// (empty choice if that size has no k_pipe3 configuration)
PipeChoice pick_pipe3(int log2n, bool inv);
// the constant-memory twiddles of kern_pipe3.cu's translation unit (same
// contents and layout as plan.cu's c_tw); 0 on success
int pipe3_upload_const(const float2* host, size_t count);
