// synth_fill.cu — the seeded generator of synth/__init__.py as a CUDA fill
// kernel (bit-identical; checked by tests/test_gpu_parity.py).  Holds none of
// the FFT's arithmetic: SplitMix64 in counter mode,
//   out(seed, i) = mix(seed + (i + 1) * 0x9E3779B97F4A7C15),
//   f(h) = (h >> 40) * 2^-23 - 1   (exact in fp32, uniform on [-1, 1)),
// complex sample s: re = f(out(seed, 2s)), im = f(out(seed, 2s + 1)).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t sm64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float unit(uint64_t h) {
    return (float)((double)(h >> 40) * (1.0 / 8388608.0) - 1.0);
}

__global__ void k_synth_random(float2* __restrict__ out, int64_t first, int64_t count, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t s = (uint64_t)(first + i);
        out[i] = make_float2(unit(sm64(seed, 2 * s)), unit(sm64(seed, 2 * s + 1)));
    }
}

// Fill `count` complex64 samples at device pointer `out` with global samples
// [first, first + count) of the stream `seed`, on `stream`.  Returns a
// cudaError_t value (0 = success).
extern "C" int synth_fill_random(void* out, int64_t first, int64_t count, uint64_t seed, void* stream) {
    if (count <= 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (count + 255) / 256;
    const int grid = (int)(want < (int64_t)sms * 32 ? want : (int64_t)sms * 32);
    k_synth_random<<<grid, 256, 0, (cudaStream_t)stream>>>((float2*)out, first, count, seed);
    return (int)cudaGetLastError();
}
