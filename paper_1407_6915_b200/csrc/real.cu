// real.cu — real-input records (the
// paper's record is 1024 single-precision samples, 4096 bytes).
//
// A real record x[0..n) is read as the n/2-point complex signal
// z[m] = x[2m] + i x[2m+1] (the same bytes: no copy), transformed by the
// complex plan, and split (forward, "post") with E, O the spectra of the even
// and odd samples:
//     E[k] = (Z[k] + conj Z[n/2-k]) / 2,   O[k] = (Z[k] - conj Z[n/2-k]) / (2i),
//     X[k] = E[k] + W_n^k O[k],             X[n/2-k] = conj(E[k] - W_n^k O[k]),
// for k = 1 .. n/4 (one thread per pair; k = n/4 pairs with itself), and
// X[0] = E[0] + O[0], X[n/2] = E[0] - O[0] from Z[0] = (E[0], O[0]).  The
// output is the packed Hermitian half spectrum: out[0] = (X[0], X[n/2]) (both
// real), out[k] = X[k] for 0 < k < n/2 — n/2 complex64 values, 4n bytes, the
// size of the input.  The inverse ("pre") undoes the split:
//     E[k] = (X[k] + conj X[n/2-k]) / 2,    O[k] = (X[k] - conj X[n/2-k]) conj(W_n^k) / 2,
//     Z[k] = E[k] + i O[k],                 Z[n/2-k] = conj(E[k]) + i conj(O[k]),
// then the complex inverse of n/2 points (its 1/(n/2) and the /2 above give
// the 1/n of reading c3) leaves x[2m] = Re z[m], x[2m+1] = Im z[m].
// W_n^k = hi[k >> lb] * lo[k & (2^lb - 1)] from fp64-computed tables (one
// extra rounding).  Memory: partners k and n/2-k are read ascending and
// descending by consecutive threads: both coalesced.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "fft_device.cuh"
#include "plan_internal.h"

using namespace bfft;

namespace {

__device__ __forceinline__ float2 tw_real(const float2* __restrict__ hi, const float2* __restrict__ lo, int lb,
                                          int64_t k) {
    return cmul(__ldg(hi + (k >> lb)), __ldg(lo + (k & ((1ll << lb) - 1))));
}
__device__ __forceinline__ float2 half2(float2 a) { return __fmul2_rn(a, make_float2(0.5f, 0.5f)); }

// forward split of Z (in place in `data`): X[k] = E + W O, X[h-k] = conj(E - W O)
// inverse merge (in -> out): Z[k] = E + i O, Z[h-k] = conj(E) + i conj(O)
template <bool INV>
__global__ void __launch_bounds__(256) k_real_split(const float2* __restrict__ in, float2* __restrict__ out,
                                                     int64_t nrec, int64_t h, const float2* __restrict__ hi,
                                                     const float2* __restrict__ lo, int lb) {
    const int64_t pairs = h / 2 + 1;   // k = 0 .. h/2
    // a block takes 256 consecutive k of one record: one division per block, not per element
    const int64_t bpr = (pairs + 255) / 256;
    for (int64_t bt = blockIdx.x; bt < nrec * bpr; bt += gridDim.x) {
        const int64_t r = bt / bpr, k = (bt - r * bpr) * 256 + threadIdx.x;
        if (k >= pairs) continue;
        const float2* src = in + r * h;
        float2* dst = out + r * h;
        if (k == 0) {
            const float2 a = src[0];
            if (!INV) {
                dst[0] = make_float2(a.x + a.y, a.x - a.y);                    // (X[0], X[h])
            } else {
                dst[0] = make_float2(0.5f * (a.x + a.y), 0.5f * (a.x - a.y));  // (E[0], O[0])
            }
            continue;
        }
        const float2 a = src[k], b = src[h - k];
        const float2 w = tw_real(hi, lo, lb, k);
        const float2 e = half2(cadd(a, conjf2(b)));
        const float2 dlt = half2(csub(a, conjf2(b)));
        if (!INV) {
            const float2 o = mul_mi(dlt);                   // (A - conj B) / (2i)
            const float2 wo = cmul(o, w);
            dst[k] = cadd(e, wo);
            if (h - k != k) dst[h - k] = conjf2(csub(e, wo));
        } else {
            const float2 o = cmul(dlt, conjf2(w));          // (A - conj B) conj(W) / 2
            dst[k] = cadd(e, mul_pi(o));                    // E + i O
            if (h - k != k) dst[h - k] = cadd(conjf2(e), mul_pi(conjf2(o)));
        }
    }
}

}  // namespace

int real_split_launch(bool inv, const void* in, void* out, int64_t nrec, int64_t h, const void* hi, const void* lo,
                      int lb, int sms, cudaStream_t st) {
    const int64_t total = nrec * (h / 2 + 1);
    const int threads = 256;
    const int grid = (int)std::min<int64_t>((total + threads - 1) / threads, (int64_t)sms * 8);
    if (inv)
        k_real_split<true><<<grid, threads, 0, st>>>((const float2*)in, (float2*)out, nrec, h, (const float2*)hi,
                                                     (const float2*)lo, lb);
    else
        k_real_split<false><<<grid, threads, 0, st>>>((const float2*)in, (float2*)out, nrec, h, (const float2*)hi,
                                                      (const float2*)lo, lb);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
