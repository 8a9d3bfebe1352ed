// dist.cu — one transform larger than a GPU (the
// out-of-card and GPU-cluster FFTs the paper cites as prior art, PAPER.md:41,
// :43): a single record of N = N1 * N2 complex64 points held as G contiguous
// slabs, one per GPU (GPU g holds x[g N/G, (g+1) N/G)), transformed with a
// distributed four-step whose transposes cross NVLink / NVSwitch as peer
// stores written by the kernels themselves — the pack kernel that computes a
// step's twiddle and transpose stores every element straight into the peer
// GPU's receive buffer, so the all-to-all and the arithmetic are one kernel
// (no NCCL, no staging copy).
//
// With n = N2 n1 + n2, k = k1 + N1 k2, R = N1/G, C = N2/G:
//   pack1  (GPU h, its rows n1 in [hR, hR+R)): x[n1][n2] -> GPU n2/C's
//          buffer A at [n2 mod C][n1]          (column records, all-to-all #1)
//   fft1   (each GPU): C records of N1 points over n1 -> A[c][k1]
//   pack2  (GPU g): A[c][k1] * W_N^{(gC+c) k1} -> GPU k1/R's buffer B at
//          [k1 mod R][gC + c]                    (twiddle + all-to-all #2)
//   fft2   (each GPU): R records of N2 points over n2 -> B[k1 mod R][k2]
//   pack3  (GPU g'): B[kl][k2] -> GPU k2/C's output slab at
//          [(k2 mod C) N1 + g'R + kl]            (natural order, all-to-all #3)
// GPU g then holds X[g N/G, (g+1) N/G) — natural order in, natural order out.
// Every pack is a 32 x 32 shared-memory tile transpose: reads are coalesced
// along the source rows, peer writes are 256-byte runs along the destination
// rows.  Steps are ordered across GPUs by events (each GPU's stream waits for
// every peer's pack before its FFT reads what the peers wrote).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/blockfft.h"
#include "common.h"
#include "fft_device.cuh"

using namespace bfft;

namespace {

// transpose tiles: TR source rows x TC source columns; a row is read as a
// TC*8-byte run, a destination row written as a TR*8-byte run
constexpr int TR = 256, TC = 64, PACK_THREADS = 1024;
constexpr size_t PACK_SMEM = sizeof(float2) * TR * (TC + 1);

struct Tw2 {   // W_N^m (or its conjugate for the inverse) = hi[m >> lb] * lo[m & mask]
    const float2* hi;
    const float2* lo;
    int lb;
    uint64_t nmask;
    __device__ __forceinline__ float2 operator()(uint64_t m) const {
        m &= nmask;
        return cmul(__ldg(hi + (m >> lb)), __ldg(lo + (m & ((1ull << lb) - 1))));
    }
};

// Generic tile transpose: element (r, c) of the local [rows][cols] matrix
// `in` (row-major) goes to dst(r, c), consecutive r landing at consecutive
// addresses; step 2 multiplies by tw((me C + r) * c) first.  Tiles are
// TR x TC (TC*8-byte reads, TR*8-byte writes); when the destination split
// DIV is a multiple of TC a tile's columns share one GPU, so the destination
// is resolved once per tile (a 64-bit division per element held the kernel
// near 2.6 TB/s).
template <int STEP>
__global__ void __launch_bounds__(PACK_THREADS, 1) k_dist_pack(const float2* __restrict__ in, int64_t rows,
                                                             int64_t cols, float2* const* __restrict__ dst,
                                                             int64_t R, int64_t C, int64_t N1, int64_t N2, int me,
                                                             Tw2 tw) {
    extern __shared__ float2 tile[];   // [TR][TC + 1]
    const int l = threadIdx.x;
    const int64_t tiles_c = (cols + TC - 1) / TC, tiles_r = (rows + TR - 1) / TR;
    //   step 1: x slab [R][N2] (n1 = me R + r, n2 = c) -> A_{c/C}[c mod C][n1]
    //   step 2: A [C][N1] (n2 = me C + r, k1 = c)     -> B_{k1/R}[k1 mod R][n2]
    //   step 3: B [R][N2] (k1 = me R + r, k2 = c)     -> out_{k2/C}[(k2 mod C) N1 + k1]
    const int64_t DIV = STEP == 2 ? R : C, STR = STEP == 2 ? N2 : N1;
    const int64_t OFF = STEP == 2 ? (int64_t)me * C : (int64_t)me * R;
    for (int64_t t = blockIdx.x; t < tiles_r * tiles_c; t += gridDim.x) {
        const int64_t r0 = (t / tiles_c) * TR, c0 = (t % tiles_c) * TC;
        __syncthreads();
        {   // load along the source rows: TC consecutive columns per row
            const int cc = l % TC;
            const int64_t c = c0 + cc;
#pragma unroll 4
            for (int rr = l / TC; rr < TR; rr += PACK_THREADS / TC) {
                const int64_t r = r0 + rr;
                if (r < rows && c < cols) {
                    float2 v = __ldcs(in + r * cols + c);
                    if (STEP == 2) v = cmul(v, tw((uint64_t)(me * C + r) * (uint64_t)c));   // W^{n2 k1}
                    tile[rr * (TC + 1) + cc] = v;
                }
            }
        }
        __syncthreads();
        {   // store along the destination rows: TR consecutive r per destination row
            const int rr = l % TR;
            const int64_t r = r0 + rr;
            if (r < rows) {
                if (DIV % TC == 0) {
                    const int64_t gd = c0 / DIV, cm0 = c0 - gd * DIV;
                    float2* __restrict__ d = dst[gd] + OFF + r;
#pragma unroll 4
                    for (int cc = l / TR; cc < TC; cc += PACK_THREADS / TR)
                        if (c0 + cc < cols) d[(cm0 + cc) * STR] = tile[rr * (TC + 1) + cc];
                } else {
                    for (int cc = l / TR; cc < TC; cc += PACK_THREADS / TR) {
                        const int64_t c = c0 + cc;
                        if (c < cols) dst[c / DIV][(c % DIV) * STR + OFF + r] = tile[rr * (TC + 1) + cc];
                    }
                }
            }
        }
    }
}

}  // namespace

struct fft_dplan {
    int64_t n = 0, n1 = 0, n2 = 0;
    int G = 0, dir = 0, lb = 0;
    std::vector<int> dev;
    std::vector<fft_plan*> p1, p2;
    std::vector<float2*> a, b, hi, lo;
    std::vector<float2**> dst;   // per GPU: 3 x G peer pointers (A buffers | B buffers | output slabs)
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;
};

static void dplan_free(fft_dplan* p) {
    if (!p) return;
    for (int g = 0; g < (int)p->dev.size(); ++g) {
        cudaSetDevice(p->dev[g]);
        if (g < (int)p->st.size() && p->st[g]) cudaStreamSynchronize(p->st[g]);
        if (g < (int)p->p1.size()) fft_plan_destroy(p->p1[g]);
        if (g < (int)p->p2.size()) fft_plan_destroy(p->p2[g]);
        for (auto* v : {&p->a, &p->b, &p->hi, &p->lo})
            if (g < (int)v->size() && (*v)[g]) cudaFree((*v)[g]);
        if (g < (int)p->dst.size() && p->dst[g]) cudaFree(p->dst[g]);
        if (g < (int)p->ev.size() && p->ev[g]) cudaEventDestroy(p->ev[g]);
        if (g < (int)p->st.size() && p->st[g]) cudaStreamDestroy(p->st[g]);
    }
    delete p;
}

#define DTRY(call)                                                                                    \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            bfft_set_error(FFT_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));              \
            return fail();                                                                            \
        }                                                                                             \
    } while (0)

extern "C" fft_dplan* fft_dplan_create(int64_t n, int ngpu, const int* devices, int dir) {
    bfft_clear_error();
    if (n < 4 || (n & (n - 1)) || n > (1ll << 44)) {
        bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
        return nullptr;
    }
    if (dir != FFT_FORWARD && dir != FFT_INVERSE) {
        bfft_set_error(FFT_E_DIR, "direction must be -1 or +1: %d", dir);
        return nullptr;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    if (ngpu < 1 || ngpu > ndev || (ngpu & (ngpu - 1))) {
        bfft_set_error(FFT_E_DEVICE, "ngpu must be a power of two in 1..%d: %d", ndev, ngpu);
        return nullptr;
    }
    int k = 0;
    while ((1ll << k) < n) ++k;
    const int k1 = (k + 1) / 2, k2 = k - k1;   // N1 >= N2, both <= 2^22
    const int64_t n1 = 1ll << k1, n2 = 1ll << k2;
    if (n1 > (1 << 22) || n2 < 2 || n1 % ngpu || n2 % ngpu) {
        bfft_set_error(FFT_E_SIZE, "unsupported transform size for %d GPUs: %lld", ngpu, (long long)n);
        return nullptr;
    }
    fft_dplan* p = new (std::nothrow) fft_dplan();
    if (!p) {
        bfft_set_error(FFT_E_NOMEM, "out of host memory");
        return nullptr;
    }
    auto fail = [&]() -> fft_dplan* {
        std::string keep = fft_last_error();
        int code = fft_last_status();
        dplan_free(p);
        bfft_set_error(code ? code : FFT_E_CUDA, "%s", keep.c_str());
        return nullptr;
    };
    p->n = n;
    p->n1 = n1;
    p->n2 = n2;
    p->G = ngpu;
    p->dir = dir;
    for (int g = 0; g < ngpu; ++g) {
        const int d = devices ? devices[g] : g;
        if (d < 0 || d >= ndev) {
            bfft_set_error(FFT_E_DEVICE, "no such device: %d", d);
            return fail();
        }
        p->dev.push_back(d);
    }
    // peer access between every pair (NVLink / NVSwitch); the packs store into peers
    for (int g = 0; g < ngpu; ++g)
        for (int h = 0; h < ngpu; ++h) {
            if (g == h) continue;
            int ok = 0;
            DTRY(cudaDeviceCanAccessPeer(&ok, p->dev[g], p->dev[h]));
            if (!ok) {
                bfft_set_error(FFT_E_DEVICE, "device %d cannot access peer %d", p->dev[g], p->dev[h]);
                return fail();
            }
            DTRY(cudaSetDevice(p->dev[g]));
            cudaError_t e = cudaDeviceEnablePeerAccess(p->dev[h], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) {
                bfft_set_error(FFT_E_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", p->dev[g], p->dev[h],
                               cudaGetErrorString(e));
                return fail();
            }
        }
    // twiddles W_N^m = hi[m >> lb] lo[m & mask], fp64 -> fp32 (reading c9); inverse: conjugates
    p->lb = (k + 1) / 2;
    const int64_t nhi = n >> p->lb, nlo = 1ll << p->lb;
    std::vector<float2> thi(nhi), tlo(nlo);
    const double sgn = dir == FFT_FORWARD ? -1.0 : 1.0;
    for (int64_t i = 0; i < nhi; ++i) {
        const double ang = sgn * 2.0 * M_PI * (double)(i << p->lb) / (double)n;
        thi[i] = make_float2((float)cos(ang), (float)sin(ang));
    }
    for (int64_t i = 0; i < nlo; ++i) {
        const double ang = sgn * 2.0 * M_PI * (double)i / (double)n;
        tlo[i] = make_float2((float)cos(ang), (float)sin(ang));
    }
    const int64_t slab = n / ngpu;
    p->a.assign(ngpu, nullptr);
    p->b.assign(ngpu, nullptr);
    p->hi.assign(ngpu, nullptr);
    p->lo.assign(ngpu, nullptr);
    p->dst.assign(ngpu, nullptr);
    p->st.assign(ngpu, nullptr);
    p->ev.assign(ngpu, nullptr);
    p->p1.assign(ngpu, nullptr);
    p->p2.assign(ngpu, nullptr);
    for (int g = 0; g < ngpu; ++g) {
        DTRY(cudaSetDevice(p->dev[g]));
        cudaError_t e = cudaMalloc(&p->a[g], slab * sizeof(float2));
        if (e == cudaSuccess) e = cudaMalloc(&p->b[g], slab * sizeof(float2));
        if (e != cudaSuccess) {
            bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%lld) of distributed scratch failed: %s",
                           (long long)(slab * 8), cudaGetErrorString(e));
            return fail();
        }
        DTRY(cudaMalloc(&p->hi[g], nhi * sizeof(float2)));
        DTRY(cudaMalloc(&p->lo[g], nlo * sizeof(float2)));
        DTRY(cudaMemcpy(p->hi[g], thi.data(), nhi * sizeof(float2), cudaMemcpyHostToDevice));
        DTRY(cudaMemcpy(p->lo[g], tlo.data(), nlo * sizeof(float2), cudaMemcpyHostToDevice));
        DTRY(cudaMalloc(&p->dst[g], 3 * ngpu * sizeof(float2*)));
        DTRY(cudaFuncSetAttribute(k_dist_pack<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
        DTRY(cudaFuncSetAttribute(k_dist_pack<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
        DTRY(cudaFuncSetAttribute(k_dist_pack<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PACK_SMEM));
        DTRY(cudaStreamCreateWithFlags(&p->st[g], cudaStreamNonBlocking));
        DTRY(cudaEventCreateWithFlags(&p->ev[g], cudaEventDisableTiming));
        p->p1[g] = fft_plan_create(n1, n2 / ngpu, dir);   // C column records of N1 points
        if (!p->p1[g]) return fail();
        p->p2[g] = fft_plan_create(n2, n1 / ngpu, dir);   // R row records of N2 points
        if (!p->p2[g]) return fail();
    }
    std::vector<float2*> tab(2 * ngpu);
    for (int g = 0; g < ngpu; ++g) {
        tab[g] = p->a[g];
        tab[ngpu + g] = p->b[g];
    }
    for (int g = 0; g < ngpu; ++g) {
        DTRY(cudaSetDevice(p->dev[g]));
        DTRY(cudaMemcpy(p->dst[g], tab.data(), 2 * ngpu * sizeof(float2*), cudaMemcpyHostToDevice));
    }
    return p;
}

extern "C" void fft_dplan_destroy(fft_dplan* p) { dplan_free(p); }

extern "C" int fft_dplan_geometry(const fft_dplan* p, int64_t* n1, int64_t* n2, int* ngpu) {
    if (!p) return bfft_set_error(FFT_E_ARG, "null plan");
    if (n1) *n1 = p->n1;
    if (n2) *n2 = p->n2;
    if (ngpu) *ngpu = p->G;
    return FFT_OK;
}

extern "C" int fft_dplan_exec(fft_dplan* p, void* const* in, void* const* out) {
    bfft_clear_error();
    if (!p || !in || !out) return bfft_set_error(FFT_E_ARG, "null plan or slab array");
    const int G = p->G;
    const int64_t R = p->n1 / G, C = p->n2 / G;
    for (int g = 0; g < G; ++g)
        if (!in[g] || !out[g] || ((uintptr_t)in[g] & 15) || ((uintptr_t)out[g] & 15))
            return bfft_set_error(FFT_E_ARG, "slab %d: null or not 16-byte aligned", g);
    int cur = 0;
    cudaGetDevice(&cur);
    auto err = [&](cudaError_t e, const char* what) {
        cudaSetDevice(cur);
        return bfft_set_error(FFT_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
    };
    // every GPU's stream waits for every peer's last pack (all-to-all complete)
    auto barrier = [&]() -> cudaError_t {
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(p->dev[g]);
            cudaError_t e = cudaEventRecord(p->ev[g], p->st[g]);
            if (e != cudaSuccess) return e;
        }
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(p->dev[g]);
            for (int h = 0; h < G; ++h)
                if (h != g) {
                    cudaError_t e = cudaStreamWaitEvent(p->st[g], p->ev[h], 0);
                    if (e != cudaSuccess) return e;
                }
        }
        return cudaSuccess;
    };
    const Tw2 tw{nullptr, nullptr, p->lb, (uint64_t)(p->n - 1)};
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->dev[0]);
    const dim3 blk(PACK_THREADS);
    auto grid_for = [&](int64_t rows, int64_t cols) {
        const int64_t t = ((rows + TR - 1) / TR) * ((cols + TC - 1) / TC);
        return (unsigned)std::min<int64_t>(t, (int64_t)sms);
    };
    cudaError_t e;
    // inputs must be readable before anyone writes: start every stream after the caller's work
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        if ((e = cudaStreamSynchronize(p->st[g])) != cudaSuccess) return err(e, "cudaStreamSynchronize");
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return err(e, "cudaDeviceSynchronize");
    // this call's output slabs: the third destination table of every GPU
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        if ((e = cudaMemcpy(p->dst[g] + 2 * G, out, G * sizeof(float2*), cudaMemcpyHostToDevice)) != cudaSuccess)
            return err(e, "destination table upload");
    }
    // ---- step 1: transpose + all-to-all into A
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        k_dist_pack<1><<<grid_for(R, p->n2), blk, PACK_SMEM, p->st[g]>>>((const float2*)in[g], R, p->n2, p->dst[g], R, C,
                                                                 p->n1, p->n2, g, tw);
        if ((e = cudaGetLastError()) != cudaSuccess) return err(e, "pack kernel launch");
    }
    if ((e = barrier()) != cudaSuccess) return err(e, "cross-GPU ordering");
    // ---- column FFTs (C records of N1), then twiddle + transpose + all-to-all into B
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        int rc = fft_exec(p->p1[g], p->a[g], p->a[g], p->st[g]);
        if (rc) {
            cudaSetDevice(cur);
            return rc;
        }
    }
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        const Tw2 t{p->hi[g], p->lo[g], p->lb, (uint64_t)(p->n - 1)};
        k_dist_pack<2><<<grid_for(C, p->n1), blk, PACK_SMEM, p->st[g]>>>(p->a[g], C, p->n1, p->dst[g] + G, R, C, p->n1,
                                                                 p->n2, g, t);
        if ((e = cudaGetLastError()) != cudaSuccess) return err(e, "pack kernel launch");
    }
    if ((e = barrier()) != cudaSuccess) return err(e, "cross-GPU ordering");
    // ---- row FFTs (R records of N2), then transpose + all-to-all into the output slabs
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        int rc = fft_exec(p->p2[g], p->b[g], p->b[g], p->st[g]);
        if (rc) {
            cudaSetDevice(cur);
            return rc;
        }
    }
    if ((e = barrier()) != cudaSuccess) return err(e, "cross-GPU ordering");
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        k_dist_pack<3><<<grid_for(R, p->n2), blk, PACK_SMEM, p->st[g]>>>(p->b[g], R, p->n2, p->dst[g] + 2 * G, R, C,
                                                                 p->n1, p->n2, g, tw);
        if ((e = cudaGetLastError()) != cudaSuccess) return err(e, "pack kernel launch");
    }
    for (int g = 0; g < G; ++g) {
        cudaSetDevice(p->dev[g]);
        if ((e = cudaStreamSynchronize(p->st[g])) != cudaSuccess) return err(e, "distributed FFT");
    }
    cudaSetDevice(cur);
    return FFT_OK;
}
