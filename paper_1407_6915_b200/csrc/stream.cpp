// stream.cpp — out-of-core streamer and the file entry point (fft_file /
// fft_file_ex / fft_exec_host; include/blockfft.h).
//
// The paper moves one 512 MB HDFS block to the GPU with a single synchronous
// allocate+copy pair, runs the batched FFT, copies back and writes a part file
// per map task (§III).  Here one host thread per GPU
// runs a chunk pipeline: read chunk c into pinned slot c mod D, H2D on a copy
// stream, fft_exec_range on a compute stream, D2H on a second copy stream,
// write at the chunk's byte offset.  D slots are in flight, so the host-link
// copies overlap the kernels in both directions (the PCIe link,
// not the GPU, is the bottleneck — "minimize memory transfers").  GPU g owns
// the contiguous record range fft_partition(R, G, g) and writes it at byte
// offset first*8N of one pre-sized output file: the zero-reducer design of
// PAPER.md:63 with the -getmerge step gone and no collective.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blockfft.h"
#include "common.h"

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// A source yields records [first, first+count) into a host buffer; a sink
// consumes them.  Either may instead expose pinned memory for direct copies.
struct Source {
    virtual ~Source() = default;
    virtual const void* direct(int64_t first) { (void)first; return nullptr; }  // pinned, no staging
    virtual int read(int64_t first, int64_t count, void* dst) = 0;
};
struct Sink {
    virtual ~Sink() = default;
    virtual void* direct(int64_t first) { (void)first; return nullptr; }
    virtual int write(int64_t first, int64_t count, const void* src) = 0;
};

int io_err(const char* what, const char* path, int64_t off, int64_t want, int64_t got) {
    return bfft_set_error(FFT_E_IO, "%s %s at offset %lld: expected %lld bytes, got %lld (%s)", what, path,
                          (long long)off, (long long)want, (long long)got, got < 0 ? strerror(errno) : "short");
}

int pread_full(int fd, void* buf, int64_t len, int64_t off, int64_t* got) {
    char* p = (char*)buf;
    int64_t done = 0;
    while (done < len) {
        ssize_t r = pread(fd, p + done, (size_t)std::min<int64_t>(len - done, 1ll << 30), off + done);
        if (r < 0) {
            if (errno == EINTR) continue;
            *got = -1;
            return -1;
        }
        if (r == 0) break;
        done += r;
    }
    *got = done;
    return 0;
}

int pwrite_full(int fd, const void* buf, int64_t len, int64_t off) {
    const char* p = (const char*)buf;
    int64_t done = 0;
    while (done < len) {
        ssize_t r = pwrite(fd, p + done, (size_t)std::min<int64_t>(len - done, 1ll << 30), off + done);
        if (r < 0) {
            if (errno == EINTR) continue;
            return -1;
        }
        done += r;
    }
    return 0;
}

// A chunk's pread/pwrite split over `nt` threads (>= 8 MiB each): one thread
// moves only a few GB/s through the page cache, the host's memory system far
// more, and the file path is host-I/O bound (I/O dominates).
template <class F>
int parallel_io(int64_t len, int nt, F&& piece) {
    const int64_t min_piece = 8ll << 20;
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, len / min_piece));
    if (nt == 1) return piece(0, len);
    std::vector<std::thread> th;
    std::vector<int> rc(nt, 0);
    const int64_t step = ((len / nt) + 4095) & ~4095ll;
    for (int i = 0; i < nt; ++i) {
        const int64_t a = i * step, b = std::min<int64_t>(len, a + step);
        if (a >= b) break;
        th.emplace_back([&, i, a, b]() { rc[i] = piece(a, b - a); });
    }
    for (auto& t : th) t.join();
    for (int r : rc)
        if (r) return r;
    return 0;
}

// File source: record r is at byte r*rb; bytes past EOF read as zero
// (the final record is zero-padded, reading c6).
struct FileSource : Source {
    int fd;
    int64_t size, rb;
    const char* path;
    int nt;
    FileSource(int f, int64_t s, int64_t recbytes, const char* p, int threads)
        : fd(f), size(s), rb(recbytes), path(p), nt(threads) {}
    int read(int64_t first, int64_t count, void* dst) override {
        const int64_t off = first * rb, len = count * rb;
        const int64_t avail = std::max<int64_t>(0, std::min<int64_t>(len, size - off));
        if (avail > 0) {
            int64_t bad_got = 0, bad_off = 0, bad_want = 0;
            std::mutex m;
            int r = parallel_io(avail, nt, [&](int64_t a, int64_t n) {
                int64_t got = 0;
                if (pread_full(fd, (char*)dst + a, n, off + a, &got) != 0 || got != n) {
                    std::lock_guard<std::mutex> g(m);
                    bad_got = got;
                    bad_off = off + a;
                    bad_want = n;
                    return 1;
                }
                return 0;
            });
            if (r) return io_err("short read of", path, bad_off, bad_want, bad_got);
        }
        if (avail < len) memset((char*)dst + avail, 0, (size_t)(len - avail));
        return FFT_OK;
    }
};
struct FileSink : Sink {
    int fd;
    int64_t rb;
    const char* path;
    int nt;
    FileSink(int f, int64_t recbytes, const char* p, int threads) : fd(f), rb(recbytes), path(p), nt(threads) {}
    int write(int64_t first, int64_t count, const void* src) override {
        const int64_t off = first * rb;
        int err = 0;
        int r = parallel_io(count * rb, nt, [&](int64_t a, int64_t n) {
            if (pwrite_full(fd, (const char*)src + a, n, off + a) != 0) {
                err = errno;
                return 1;
            }
            return 0;
        });
        if (r)
            return bfft_set_error(FFT_E_IO, "write of %s at offset %lld failed: %s", path, (long long)off,
                                  strerror(err));
        return FFT_OK;
    }
};
// Memory source/sink (fft_exec_host).  Pinned memory is copied directly.
struct MemSource : Source {
    const char* base;
    int64_t rb;
    bool pinned;
    MemSource(const void* b, int64_t recbytes, bool pin) : base((const char*)b), rb(recbytes), pinned(pin) {}
    const void* direct(int64_t first) override { return pinned ? base + first * rb : nullptr; }
    int read(int64_t first, int64_t count, void* dst) override {
        memcpy(dst, base + first * rb, (size_t)(count * rb));
        return FFT_OK;
    }
};
struct MemSink : Sink {
    char* base;
    int64_t rb;
    bool pinned;
    MemSink(void* b, int64_t recbytes, bool pin) : base((char*)b), rb(recbytes), pinned(pin) {}
    void* direct(int64_t first) override { return pinned ? base + first * rb : nullptr; }
    int write(int64_t first, int64_t count, const void* src) override {
        memcpy(base + first * rb, src, (size_t)(count * rb));
        return FFT_OK;
    }
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

struct Stats {
    std::mutex mu;
    fft_stream_stats s{};
    void add(const fft_stream_stats& o) {
        std::lock_guard<std::mutex> g(mu);
        s.records += o.records;
        s.chunks += o.chunks;
        s.bytes_in += o.bytes_in;
        s.bytes_out += o.bytes_out;
        s.read_s += o.read_s;
        s.h2d_s += o.h2d_s;
        s.fft_s += o.fft_s;
        s.d2h_s += o.d2h_s;
        s.write_s += o.write_s;
    }
};


struct Opts {
    int64_t chunk_bytes = 256ll << 20;
    int depth = 3;
    int variant = FFT_VARIANT_AUTO;
    int io_threads = 8;
};

Opts resolve(const fft_stream_opts* o) {
    Opts r;
    if (const char* e = getenv("BLOCKFFT_CHUNK_BYTES")) r.chunk_bytes = std::max(1ll, atoll(e));
    if (o) {
        if (o->chunk_bytes > 0) r.chunk_bytes = o->chunk_bytes;
        if (o->depth >= 2) r.depth = o->depth;
        r.variant = o->variant;
        if (o->io_threads > 0) r.io_threads = o->io_threads;
    }
    return r;
}

// Per-GPU pipeline resources (plan, streams, events, device slots, pinned
// staging), cached across calls: allocating and freeing hundreds of MiB of
// device and pinned memory per call costs tens of ms and synchronises the
// device.  A context is used by one call at a time; fft_stream_release()
// frees every idle context.
struct StreamCtx {
    int device = 0, dir = 0, variant = 0, depth = 0;
    int64_t n = 0, crec = 0;
    bool staging = false, busy = false;
    fft_plan* plan = nullptr;
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    std::vector<cudaEvent_t> e0, e1, e2, e3;
    std::vector<void*> dbuf, hbuf;
    void release() {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        if (sh) cudaStreamSynchronize(sh);
        if (sc) cudaStreamSynchronize(sc);
        if (sd) cudaStreamSynchronize(sd);
        for (auto* v : {&e0, &e1, &e2, &e3})
            for (auto ev : *v)
                if (ev) cudaEventDestroy(ev);
        for (void* b : dbuf)
            if (b) cudaFree(b);
        for (void* b : hbuf)
            if (b) cudaFreeHost(b);
        if (sh) cudaStreamDestroy(sh);
        if (sc) cudaStreamDestroy(sc);
        if (sd) cudaStreamDestroy(sd);
        fft_plan_destroy(plan);
        cudaSetDevice(cur);
    }
};

std::mutex g_ctx_mu;
std::vector<StreamCtx*> g_ctx;

#define CKC(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            int rc_ = bfft_set_error(FFT_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));   \
            c->release();                                                                           \
            delete c;                                                                               \
            *out = nullptr;                                                                         \
            return rc_;                                                                             \
        }                                                                                           \
    } while (0)

int acquire_ctx(int device, int64_t n, int dir, int variant, int64_t crec, int D, bool staging, StreamCtx** out) {
    {
        std::lock_guard<std::mutex> g(g_ctx_mu);
        for (StreamCtx* c : g_ctx)
            if (!c->busy && c->device == device && c->n == n && c->dir == dir && c->variant == variant &&
                c->crec == crec && c->depth == D && c->staging == staging) {
                c->busy = true;
                *out = c;
                return FFT_OK;
            }
    }
    StreamCtx* c = new StreamCtx();
    *out = c;
    c->device = device;
    c->n = n;
    c->dir = dir;
    c->variant = variant;
    c->crec = crec;
    c->depth = D;
    c->staging = staging;
    c->busy = true;
    CKC(cudaSetDevice(device));
    c->plan = fft_plan_create_ex(n, crec, dir, dir == 0 ? FFT_VARIANT_IDENTITY : variant);
    if (!c->plan) {
        const int code = bfft_last_code();
        delete c;
        *out = nullptr;
        return code;  // message already set by the plan layer
    }
    CKC(cudaStreamCreateWithFlags(&c->sh, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->sd, cudaStreamNonBlocking));
    for (auto* v : {&c->e0, &c->e1, &c->e2, &c->e3}) {
        v->assign(D, nullptr);
        for (int i = 0; i < D; ++i) CKC(cudaEventCreate(&(*v)[i]));
    }
    c->dbuf.assign(D, nullptr);
    c->hbuf.assign(D, nullptr);
    const size_t bytes = (size_t)(crec * 8 * n);
    for (int i = 0; i < D; ++i) {
        cudaError_t e = cudaMalloc(&c->dbuf[i], bytes);
        if (e != cudaSuccess) {
            int rc = bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for stream slot failed: %s", bytes, cudaGetErrorString(e));
            c->release();
            delete c;
            *out = nullptr;
            return rc;
        }
        if (staging) {
            e = cudaHostAlloc(&c->hbuf[i], bytes, cudaHostAllocPortable);
            if (e != cudaSuccess) {
                int rc = bfft_set_error(FFT_E_NOMEM, "cudaHostAlloc(%zu) for stream slot failed: %s", bytes, cudaGetErrorString(e));
                c->release();
                delete c;
                *out = nullptr;
                return rc;
            }
        }
    }
    std::lock_guard<std::mutex> g(g_ctx_mu);
    g_ctx.push_back(c);
    return FFT_OK;
}

void release_ctx(StreamCtx* c, bool broken) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    if (broken) {  // a failed pipeline may leave work queued: do not reuse it
        for (size_t i = 0; i < g_ctx.size(); ++i)
            if (g_ctx[i] == c) {
                g_ctx.erase(g_ctx.begin() + (long)i);
                break;
            }
        c->release();
        delete c;
        return;
    }
    c->busy = false;
}

// The per-GPU pipeline over records [first, first+count).
int run_pipeline(int device, int64_t n, int dir, int64_t first, int64_t count, Source* src, Sink* dst,
                 const Opts& o, fft_stream_stats* st) {
    const int64_t rb = 8 * n;
    const int64_t crec = std::max<int64_t>(1, std::min<int64_t>(count, o.chunk_bytes / rb));
    const int D = o.depth;
    const bool staging = !src->direct(first) || !dst->direct(first);
    StreamCtx* c = nullptr;
    int rc = acquire_ctx(device, n, dir, o.variant, crec, D, staging, &c);
    if (rc) return rc;
    std::vector<int64_t> slot_first(D, -1), slot_count(D, 0);
    const int64_t nchunks = (count + crec - 1) / crec;
    auto retire = [&](int i) -> int {
        // wait for slot i's D2H, account its times, hand its output to the sink
        if (slot_first[i] < 0) return FFT_OK;
        cudaError_t e = cudaEventSynchronize(c->e3[i]);
        if (e != cudaSuccess) return bfft_set_error(FFT_E_CUDA, "pipeline failed: %s", cudaGetErrorString(e));
        float a = 0, b = 0, cc = 0;
        cudaEventElapsedTime(&a, c->e0[i], c->e1[i]);
        cudaEventElapsedTime(&b, c->e1[i], c->e2[i]);
        cudaEventElapsedTime(&cc, c->e2[i], c->e3[i]);
        st->h2d_s += a * 1e-3;
        st->fft_s += b * 1e-3;
        st->d2h_s += cc * 1e-3;
        if (!dst->direct(slot_first[i])) {
            double t0 = now_s();
            int r = dst->write(slot_first[i], slot_count[i], c->hbuf[i]);
            st->write_s += now_s() - t0;
            if (r) return r;
        }
        st->bytes_out += slot_count[i] * rb;
        slot_first[i] = -1;
        return FFT_OK;
    };
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) rc = bfft_set_error(FFT_E_CUDA, "cudaSetDevice(%d) failed: %s", device, cudaGetErrorString(ce));
    for (int64_t k = 0; rc == FFT_OK && k < nchunks; ++k) {
        const int i = (int)(k % D);
        rc = retire(i);
        if (rc) break;
        const int64_t f = first + k * crec;
        const int64_t cnt = std::min<int64_t>(crec, first + count - f);
        const void* hin = src->direct(f);
        if (!hin) {
            double t0 = now_s();
            rc = src->read(f, cnt, c->hbuf[i]);
            st->read_s += now_s() - t0;
            if (rc) break;
            hin = c->hbuf[i];
        }
        void* hout = dst->direct(f);
        if (!hout) hout = c->hbuf[i];
#define CKL(call)                                                                                       \
        if ((ce = (call)) != cudaSuccess) {                                                             \
            rc = bfft_set_error(FFT_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(ce));            \
            break;                                                                                      \
        }
        CKL(cudaEventRecord(c->e0[i], c->sh));
        CKL(cudaMemcpyAsync(c->dbuf[i], hin, (size_t)(cnt * rb), cudaMemcpyHostToDevice, c->sh));
        CKL(cudaEventRecord(c->e1[i], c->sh));
        CKL(cudaStreamWaitEvent(c->sc, c->e1[i], 0));
        rc = fft_exec_range(c->plan, c->dbuf[i], c->dbuf[i], cnt, c->sc);
        if (rc) break;
        CKL(cudaEventRecord(c->e2[i], c->sc));
        CKL(cudaStreamWaitEvent(c->sd, c->e2[i], 0));
        CKL(cudaMemcpyAsync(hout, c->dbuf[i], (size_t)(cnt * rb), cudaMemcpyDeviceToHost, c->sd));
        CKL(cudaEventRecord(c->e3[i], c->sd));
#undef CKL
        slot_first[i] = f;
        slot_count[i] = cnt;
        st->records += cnt;
        st->chunks += 1;
        st->bytes_in += cnt * rb;
    }
    for (int64_t k = nchunks; rc == FFT_OK && k < nchunks + D; ++k) rc = retire((int)(k % D));
    if (rc) {
        cudaStreamSynchronize(c->sh);
        cudaStreamSynchronize(c->sc);
        cudaStreamSynchronize(c->sd);
    }
    release_ctx(c, rc != FFT_OK);
    return rc;
}

}  // namespace

extern "C" int fft_exec_host(int64_t n, int64_t batch, int dir, const void* host_in, void* host_out, int device,
                             const fft_stream_opts* opts, fft_stream_stats* stats) {
    bfft_clear_error();
    if (!host_in || !host_out) return bfft_set_error(FFT_E_ARG, "null host pointer");
    if (n < 2 || n > (1 << 22) || (n & (n - 1)))
        return bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
    if (batch < 1) return bfft_set_error(FFT_E_BATCH, "batch must be >= 1: %lld", (long long)batch);
    if (dir != FFT_FORWARD && dir != FFT_INVERSE && dir != 0)
        return bfft_set_error(FFT_E_DIR, "direction must be -1 or +1: %d", dir);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return bfft_set_error(FFT_E_DEVICE, "no such device: %d (visible devices: %d)", device, ndev);
    }
    const Opts o = resolve(opts);
    MemSource src(host_in, 8 * n, is_pinned(host_in));
    MemSink dst(host_out, 8 * n, is_pinned(host_out));
    fft_stream_stats st{};
    const double t0 = now_s();
    int rc = run_pipeline(device, n, dir, 0, batch, &src, &dst, o, &st);
    st.wall_s = now_s() - t0;
    st.ngpu = 1;
    if (stats) *stats = st;
    return rc;
}

extern "C" int fft_file_ex(const char* in_path, const char* out_path, int64_t n, int ngpu, int dir,
                           const fft_stream_opts* opts, fft_stream_stats* stats) {
    bfft_clear_error();
    if (!in_path || !out_path) return bfft_set_error(FFT_E_ARG, "null path");
    if (n < 2 || n > (1 << 22) || (n & (n - 1)))
        return bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
    if (dir != FFT_FORWARD && dir != FFT_INVERSE && dir != 0)
        return bfft_set_error(FFT_E_DIR, "direction must be -1 or +1: %d", dir);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    if (ngpu < 1 || ngpu > ndev)
        return bfft_set_error(FFT_E_DEVICE, "ngpu must be in 1..%d: %d", ndev, ngpu);
    const int fd = open(in_path, O_RDONLY);
    if (fd < 0) return bfft_set_error(FFT_E_IO, "cannot open %s: %s", in_path, strerror(errno));
    struct stat sb;
    if (fstat(fd, &sb) != 0) {
        close(fd);
        return bfft_set_error(FFT_E_IO, "cannot stat %s: %s", in_path, strerror(errno));
    }
    const int64_t size = sb.st_size;
    const int64_t R = fft_file_records(size, n);
    if (R < 0) {
        close(fd);
        return (int)-R;  // message set by fft_file_records
    }
    const std::string tmp = std::string(out_path) + ".tmp";
    const int ofd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (ofd < 0) {
        close(fd);
        return bfft_set_error(FFT_E_IO, "cannot create %s: %s", tmp.c_str(), strerror(errno));
    }
    int rc = FFT_OK;
    const int64_t out_bytes = R * 8 * n;
    if (ftruncate(ofd, out_bytes) != 0)
        rc = bfft_set_error(FFT_E_IO, "cannot size %s to %lld bytes: %s", tmp.c_str(), (long long)out_bytes, strerror(errno));
    const Opts o = resolve(opts);
    Stats agg;
    const double t0 = now_s();
    if (rc == FFT_OK) {
        std::vector<std::thread> th;
        std::vector<int> rcs(ngpu, FFT_OK);
        std::vector<std::string> msgs(ngpu);
        for (int g = 0; g < ngpu; ++g) {
            th.emplace_back([&, g]() {
                int64_t first = 0, count = 0;
                fft_partition(R, ngpu, g, &first, &count);
                if (count == 0) return;
                FileSource src(fd, size, 8 * n, in_path, o.io_threads);
                FileSink dst(ofd, 8 * n, tmp.c_str(), o.io_threads);
                fft_stream_stats st{};
                rcs[g] = run_pipeline(g, n, dir, first, count, &src, &dst, o, &st);
                if (rcs[g]) msgs[g] = fft_last_error();
                agg.add(st);
            });
        }
        for (auto& t : th) t.join();
        for (int g = 0; g < ngpu; ++g)
            if (rcs[g]) {
                rc = rcs[g];
                bfft_set_error(rc, "gpu %d: %s", g, msgs[g].c_str());
                break;
            }
    }
    close(fd);
    if (close(ofd) != 0 && rc == FFT_OK)
        rc = bfft_set_error(FFT_E_IO, "close of %s failed: %s", tmp.c_str(), strerror(errno));
    if (rc == FFT_OK && rename(tmp.c_str(), out_path) != 0)
        rc = bfft_set_error(FFT_E_IO, "rename %s -> %s failed: %s", tmp.c_str(), out_path, strerror(errno));
    if (rc != FFT_OK) unlink(tmp.c_str());
    agg.s.wall_s = now_s() - t0;
    agg.s.ngpu = ngpu;
    if (stats) *stats = agg.s;
    return rc;
}

extern "C" int fft_stream_release(void) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    int freed = 0;
    for (size_t i = 0; i < g_ctx.size();) {
        if (!g_ctx[i]->busy) {
            g_ctx[i]->release();
            delete g_ctx[i];
            g_ctx.erase(g_ctx.begin() + (long)i);
            ++freed;
        } else {
            ++i;
        }
    }
    return freed;
}

extern "C" int fft_file(const char* in_path, const char* out_path, int64_t record_len, int ngpu) {
    return fft_file_ex(in_path, out_path, record_len, ngpu, FFT_FORWARD, nullptr, nullptr);
}
