// stream.cpp — out-of-core streamer and the file entry points (fft_file /
// fft_file_ex / fft_file_range / fft_exec_host / fft_stream_host;
// include/blockfft.h).
//
// The paper moves one 512 MB HDFS block to the GPU with a single synchronous
// allocate+copy pair, runs the batched FFT, copies back and writes a part file
// per map task (§III).  Here each GPU runs a chunk
// pipeline with three host threads:
//   reader     reads chunk k into the pinned input slot k mod D (file or
//              pageable memory; skipped when the source is pinned memory);
//   submitter  enqueues H2D on a copy stream, fft_exec_range on a compute
//              stream and D2H on a second copy stream, ordered by events;
//   writer     waits for chunk k's D2H, writes the pinned output slot at the
//              chunk's byte offset (file or pageable memory), copies tapped
//              records, accounts per-stage times.
// Input and output slots are separate, so reading chunk k + D overlaps writing
// chunk k, and D chunks are in flight, so the host-link copies overlap the
// kernels in both directions (the PCIe link, not the GPU, is the
// bottleneck — "minimize memory transfers").  Pinned buffers are allocated on
// the GPU's NUMA node and the pipeline threads run on that node's cores.
// GPU g owns the contiguous record range fft_partition(R, G, g) and writes it
// at byte offset first*8N of one pre-sized output file: the zero-reducer
// design of PAPER.md:63 with the -getmerge step gone and no collective.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <sys/types.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cerrno>
#include <chrono>
#include <condition_variable>
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

// ------------------------------------------------------------------ NUMA
// The GPU's NUMA node from sysfs (no libnuma in the image): -1 if unknown.
int gpu_numa_node(int device) {
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    for (char* p = bus; *p; ++p) *p = (char)tolower(*p);
    char path[128];
    snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
}

bool node_cpus(int node, cpu_set_t* set) {
    char path[96];
    snprintf(path, sizeof path, "/sys/devices/system/node/node%d/cpulist", node);
    FILE* f = fopen(path, "r");
    if (!f) return false;
    char buf[4096];
    const bool ok = fgets(buf, sizeof buf, f) != nullptr;
    fclose(f);
    if (!ok) return false;
    CPU_ZERO(set);
    int n = 0;
    for (char* p = buf; *p && *p != '\n';) {
        char* e;
        long a = strtol(p, &e, 10), b = a;
        if (e == p) break;
        if (*e == '-') b = strtol(e + 1, &e, 10);
        for (long c = a; c <= b && c < CPU_SETSIZE; ++c, ++n) CPU_SET((int)c, set);
        p = (*e == ',') ? e + 1 : e;
    }
    return n > 0;
}

constexpr int kMpolDefault = 0, kMpolPreferred = 1;   // <numaif.h> values

// Binds the calling thread's CPU affinity and page-allocation preference to
// `node` for its lifetime (restored by the destructor).  node < 0: no-op.
struct NumaScope {
    bool aff = false, pol = false;
    cpu_set_t saved;
    explicit NumaScope(int node) {
        if (node < 0) return;
        cpu_set_t set;
        if (node_cpus(node, &set) && sched_getaffinity(0, sizeof saved, &saved) == 0)
            aff = sched_setaffinity(0, sizeof set, &set) == 0;
        unsigned long mask[16] = {0};
        if (node < 1024) {
            mask[node / 64] = 1ul << (node % 64);
            pol = syscall(SYS_set_mempolicy, kMpolPreferred, mask, 1024ul) == 0;
        }
    }
    ~NumaScope() {
        if (aff) sched_setaffinity(0, sizeof saved, &saved);
        if (pol) syscall(SYS_set_mempolicy, kMpolDefault, nullptr, 0ul);
    }
};

// ------------------------------------------------------------------ sources / sinks
// A span of pinned host memory holding consecutive records.
struct Span {
    char* p;
    int64_t bytes;
};

// A source yields the bytes [off, off+len) of the logical input stream; a
// sink consumes bytes at their offsets of the output.  Pinned memory sources
// and sinks expose the bytes directly (up to two spans: rings wrap), else the
// reader / writer copy through a pinned slot.  Offsets are bytes so a chunk of
// STFT frames can read its halo (the N - hop samples it shares with the next).
struct Source {
    virtual ~Source() = default;
    virtual int direct(int64_t off, int64_t len, Span out[2]) { (void)off; (void)len; (void)out; return 0; }
    virtual int read(int64_t off, int64_t len, void* dst) = 0;
};
struct Sink {
    virtual ~Sink() = default;
    virtual int direct(int64_t off, int64_t len, Span out[2]) { (void)off; (void)len; (void)out; return 0; }
    virtual int write(int64_t off, int64_t len, const void* src) = 0;
};

int io_err(const char* what, const char* path, int64_t off, int64_t want, int64_t got, int err) {
    return bfft_set_error(FFT_E_IO, "%s %s at offset %lld: expected %lld bytes, got %lld (%s)", what, path,
                          (long long)off, (long long)want, (long long)got, got < 0 ? strerror(err) : "short");
}

int pread_full(int fd, void* buf, int64_t len, int64_t off, int64_t* got, int* err) {
    char* p = (char*)buf;
    int64_t done = 0;
    while (done < len) {
        ssize_t r = pread(fd, p + done, (size_t)std::min<int64_t>(len - done, 1ll << 30), off + done);
        if (r < 0) {
            if (errno == EINTR) continue;
            *got = -1;
            *err = errno;
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

// A chunk's pread/pwrite split over `nt` threads (>= 8 MiB each, 4 KiB-aligned
// pieces so O_DIRECT stays aligned): one thread moves only a few GB/s, the
// host's memory system far more (I/O dominates).  The pieces
// always cover exactly len bytes (ceiling division).
template <class F>
int parallel_io(int64_t len, int nt, F&& piece) {
    const int64_t min_piece = 8ll << 20;
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, len / min_piece));
    if (nt == 1) return piece(0, len);
    std::vector<std::thread> th;
    std::vector<int> rc(nt, 0);
    const int64_t step = (((len + nt - 1) / nt) + 4095) & ~4095ll;
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

// File source: bytes past EOF read as zero (the final record or frame is
// zero-padded, reading c6).  With O_DIRECT the read of the
// last partial block is rounded up to 4 KiB (the pinned slot has room: slots
// are whole 4 KiB-multiple records then).
struct FileSource : Source {
    int fd;
    int64_t size;
    const char* path;
    int nt;
    bool odirect;
    FileSource(int f, int64_t s, const char* p, int threads, bool od)
        : fd(f), size(s), path(p), nt(threads), odirect(od) {}
    int read(int64_t off, int64_t len, void* dst) override {
        const int64_t avail = std::max<int64_t>(0, std::min<int64_t>(len, size - off));
        if (avail > 0) {
            const int64_t want = odirect ? std::min<int64_t>(len, (avail + 4095) & ~4095ll) : avail;
            int64_t bad_got = 0, bad_off = 0, bad_want = 0;
            int bad_err = 0;
            std::mutex m;
            int r = parallel_io(want, nt, [&](int64_t a, int64_t n) {
                int64_t got = 0;
                int err = 0;
                const int64_t need = std::max<int64_t>(0, std::min<int64_t>(n, avail - a));
                if (pread_full(fd, (char*)dst + a, n, off + a, &got, &err) != 0 || got < need) {
                    std::lock_guard<std::mutex> g(m);
                    bad_got = got;
                    bad_off = off + a;
                    bad_want = need;
                    bad_err = err;
                    return 1;
                }
                return 0;
            });
            if (r) return io_err("short read of", path, bad_off, bad_want, bad_got, bad_err);
        }
        if (avail < len) memset((char*)dst + avail, 0, (size_t)(len - avail));
        return FFT_OK;
    }
};
struct FileSink : Sink {
    int fd;
    const char* path;
    int nt;
    FileSink(int f, const char* p, int threads) : fd(f), path(p), nt(threads) {}
    int write(int64_t off, int64_t len, const void* src) override {
        std::atomic<int> err{0};
        int r = parallel_io(len, nt, [&](int64_t a, int64_t n) {
            if (pwrite_full(fd, (const char*)src + a, n, off + a) != 0) {
                err = errno;
                return 1;
            }
            return 0;
        });
        if (r)
            return bfft_set_error(FFT_E_IO, "write of %s at offset %lld failed: %s", path, (long long)off,
                                  strerror(err.load()));
        return FFT_OK;
    }
};
// Host-memory ring source / sink (fft_stream_host, fft_exec_host): logical
// byte b lives at ring byte b mod cap (cap = ring records x record bytes).
// Pinned memory is copied directly.
int ring_spans(char* base, int64_t cap, int64_t off, int64_t len, Span out[2]) {
    const int64_t s = off % cap, n1 = std::min<int64_t>(len, cap - s);
    out[0] = Span{base + s, n1};
    if (n1 == len) return 1;
    out[1] = Span{base, len - n1};
    return 2;
}
struct MemSource : Source {
    char* base;
    int64_t cap;
    bool pinned;
    MemSource(const void* b, int64_t c, bool pin) : base((char*)b), cap(c), pinned(pin) {}
    int direct(int64_t off, int64_t len, Span out[2]) override {
        return pinned ? ring_spans(base, cap, off, len, out) : 0;
    }
    int read(int64_t off, int64_t len, void* dst) override {
        Span sp[2];
        const int ns = ring_spans(base, cap, off, len, sp);
        char* d = (char*)dst;
        for (int i = 0; i < ns; ++i) {
            memcpy(d, sp[i].p, (size_t)sp[i].bytes);
            d += sp[i].bytes;
        }
        return FFT_OK;
    }
};
struct MemSink : Sink {
    char* base;
    int64_t cap;
    bool pinned;
    MemSink(void* b, int64_t c, bool pin) : base((char*)b), cap(c), pinned(pin) {}
    int direct(int64_t off, int64_t len, Span out[2]) override {
        return pinned ? ring_spans(base, cap, off, len, out) : 0;
    }
    int write(int64_t off, int64_t len, const void* src) override {
        Span sp[2];
        const int ns = ring_spans(base, cap, off, len, sp);
        const char* s = (const char*)src;
        for (int i = 0; i < ns; ++i) {
            memcpy(sp[i].p, s, (size_t)sp[i].bytes);
            s += sp[i].bytes;
        }
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
        s.taps += o.taps;
        if (o.numa_node >= 0) s.numa_node = o.numa_node;
        s.direct_io |= o.direct_io;
    }
};

struct Opts {
    int64_t chunk_bytes = 256ll << 20;
    int depth = 3;
    int variant = FFT_VARIANT_AUTO;
    int io_threads = 8;
    int direct_io = 0;
    int numa = 0;
    const int64_t* tap_records = nullptr;
    int64_t tap_count = 0;
    char* tap_out = nullptr;
    double* timeline = nullptr;
    int64_t timeline_chunks = 0;
    int real = 0;
    int64_t hop = 0;              // > 0: STFT frames every hop samples (fft_plan_create_stft)
    std::vector<float> window;    // STFT window (empty = rectangular)
};

// Runtime options of the streamer: the chunk size is the paper's one tunable
// (dfs.block.size); BLOCKFFT_CHUNK_BYTES sets its default.
Opts resolve(const fft_stream_opts* o) {
    Opts r;
    if (const char* e = getenv("BLOCKFFT_CHUNK_BYTES")) r.chunk_bytes = std::max(1ll, atoll(e));
    if (o) {
        if (o->chunk_bytes > 0) r.chunk_bytes = o->chunk_bytes;
        if (o->depth >= 2) r.depth = o->depth;
        r.variant = o->variant;
        if (o->io_threads > 0) r.io_threads = o->io_threads;
        r.direct_io = o->direct_io;
        r.numa = o->numa;
        r.tap_records = o->tap_records;
        r.tap_count = o->tap_out ? o->tap_count : 0;
        r.tap_out = (char*)o->tap_out;
        r.timeline = o->timeline;
        r.timeline_chunks = o->timeline ? o->timeline_chunks : 0;
        r.real = o->real != 0;
        r.hop = o->hop;
        if (o->hop > 0 && o->window) r.window.assign(o->window, o->window + o->window_len);
    }
    return r;
}

// bytes per record: n complex64 (8n), or n float32 / n/2 packed complex64 (4n)
int64_t rec_bytes(int64_t n, const Opts& o) { return o.real ? 4 * n : 8 * n; }

// Byte geometry of the logical input and output streams, per record (or STFT
// frame) f: input bytes [f*in_rb, f*in_rb + in_rb + in_extra) — in_extra > 0
// is the halo an STFT frame shares with the next — output [f*out_rb, +out_rb).
struct Geom {
    int64_t in_rb, in_extra, out_rb;
    int64_t in_off(int64_t f) const { return f * in_rb; }
    int64_t in_len(int64_t cnt) const { return cnt * in_rb + in_extra; }
};
Geom geom_of(int64_t n, const Opts& o) {
    if (o.hop > 0) return Geom{8 * o.hop, 8 * (n - o.hop), 8 * n};
    return Geom{rec_bytes(n, o), 0, rec_bytes(n, o)};
}

int check_opts(const fft_stream_opts* o) {
    if (!o) return FFT_OK;
    if (o->chunk_bytes < 0 || o->depth < 0 || o->io_threads < 0 || o->tap_count < 0 || o->timeline_chunks < 0)
        return bfft_set_error(FFT_E_ARG, "invalid stream options: chunk_bytes=%lld depth=%d io_threads=%d "
                              "tap_count=%lld timeline_chunks=%lld", (long long)o->chunk_bytes, o->depth,
                              o->io_threads, (long long)o->tap_count, (long long)o->timeline_chunks);
    if (o->hop < 0 || (o->hop > 0 && o->real))
        return bfft_set_error(FFT_E_ARG, "invalid stream options: hop=%lld real=%d (STFT frames are complex)",
                              (long long)o->hop, o->real);
    if (o->hop > 0 && o->window && o->window_len <= 0)
        return bfft_set_error(FFT_E_ARG, "window_len must be the frame length: %lld", (long long)o->window_len);
    if (o->tap_count > 0 && (!o->tap_records || !o->tap_out))
        return bfft_set_error(FFT_E_ARG, "tap_count %lld needs tap_records and tap_out", (long long)o->tap_count);
    for (int64_t i = 1; i < o->tap_count; ++i)
        if (o->tap_records[i] <= o->tap_records[i - 1])
            return bfft_set_error(FFT_E_ARG, "tap_records must be strictly increasing (index %lld)", (long long)i);
    return FFT_OK;
}

// Per-GPU pipeline resources (plan, streams, events, device slots, pinned
// slots), cached across calls: allocating and freeing hundreds of MiB of
// device and pinned memory per call costs tens of ms and synchronises the
// device.  A context is used by one call at a time; fft_stream_release()
// frees every idle context.
struct StreamCtx {
    int device = 0, dir = 0, variant = 0, depth = 0, node = -1, real = 0;
    int64_t n = 0, crec = 0, hop = 0;
    std::vector<float> window;
    bool stage_in = false, stage_out = false, busy = false;
    fft_plan* plan = nullptr;
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    cudaEvent_t base = nullptr;
    std::vector<cudaEvent_t> e0, e1, e2, e3;
    std::vector<void*> dbuf, dout, hin, hout;   // dout: STFT output slots (records: in place in dbuf)
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
        if (base) cudaEventDestroy(base);
        for (auto* v : {&dbuf, &dout})
            for (void* b : *v)
                if (b) cudaFree(b);
        for (auto* v : {&hin, &hout})
            for (void* b : *v)
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

int ctx_fail(StreamCtx* c, StreamCtx** out, int rc) {
    c->release();
    delete c;
    *out = nullptr;
    return rc;
}
#define CKC(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return ctx_fail(c, out, bfft_set_error(FFT_E_CUDA, "%s failed: %s", #call,              \
                                                   cudaGetErrorString(e_)));                        \
    } while (0)

int acquire_ctx(int device, int64_t n, int dir, const Opts& o, const Geom& g, int64_t crec, int D, bool stage_in,
                bool stage_out, int node, StreamCtx** out) {
    {
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        for (StreamCtx* c : g_ctx)
            if (!c->busy && c->device == device && c->n == n && c->dir == dir && c->variant == o.variant &&
                c->crec == crec && c->depth == D && c->stage_in == stage_in && c->stage_out == stage_out &&
                c->node == node && c->real == o.real && c->hop == o.hop && c->window == o.window) {
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
    c->variant = o.variant;
    c->crec = crec;
    c->depth = D;
    c->stage_in = stage_in;
    c->stage_out = stage_out;
    c->node = node;
    c->real = o.real;
    c->hop = o.hop;
    c->window = o.window;
    c->busy = true;
    CKC(cudaSetDevice(device));
    if (o.hop > 0)
        c->plan = fft_plan_create_stft(n, o.hop, crec, dir, o.window.empty() ? nullptr : o.window.data());
    else if (o.real)
        c->plan = fft_plan_create_real(n, crec, dir);
    else
        c->plan = fft_plan_create_ex(n, crec, dir, dir == 0 ? FFT_VARIANT_IDENTITY : o.variant);
    if (!c->plan) {
        const int code = bfft_last_code();
        delete c;
        *out = nullptr;
        return code;  // message already set by the plan layer
    }
    CKC(cudaStreamCreateWithFlags(&c->sh, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->sd, cudaStreamNonBlocking));
    CKC(cudaEventCreate(&c->base));
    for (auto* v : {&c->e0, &c->e1, &c->e2, &c->e3}) {
        v->assign(D, nullptr);
        for (int i = 0; i < D; ++i) CKC(cudaEventCreate(&(*v)[i]));
    }
    c->dbuf.assign(D, nullptr);
    c->dout.assign(D, nullptr);
    c->hin.assign(D, nullptr);
    c->hout.assign(D, nullptr);
    const size_t in_bytes = (size_t)g.in_len(crec), out_bytes = (size_t)(crec * g.out_rb);
    const bool separate = o.hop > 0;   // STFT: output slot apart from the (overlapping) input
    NumaScope numa(node);   // pinned slots on the GPU's NUMA node (first touch happens in cudaHostAlloc)
    for (int i = 0; i < D; ++i) {
        const size_t dbytes = separate ? in_bytes : std::max(in_bytes, out_bytes);
        cudaError_t e = cudaMalloc(&c->dbuf[i], dbytes);
        if (e == cudaSuccess && separate) e = cudaMalloc(&c->dout[i], out_bytes);
        if (e != cudaSuccess)
            return ctx_fail(c, out, bfft_set_error(FFT_E_NOMEM, "cudaMalloc(%zu) for stream slot failed: %s", dbytes,
                                                   cudaGetErrorString(e)));
        if (stage_in) e = cudaHostAlloc(&c->hin[i], in_bytes, cudaHostAllocPortable);
        if (e == cudaSuccess && stage_out) e = cudaHostAlloc(&c->hout[i], out_bytes, cudaHostAllocPortable);
        if (e != cudaSuccess)
            return ctx_fail(c, out, bfft_set_error(FFT_E_NOMEM, "cudaHostAlloc for stream slot failed: %s",
                                                   cudaGetErrorString(e)));
    }
    std::lock_guard<std::mutex> lk(g_ctx_mu);
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

// Progress counters shared by the reader, submitter and writer of one pipeline.
struct Progress {
    std::mutex mu;
    std::condition_variable cv;
    int64_t loaded = 0, submitted = 0, written = 0;
    int rc = FFT_OK;
    std::string msg;
    void fail(int code) {
        std::lock_guard<std::mutex> g(mu);
        if (rc == FFT_OK) {
            rc = code;
            msg = fft_last_error();
        }
        cv.notify_all();
    }
    // wait until pred() or a failure; returns false on failure
    template <class P>
    bool wait(P pred) {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return rc != FFT_OK || pred(); });
        return rc == FFT_OK;
    }
    void set(int64_t& field, int64_t v) {
        std::lock_guard<std::mutex> g(mu);
        field = v;
        cv.notify_all();
    }
};

// The per-GPU pipeline over logical records [first, first+count).
int run_pipeline(int device, int64_t n, int dir, int64_t first, int64_t count, Source* src, Sink* dst,
                 const Opts& o, fft_stream_stats* st) {
    const Geom g = geom_of(n, o);
    const int64_t rb = g.out_rb;
    const int64_t crec = std::max<int64_t>(1, std::min<int64_t>(count, o.chunk_bytes / std::max(g.in_rb, g.out_rb)));
    const int D = o.depth;
    Span probe[2];
    const bool stage_in = src->direct(g.in_off(first), g.in_len(1), probe) == 0;
    const bool stage_out = dst->direct(first * rb, rb, probe) == 0;
    const int node = o.numa < 0 ? -1 : gpu_numa_node(device);
    st->numa_node = node;
    StreamCtx* c = nullptr;
    int rc = acquire_ctx(device, n, dir, o, g, crec, D, stage_in, stage_out, node, &c);
    if (rc) return rc;
    const int64_t nchunks = (count + crec - 1) / crec;
    auto chunk_first = [&](int64_t k) { return first + k * crec; };
    auto chunk_count = [&](int64_t k) { return std::min<int64_t>(crec, first + count - chunk_first(k)); };
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess)
        rc = bfft_set_error(FFT_E_CUDA, "cudaSetDevice(%d) failed: %s", device, cudaGetErrorString(ce));
    // host/GPU clock alignment for the timeline: the base event completes ~t0
    double t0 = now_s();
    if (rc == FFT_OK) {
        cudaEventRecord(c->base, c->sh);
        cudaEventSynchronize(c->base);
        t0 = now_s();
    }
    Progress pg;
    if (rc) pg.rc = rc;
    double read_s = 0, write_s = 0, h2d_s = 0, fft_s = 0, d2h_s = 0;
    int64_t taps = 0;
    double* tl = o.timeline;
    auto tl_set = [&](int64_t k, int f, double v) {
        if (k < o.timeline_chunks) tl[k * FFT_TIMELINE_FIELDS + f] = v;
    };

    // ---------------------------------------------------------------- reader
    std::thread reader;
    if (stage_in && pg.rc == FFT_OK) {
        reader = std::thread([&]() {
            NumaScope numa(node);
            cudaSetDevice(device);
            for (int64_t k = 0; k < nchunks; ++k) {
                const int i = (int)(k % D);
                if (k >= D) {   // the slot's previous chunk must have left the pinned input slot
                    if (!pg.wait([&] { return pg.submitted > k - D; })) return;
                    cudaError_t e = cudaEventSynchronize(c->e1[i]);
                    if (e != cudaSuccess) {
                        pg.fail(bfft_set_error(FFT_E_CUDA, "pipeline failed: %s", cudaGetErrorString(e)));
                        return;
                    }
                }
                const double a = now_s();
                const int r = src->read(g.in_off(chunk_first(k)), g.in_len(chunk_count(k)), c->hin[i]);
                const double b = now_s();
                read_s += b - a;
                tl_set(k, 0, a - t0);
                tl_set(k, 1, b - t0);
                if (r) {
                    pg.fail(r);
                    return;
                }
                pg.set(pg.loaded, k + 1);
            }
        });
    }
    // ---------------------------------------------------------------- writer
    std::thread writer([&]() {
        NumaScope numa(node);
        cudaSetDevice(device);
        int64_t tap = 0;
        while (tap < o.tap_count && o.tap_records[tap] < first) ++tap;
        for (int64_t k = 0; k < nchunks; ++k) {
            const int i = (int)(k % D);
            if (!pg.wait([&] { return pg.submitted > k; })) return;
            cudaError_t e = cudaEventSynchronize(c->e3[i]);
            if (e != cudaSuccess) {
                pg.fail(bfft_set_error(FFT_E_CUDA, "pipeline failed: %s", cudaGetErrorString(e)));
                return;
            }
            float a = 0, b = 0, cc = 0, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
            cudaEventElapsedTime(&a, c->e0[i], c->e1[i]);
            cudaEventElapsedTime(&b, c->e1[i], c->e2[i]);
            cudaEventElapsedTime(&cc, c->e2[i], c->e3[i]);
            h2d_s += a * 1e-3;
            fft_s += b * 1e-3;
            d2h_s += cc * 1e-3;
            if (k < o.timeline_chunks) {
                cudaEventElapsedTime(&s0, c->base, c->e0[i]);
                cudaEventElapsedTime(&s1, c->base, c->e1[i]);
                cudaEventElapsedTime(&s2, c->base, c->e2[i]);
                cudaEventElapsedTime(&s3, c->base, c->e3[i]);
                tl_set(k, 2, s0 * 1e-3);
                tl_set(k, 3, s1 * 1e-3);
                tl_set(k, 4, s2 * 1e-3);
                tl_set(k, 5, s3 * 1e-3);
            }
            const int64_t f = chunk_first(k), cnt = chunk_count(k);
            const char* outp = nullptr;   // this chunk's output in host memory
            Span sp[2];
            if (stage_out) {
                const double t_a = now_s();
                const int r = dst->write(f * rb, cnt * rb, c->hout[i]);
                const double t_b = now_s();
                write_s += t_b - t_a;
                tl_set(k, 6, t_a - t0);
                tl_set(k, 7, t_b - t0);
                if (r) {
                    pg.fail(r);
                    return;
                }
                outp = (const char*)c->hout[i];
            } else {
                dst->direct(f * rb, cnt * rb, sp);
                tl_set(k, 6, now_s() - t0);
                tl_set(k, 7, now_s() - t0);
            }
            // taps: copies of selected records' outputs (sampled parity of long streams)
            for (; tap < o.tap_count && o.tap_records[tap] < f + cnt; ++tap) {
                const int64_t j = o.tap_records[tap] - f;
                const char* rec = nullptr;
                if (outp) {
                    rec = outp + j * rb;
                } else {
                    const int64_t n0 = sp[0].bytes / rb;
                    rec = j < n0 ? sp[0].p + j * rb : sp[1].p + (j - n0) * rb;
                }
                memcpy(o.tap_out + tap * rb, rec, (size_t)rb);
                ++taps;
            }
            pg.set(pg.written, k + 1);
        }
    });
    // ---------------------------------------------------------------- submitter
    for (int64_t k = 0; k < nchunks; ++k) {
        const int i = (int)(k % D);
        const int64_t f = chunk_first(k), cnt = chunk_count(k);
        // slot i free (its previous chunk retired by the writer), input loaded
        if (!pg.wait([&] { return pg.written > k - D && (!stage_in || pg.loaded > k); })) break;
        char* dptr = (char*)c->dbuf[i];
        char* optr = c->dout[i] ? (char*)c->dout[i] : dptr;   // STFT: separate output slot
        const int64_t in_len = g.in_len(cnt);
        Span sp[2];
        auto fail_cuda = [&](const char* what, cudaError_t e) {
            pg.fail(bfft_set_error(FFT_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e)));
        };
#define CKL(call)                               \
        if ((ce = (call)) != cudaSuccess) {     \
            fail_cuda(#call, ce);               \
            break;                              \
        }
        if (!stage_in) {   // pinned source: no read stage
            tl_set(k, 0, 0.0);
            tl_set(k, 1, 0.0);
        }
        CKL(cudaStreamWaitEvent(c->sh, c->e3[i], 0));   // device slot's previous D2H done
        CKL(cudaEventRecord(c->e0[i], c->sh));
        if (stage_in) {
            CKL(cudaMemcpyAsync(dptr, c->hin[i], (size_t)in_len, cudaMemcpyHostToDevice, c->sh));
        } else {
            const int ns = src->direct(g.in_off(f), in_len, sp);
            int64_t off = 0;
            for (int s = 0; s < ns; ++s) {
                if ((ce = cudaMemcpyAsync(dptr + off, sp[s].p, (size_t)sp[s].bytes, cudaMemcpyHostToDevice, c->sh)) !=
                    cudaSuccess)
                    break;
                off += sp[s].bytes;
            }
            if (ce != cudaSuccess) {
                fail_cuda("cudaMemcpyAsync(H2D)", ce);
                break;
            }
        }
        CKL(cudaEventRecord(c->e1[i], c->sh));
        CKL(cudaStreamWaitEvent(c->sc, c->e1[i], 0));
        rc = fft_exec_range(c->plan, dptr, optr, cnt, c->sc);
        if (rc) {
            pg.fail(rc);
            break;
        }
        CKL(cudaEventRecord(c->e2[i], c->sc));
        CKL(cudaStreamWaitEvent(c->sd, c->e2[i], 0));
        if (stage_out) {
            CKL(cudaMemcpyAsync(c->hout[i], optr, (size_t)(cnt * rb), cudaMemcpyDeviceToHost, c->sd));
        } else {
            const int ns = dst->direct(f * rb, cnt * rb, sp);
            int64_t off = 0;
            for (int s = 0; s < ns; ++s) {
                if ((ce = cudaMemcpyAsync(sp[s].p, optr + off, (size_t)sp[s].bytes, cudaMemcpyDeviceToHost, c->sd)) !=
                    cudaSuccess)
                    break;
                off += sp[s].bytes;
            }
            if (ce != cudaSuccess) {
                fail_cuda("cudaMemcpyAsync(D2H)", ce);
                break;
            }
        }
        CKL(cudaEventRecord(c->e3[i], c->sd));
#undef CKL
        st->records += cnt;
        st->chunks += 1;
        st->bytes_in += in_len;
        pg.set(pg.submitted, k + 1);
    }
    if (reader.joinable()) reader.join();
    writer.join();
    rc = pg.rc;
    if (rc) {
        cudaStreamSynchronize(c->sh);
        cudaStreamSynchronize(c->sc);
        cudaStreamSynchronize(c->sd);
        bfft_set_error(rc, "%s", pg.msg.c_str());
    } else {
        st->bytes_out += count * rb;
    }
    st->read_s += read_s;
    st->write_s += write_s;
    st->h2d_s += h2d_s;
    st->fft_s += fft_s;
    st->d2h_s += d2h_s;
    st->taps += taps;
    release_ctx(c, rc != FFT_OK);
    return rc;
}

int check_n_dir(int64_t n, int dir, bool real) {
    if ((real ? (n < 4 || n > (1 << 23)) : (n < 2 || n > (1 << 22))) || (n & (n - 1)))
        return bfft_set_error(FFT_E_SIZE, "unsupported transform size: %lld", (long long)n);
    if (dir != FFT_FORWARD && dir != FFT_INVERSE && (dir != 0 || real))
        return bfft_set_error(FFT_E_DIR, real ? "direction must be -1 or +1: %d"
                                              : "direction must be -1, +1 or 0 (identity): %d", dir);
    return FFT_OK;
}

// records (or STFT frames) of a file: ceil(size / record bytes), the final
// one zero-padded (reading c6); STFT over L = size/8 samples:
// F = 1 + ceil((L - n) / hop) frames (L <= n: one zero-padded frame)
int64_t file_records_of(int64_t size, int64_t n, const Opts& o) {
    if (o.hop > 0) {
        if (size % 8)
            return -bfft_set_error(FFT_E_ARG, "file size %lld is not a multiple of 8 bytes", (long long)size);
        if (size == 0) return -bfft_set_error(FFT_E_EMPTY, "empty input");
        const int64_t L = size / 8;
        return L <= n ? 1 : 1 + (L - n + o.hop - 1) / o.hop;
    }
    if (!o.real) return fft_file_records(size, n);
    if (size % 4)
        return -bfft_set_error(FFT_E_ARG, "file size %lld is not a multiple of 4 bytes", (long long)size);
    if (size == 0) return -bfft_set_error(FFT_E_EMPTY, "empty input");
    return (size + 4 * n - 1) / (4 * n);
}

int check_device(int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    if (device < 0 || device >= ndev)
        return bfft_set_error(FFT_E_DEVICE, "no such device: %d (visible devices: %d)", device, ndev);
    return FFT_OK;
}

// O_DIRECT needs 4 KiB-aligned offsets and lengths: records of 8N bytes with N >= 512.
bool direct_ok(const Opts& o, int64_t n) {
    const Geom g = geom_of(n, o);
    return o.direct_io && g.in_rb % 4096 == 0 && g.in_extra % 4096 == 0 && g.out_rb % 4096 == 0;
}

int open_input(const char* path, bool od, int* fd, int* fd_direct, int64_t* size) {
    *fd = open(path, O_RDONLY);
    if (*fd < 0) return bfft_set_error(FFT_E_IO, "cannot open %s: %s", path, strerror(errno));
    struct stat sb;
    if (fstat(*fd, &sb) != 0) {
        close(*fd);
        return bfft_set_error(FFT_E_IO, "cannot stat %s: %s", path, strerror(errno));
    }
    *size = sb.st_size;
    *fd_direct = -1;
    if (od) *fd_direct = open(path, O_RDONLY | O_DIRECT);   // falls back to buffered if unsupported
    return FFT_OK;
}

}  // namespace

extern "C" int fft_stream_host(int64_t n, int64_t total_records, int dir, const void* host_in, int64_t in_records,
                               void* host_out, int64_t out_records, int device, const fft_stream_opts* opts,
                               fft_stream_stats* stats) {
    bfft_clear_error();
    if (!host_in || !host_out) return bfft_set_error(FFT_E_ARG, "null host pointer");
    const bool real = opts && opts->real;
    int rc = check_n_dir(n, dir, real);
    if (rc) return rc;
    if (total_records < 1) return bfft_set_error(FFT_E_BATCH, "batch must be >= 1: %lld", (long long)total_records);
    if (in_records < 1 || out_records < 1)
        return bfft_set_error(FFT_E_ARG, "ring sizes must be >= 1: in_records=%lld out_records=%lld",
                              (long long)in_records, (long long)out_records);
    if ((rc = check_opts(opts)) || (rc = check_device(device))) return rc;
    if (opts && opts->hop > 0)
        return bfft_set_error(FFT_E_ARG, "STFT streaming (hop > 0) takes files (fft_file_ex / fft_file_range)");
    const Opts o = resolve(opts);
    MemSource src(host_in, in_records * rec_bytes(n, o), is_pinned(host_in));
    MemSink dst(host_out, out_records * rec_bytes(n, o), is_pinned(host_out));
    fft_stream_stats st{};
    st.numa_node = -1;
    const double t0 = now_s();
    rc = run_pipeline(device, n, dir, 0, total_records, &src, &dst, o, &st);
    st.wall_s = now_s() - t0;
    st.ngpu = 1;
    if (stats) *stats = st;
    return rc;
}

extern "C" int fft_exec_host(int64_t n, int64_t batch, int dir, const void* host_in, void* host_out, int device,
                             const fft_stream_opts* opts, fft_stream_stats* stats) {
    return fft_stream_host(n, batch, dir, host_in, batch, host_out, batch, device, opts, stats);
}

extern "C" int fft_file_ex(const char* in_path, const char* out_path, int64_t n, int ngpu, int dir,
                           const fft_stream_opts* opts, fft_stream_stats* stats) {
    bfft_clear_error();
    if (!in_path || !out_path) return bfft_set_error(FFT_E_ARG, "null path");
    int rc = check_n_dir(n, dir, opts && opts->real);
    if (rc) return rc;
    if ((rc = check_opts(opts))) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    if (ngpu < 1 || ngpu > ndev) return bfft_set_error(FFT_E_DEVICE, "ngpu must be in 1..%d: %d", ndev, ngpu);
    const Opts o = resolve(opts);
    const bool od = direct_ok(o, n);
    int fd = -1, fdd = -1;
    int64_t size = 0;
    if ((rc = open_input(in_path, od, &fd, &fdd, &size))) return rc;
    const int64_t R = file_records_of(size, n, o);
    const int64_t rb = geom_of(n, o).out_rb;
    if (R < 0) {
        close(fd);
        if (fdd >= 0) close(fdd);
        return (int)-R;  // message set by fft_file_records
    }
    const std::string tmp = std::string(out_path) + ".tmp";
    const int ofd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (ofd < 0) {
        close(fd);
        if (fdd >= 0) close(fdd);
        return bfft_set_error(FFT_E_IO, "cannot create %s: %s", tmp.c_str(), strerror(errno));
    }
    const int ofdd = od ? open(tmp.c_str(), O_WRONLY | O_DIRECT) : -1;
    const int64_t out_bytes = R * rb;
    if (ftruncate(ofd, out_bytes) != 0)
        rc = bfft_set_error(FFT_E_IO, "cannot size %s to %lld bytes: %s", tmp.c_str(), (long long)out_bytes,
                            strerror(errno));
    Stats agg;
    agg.s.numa_node = -1;
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
                FileSource src(fdd >= 0 ? fdd : fd, size, in_path, o.io_threads, fdd >= 0);
                FileSink dst(ofdd >= 0 ? ofdd : ofd, tmp.c_str(), o.io_threads);
                fft_stream_stats st{};
                st.direct_io = fdd >= 0 && ofdd >= 0;
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
    if (fdd >= 0) close(fdd);
    if (ofdd >= 0) close(ofdd);
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

extern "C" int fft_file_range(const char* in_path, const char* out_path, int64_t n, int dir, int64_t first_record,
                              int64_t count, int device, const fft_stream_opts* opts, fft_stream_stats* stats) {
    bfft_clear_error();
    if (!in_path || !out_path) return bfft_set_error(FFT_E_ARG, "null path");
    int rc = check_n_dir(n, dir, opts && opts->real);
    if (rc) return rc;
    if ((rc = check_opts(opts))) return rc;
    const Opts o = resolve(opts);
    const bool od = direct_ok(o, n);
    int fd = -1, fdd = -1;
    int64_t size = 0;
    if ((rc = open_input(in_path, od, &fd, &fdd, &size))) return rc;
    const int64_t R = file_records_of(size, n, o);
    auto done = [&](int code) {
        close(fd);
        if (fdd >= 0) close(fdd);
        return code;
    };
    if (R < 0) return done((int)-R);
    if (first_record < 0 || count < 0 || first_record + count > R)
        return done(bfft_set_error(FFT_E_ARG, "record range out of bounds: first=%lld count=%lld, file has %lld records",
                                   (long long)first_record, (long long)count, (long long)R));
    if ((rc = check_device(device))) return done(rc);
    fft_stream_stats st{};
    st.numa_node = -1;
    st.ngpu = 1;
    if (count == 0) {
        if (stats) *stats = st;
        return done(FFT_OK);
    }
    // the output is shared by every range (one process per GPU / node): no
    // truncation, no rename here; its owner pre-sizes it and renames it when
    // every range has finished (paper_1407_6915_b200.dist.fan_out)
    const int ofd = open(out_path, O_WRONLY | O_CREAT, 0644);
    if (ofd < 0) return done(bfft_set_error(FFT_E_IO, "cannot open %s: %s", out_path, strerror(errno)));
    const int ofdd = od ? open(out_path, O_WRONLY | O_DIRECT) : -1;
    FileSource src(fdd >= 0 ? fdd : fd, size, in_path, o.io_threads, fdd >= 0);
    FileSink dst(ofdd >= 0 ? ofdd : ofd, out_path, o.io_threads);
    st.direct_io = fdd >= 0 && ofdd >= 0;
    const double t0 = now_s();
    rc = run_pipeline(device, n, dir, first_record, count, &src, &dst, o, &st);
    st.wall_s = now_s() - t0;
    if (ofdd >= 0) close(ofdd);
    if (close(ofd) != 0 && rc == FFT_OK)
        rc = bfft_set_error(FFT_E_IO, "close of %s failed: %s", out_path, strerror(errno));
    if (stats) *stats = st;
    return done(rc);
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

extern "C" int fft_numa_node(int device) { return gpu_numa_node(device); }

extern "C" void* fft_host_alloc(int64_t bytes, int device) {
    bfft_clear_error();
    if (bytes <= 0) {
        bfft_set_error(FFT_E_ARG, "bytes must be > 0: %lld", (long long)bytes);
        return nullptr;
    }
    if (check_device(device)) return nullptr;
    NumaScope numa(gpu_numa_node(device));
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        bfft_set_error(FFT_E_NOMEM, "cudaHostAlloc(%lld) failed: %s", (long long)bytes, cudaGetErrorString(e));
        return nullptr;
    }
    return p;
}

extern "C" void fft_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// Host-link probe: H2D alone, D2H alone and both directions at once between
// pinned host buffers and a device buffer of `bytes`, best of `reps` (CUDA
// events).  gbs[0] = H2D GB/s, gbs[1] = D2H GB/s, gbs[2] / gbs[3] = H2D / D2H
// GB/s while both run concurrently on two streams.
extern "C" int fft_link_probe(int device, const void* host_src, void* host_dst, int64_t bytes, int reps,
                              double* gbs) {
    bfft_clear_error();
    if (!host_src || !host_dst || !gbs || bytes <= 0 || reps < 1)
        return bfft_set_error(FFT_E_ARG, "invalid link probe arguments");
    int rc = check_device(device);
    if (rc) return rc;
    cudaSetDevice(device);
    void *da = nullptr, *db = nullptr;
    cudaStream_t s1 = nullptr, s2 = nullptr;
    cudaEvent_t ev[6] = {};
    cudaError_t e = cudaMalloc(&da, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMalloc(&db, (size_t)bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreate(&ev[i]);
    double best[4] = {0, 0, 0, 0};
    double sum_t = 0;   // concurrent rounds: total time (sustained rate)
    for (int r = 0; r < reps + 1 && e == cudaSuccess; ++r) {   // one warm-up round
        float t0 = 0, t1 = 0, t2 = 0, t3 = 0;
        cudaEventRecord(ev[0], s1);
        cudaMemcpyAsync(da, host_src, (size_t)bytes, cudaMemcpyHostToDevice, s1);
        cudaEventRecord(ev[1], s1);
        cudaMemcpyAsync(host_dst, db, (size_t)bytes, cudaMemcpyDeviceToHost, s1);
        cudaEventRecord(ev[2], s1);
        cudaStreamSynchronize(s1);
        cudaEventElapsedTime(&t0, ev[0], ev[1]);
        cudaEventElapsedTime(&t1, ev[1], ev[2]);
        cudaEventRecord(ev[3], s1);
        cudaStreamWaitEvent(s2, ev[3], 0);
        cudaMemcpyAsync(da, host_src, (size_t)bytes, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(host_dst, db, (size_t)bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(ev[4], s1);
        cudaEventRecord(ev[5], s2);
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        cudaEventElapsedTime(&t2, ev[3], ev[4]);
        cudaEventElapsedTime(&t3, ev[3], ev[5]);
        e = cudaGetLastError();
        if (r == 0) continue;
        sum_t += std::max(t2, t3) * 1e-3;
        const double g[4] = {bytes / (t0 * 1e-3) / 1e9, bytes / (t1 * 1e-3) / 1e9, bytes / (t2 * 1e-3) / 1e9,
                             bytes / (t3 * 1e-3) / 1e9};
        if (g[0] > best[0]) best[0] = g[0];
        if (g[1] > best[1]) best[1] = g[1];
        if (g[2] + g[3] > best[2] + best[3]) {
            best[2] = g[2];
            best[3] = g[3];
        }
    }
    if (e != cudaSuccess) rc = bfft_set_error(FFT_E_CUDA, "link probe failed: %s", cudaGetErrorString(e));
    for (int i = 0; i < 6; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    if (s1) cudaStreamDestroy(s1);
    if (s2) cudaStreamDestroy(s2);
    if (da) cudaFree(da);
    if (db) cudaFree(db);
    for (int i = 0; i < 4; ++i) gbs[i] = best[i];
    gbs[4] = sum_t > 0 ? (double)bytes * reps / sum_t / 1e9 : 0;   // sustained, each direction
    return rc;
}
