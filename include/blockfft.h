/*
 * blockfft.h — C ABI of the B200-native per-record FFT (arXiv 1407.6915).
 *
 * The method (§III): a very large signal file is split into
 * fixed-length records ("FFT segments"), each record is
 * transformed independently by a Cooley–Tukey FFT (§I), the
 * transform is run as one batched plan over many records at once
 * ("partitioning of FFT segments can be done inside memory using CUFFT's
 * batched FFT plan"), and the outputs are written back in file
 * order ("named by their position in the original file").
 *
 * Conventions:
 *   - A record is N complex64 samples: interleaved little-endian float32
 *     (re, im), record-major, 8*N bytes (reading c1).
 *   - N is a power of two, 2 <= N <= 2^22 (reading c7).
 *   - FFT_FORWARD: X[k] = sum_j x[j] exp(-2 pi i jk/N), unnormalised.
 *     FFT_INVERSE: x[j] = (1/N) sum_k X[k] exp(+2 pi i jk/N)
 *     (readings c2/c3).
 *   - Bin k of a record's transform is at index k (natural order, c4).
 *
 * Every entry point is thread-safe.  Errors: functions returning int return
 * FFT_OK (0) or one of the FFT_E_* codes; functions returning a pointer
 * return NULL.  In both cases fft_last_error() returns a thread-local message
 * naming the offending value ("unsupported transform size" naming
 * the value; "expected vs actual").
 *
 * Nothing in this header depends on PyTorch; device pointers are plain CUDA
 * device pointers and streams are cudaStream_t passed as void*.
 */
#ifndef BLOCKFFT_H
#define BLOCKFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLOCKFFT_VERSION 1

#define FFT_FORWARD (-1) /* exp(-2 pi i jk/N), unnormalised  */
#define FFT_INVERSE (+1) /* exp(+2 pi i jk/N), scaled by 1/N     */

enum fft_status {
    FFT_OK = 0,
    FFT_E_SIZE = 1,   /* N not a power of two in [2, 2^22]                     */
    FFT_E_BATCH = 2,  /* batch < 1                                            */
    FFT_E_DIR = 3,    /* direction not -1 / +1                                */
    FFT_E_ARG = 4,    /* NULL / misaligned / partially overlapping pointers   */
    FFT_E_DEVICE = 5, /* no such device, or plan used on another device       */
    FFT_E_CUDA = 6,   /* a CUDA runtime call failed (message has its text)    */
    FFT_E_NOMEM = 7,  /* device or pinned host allocation failed              */
    FFT_E_IO = 8,     /* open/read/write/rename failed, or short read         */
    FFT_E_EMPTY = 9   /* empty input file                       */
};

/* Kernel variant of a plan.                           */
enum fft_variant {
    FFT_VARIANT_AUTO = 0,     /* choose by N (the default)                    */
    FFT_VARIANT_SINGLE = 1,   /* one kernel, record in one CTA, N <= 2^14      */
    FFT_VARIANT_CLUSTER = 2,  /* one kernel, record across a CTA cluster
                                 exchanging through DSMEM, 2^10 <= N <= 2^17   */
    FFT_VARIANT_FOURSTEP = 3, /* two kernels (column FFT + twiddle, row FFT +
                                 transposed store) through HBM scratch, N >= 256 */
    FFT_VARIANT_IDENTITY = 4, /* copy kernel: out = in bit-exactly (pipeline
                                 test mode)                      */
    FFT_VARIANT_PIPE = 5      /* four-step as ONE persistent dependency-driven
                                 kernel, intermediate in an L2-resident ring,
                                 2^14 <= N <= 2^22                            */
};

typedef struct fft_plan fft_plan; /* opaque */

/*
 * fft_plan_create — the batched plan ("CUFFT's batched FFT plan";
 * SURVEY.md §8(a) row a1; SPEC.md:42-50 plan_create).
 *   n     transform length N (power of two, 2..2^22), else FFT_E_SIZE
 *         ("unsupported transform size: <n>").
 *   batch number of records per fft_exec call (>= 1), else FFT_E_BATCH.
 *   dir   FFT_FORWARD or FFT_INVERSE, else FFT_E_DIR.
 * The plan is bound to the CUDA device current at creation.  It owns its
 * device twiddle tables (computed in fp64 on the host, rounded once to fp32)
 * and, for the four-step variant, an HBM scratch buffer of batch*8*N bytes
 * (or of one wave, see fft_plan_info).  Synchronous; allocates.
 * Returns NULL on error (see fft_last_error()).
 */
fft_plan *fft_plan_create(int64_t n, int64_t batch, int dir);

/* As fft_plan_create with an explicit kernel variant (enum fft_variant).
 * A variant that cannot handle n fails with FFT_E_SIZE.  dir may be 0 only
 * with FFT_VARIANT_IDENTITY (the bit-exact copy kernel); the
 * identity variant takes only dir 0 (else FFT_E_DIR).                       */
fft_plan *fft_plan_create_ex(int64_t n, int64_t batch, int dir, int variant);

/* Plan options (fft_plan_create_opts).  Every field 0 selects the shipped
 * default for N — the kernel measured fastest on B200 —
 * which is what fft_plan_create uses.  Non-zero values pick the measured
 * alternatives explicitly (each parity-tested, tests/test_gpu_parity.py);
 * they change speed, never the transform's definition.  No environment
 * variable changes a plan.                                                  */
typedef struct fft_plan_opts {
    int variant;      /* enum fft_variant (0 = auto)                          */
    int impl;         /* implementation inside the variant, 0 = default:
                         FFT_VARIANT_SINGLE  1 k_rows, 2 the staged kernels
                                             (k_rows_tma 2^13, k_rows_tma2 2^14);
                         FFT_VARIANT_PIPE    1 k_pipe, 2 k_pipe2, 3 k_pipe3;
                         FFT_VARIANT_CLUSTER 1 k_cluster1 (single buffer),
                                             2 k_cluster2 (pipelined),
                                             3 k_cluster (TMA-staged)          */
    int config;       /* configuration inside the implementation, 0 = default:
                         k_pipe2 1 = one compute group / two stages, 2 = two
                         groups / three stages, 3 = two groups / three 64 KiB
                         stages (2^17, 2^18); k_pipe3 0..4 = (stages, groups,
                         claim batch) sets                                     */
    int cluster_size; /* FFT_VARIANT_CLUSTER: CTAs per cluster, 0 = default */
    int ring_records; /* FFT_VARIANT_PIPE: L2 ring slots S, 0 = sized from the
                         tasks in flight (capped at 96 MiB); > 0 forces
                         max(S, LAG + 1) — e.g. to reuse slots in small batches */
    int ring_lag;     /* FFT_VARIANT_PIPE: rounds between a record's A- and
                         B-tasks (LAG), 0 = default                           */
} fft_plan_opts;

/* fft_plan_create with options (opts may be NULL = all defaults).  Negative
 * or out-of-range fields fail with FFT_E_ARG; a combination that has no
 * kernel for n fails with FFT_E_SIZE.                                        */
fft_plan *fft_plan_create_opts(int64_t n, int64_t batch, int dir, const fft_plan_opts *opts);

/*
 * fft_plan_create_real — batched transform of REAL records (SURVEY.md §8(f)
 * NEXT-1; reading c1's real reading of PAPER.md:49 "1024 ... single-precision
 * ... 4096 bytes"): n float32 samples per record, 4 <= n <= 2^23, n a power of
 * two (else FFT_E_SIZE); batch >= 1 (FFT_E_BATCH); dir FFT_FORWARD or
 * FFT_INVERSE (FFT_E_DIR).
 *   FFT_FORWARD (R2C): in = batch records of n float32 (4n bytes each), out =
 *     the packed Hermitian half spectrum, n/2 complex64 values (4n bytes):
 *       out[0] = (X[0], X[n/2])   (both are real for a real record)
 *       out[k] = X[k], 0 < k < n/2   (X[n-k] = conj(X[k]) gives the rest)
 *     with X[k] = sum_j x[j] exp(-2 pi i jk/n), unnormalised (readings c2, c3).
 *   FFT_INVERSE (C2R): the packed half spectrum -> n real samples, x[j] =
 *     (1/n) sum_k X[k] exp(+2 pi i jk/n) over the Hermitian-extended X.
 * The record is read as the n/2-point complex signal x[2m] + i x[2m+1] (the
 * same bytes), transformed by an n/2-point complex plan, and split / merged
 * with W_n^k inside the transform kernel (one launch) up to n = 2^19; longer
 * records by one more kernel (csrc/real.cu).
 * Input and output are both 4n bytes per record, so in place works and a
 * streamed real file moves half the bytes of its complex64 promotion.
 * fft_exec on such a plan: 16-byte aligned pointers to batch*4n bytes.
 */
fft_plan *fft_plan_create_real(int64_t n, int64_t batch, int dir);

/*
 * fft_plan_create_stft — overlapping records: the short-time Fourier
 * transform of a complex64 signal (the
 * paper's future work).  Frame f (0 <= f < frames) is the n samples starting
 * at sample f*hop, multiplied by window[0..n) (host pointer, n float32,
 * copied into the plan; NULL = rectangular):
 *   out[f][k] = sum_j window[j] in[f*hop + j] exp(-+2 pi i jk/n)   (dir as in
 *   fft_plan_create; FFT_INVERSE scales by 1/n per frame).
 * hop >= 1 (hop < n overlaps frames, hop == n is the record transform, hop > n
 * skips samples), else FFT_E_ARG; n, frames, dir as in fft_plan_create.
 * fft_exec(plan, in, out, stream): in = the signal, (frames-1)*hop + n
 * complex64 samples; out = frames*n complex64; in and out must not overlap.
 * Frames are framed and windowed on load by the transform kernel itself (one
 * launch) for any hop up to 2^14 points and an even hop above; an odd hop
 * above 2^14 points is framed into out by one more kernel and transformed in
 * place.
 */
fft_plan *fft_plan_create_stft(int64_t n, int64_t hop, int64_t frames, int dir, const float *window);

/*
 * fft_exec — transform `batch` records.
 *   in, out  device pointers to batch*N complex64 values, 16-byte aligned,
 *            caller-owned.  in == out (in place) is allowed; partial overlap
 *            is FFT_E_ARG.
 *   stream   cudaStream_t (as void*; NULL = legacy default stream).
 * Enqueues the plan's kernels on `stream` and returns: no allocation, no host
 * synchronisation, no host<->device copy — graph-capturable.  Argument errors
 * are returned synchronously; launch errors as FFT_E_CUDA; device faults
 * surface at the caller's next synchronisation.  Every variant enqueues only
 * kernel launches (the pipelined four-step encodes its TMA tensor map on the
 * host and resets its own counters at the end of each launch, no memset).
 * Concurrency: plans with fft_plan_info.exclusive == 0 (single-pass,
 * cluster, identity) are immutable and may run concurrently on several
 * streams; plans with exclusive == 1 (FFT_VARIANT_PIPE: L2 ring + dependency
 * counters; FFT_VARIANT_FOURSTEP: HBM scratch) must not run concurrently
 * with themselves — order their execs on one stream, or create one plan per
 * stream (as cuFFT requires).  This narrows SPEC.md:96 deliberately.
 */
int fft_exec(const fft_plan *plan, const void *in, void *out, void *stream);

/* Like fft_exec on the first `count` records at in/out (1 <= count <= batch);
 * the caller offsets the pointers.  Used by the streamer for partial chunks. */
int fft_exec_range(const fft_plan *plan, const void *in, void *out, int64_t count, void *stream);

/* Release a plan (NULL-safe).  The caller must have synchronised every stream
 * the plan was executed on.                                                  */
void fft_plan_destroy(fft_plan *plan);

typedef struct fft_plan_info {
    int64_t n, batch;
    int dir;
    int variant;          /* enum fft_variant actually used                    */
    int kernels_per_exec; /* kernel launches one fft_exec enqueues            */
    int device;
    int64_t n1, n2;       /* four-step / cluster split N = n1*n2 (else n, 1)   */
    int cluster;          /* CTAs per cluster (cluster variant), else 1        */
    int64_t scratch_bytes;/* HBM scratch owned by the plan                     */
    int64_t table_bytes;  /* device twiddle tables owned by the plan           */
    int resident;         /* co-resident clusters (cluster variant) or CTAs per
                             SM of the first kernel (other variants)          */
    int exclusive;        /* 1: the plan owns mutable device state (ring,
                             counters, scratch) and must not run concurrently
                             with itself (see fft_exec)                       */
    int ring_records;     /* FFT_VARIANT_PIPE: L2 ring slots S (else 0)      */
    int ring_lag;         /* FFT_VARIANT_PIPE: LAG (else 0)                  */
    int real;             /* 1: a real-record plan (fft_plan_create_real); n is
                             the real record length, the other fields describe
                             its n/2-point complex plan                        */
    int64_t hop;          /* STFT plan (fft_plan_create_stft): samples between
                             frames (else 0)                                   */
} fft_plan_info;

/* Fill *info for a plan.  Returns FFT_OK or FFT_E_ARG.                       */
int fft_plan_get_info(const fft_plan *plan, fft_plan_info *info);

/*
 * Partitioner (SURVEY.md §8(a) row a7; PAPER.md:49 "offset", :53 one block
 * per map task, :63 outputs named by position; SPEC.md:141-149 split_plan).
 * fft_file_records: R = ceil(file_bytes / (8*record_len)) records (the final
 *   record zero-padded).  Returns R, or -FFT_E_* (< 0).
 * fft_partition: contiguous range of part `part` of `nparts`:
 *   first = floor(part*R/nparts), count = floor((part+1)*R/nparts) - first.
 *   All arithmetic is int64 (2^40-byte files overflow 32 bits).
 *   Returns FFT_OK or FFT_E_ARG.
 */
int64_t fft_file_records(int64_t file_bytes, int64_t record_len);
int fft_partition(int64_t total_records, int nparts, int part, int64_t *first, int64_t *count);

/* Per-chunk timeline (fft_stream_opts.timeline): FFT_TIMELINE_FIELDS doubles
 * per chunk, seconds from the pipeline's start on one clock: read start, read
 * end, H2D start, H2D end, FFT end, D2H end, write start, write end (reads
 * and writes are 0 for pinned memory sources/sinks, which are copied directly).
 * The overlap evidence of the streamer.                      */
#define FFT_TIMELINE_FIELDS 8

typedef struct fft_stream_opts {
    int64_t chunk_bytes;  /* bytes per pipeline chunk (the paper's block,
                             PAPER.md:55-61 dfs.block.size); 0 = default 256 MiB,
                             or env BLOCKFFT_CHUNK_BYTES                         */
    int depth;            /* chunks in flight per GPU (>= 2); 0 = default 3      */
    int variant;          /* enum fft_variant for the per-chunk plan (0=auto)  */
    int io_threads;       /* host threads splitting each chunk's pread/pwrite; 0 = 8 */
    int direct_io;        /* 1: file I/O with O_DIRECT (page cache bypassed) when
                             records are 4 KiB multiples (N >= 512) and the file
                             system supports it; else buffered.  stats.direct_io
                             reports what was used                               */
    int numa;             /* 0: pinned slots on the GPU's NUMA node and pipeline
                             threads on its cores (default); -1: no binding      */
    const int64_t *tap_records; /* optional, strictly increasing logical record
                             indices whose outputs are copied to tap_out as they
                             stream past (sampled parity of long streams; exact
                             when a ring sink holds >= depth chunks)            */
    int64_t tap_count;
    void *tap_out;        /* tap_count * 8 * n bytes                              */
    double *timeline;     /* optional FFT_TIMELINE_FIELDS doubles per chunk       */
    int64_t timeline_chunks; /* capacity of timeline, in chunks                   */
    int real;             /* 1: REAL records (fft_plan_create_real): a record is n
                             float32 samples in, n/2 packed complex64 bins out
                             (or back, inverse), 4n bytes both ways; a file holds
                             ceil(bytes / 4n) records (size a multiple of 4)    */
    int64_t hop;          /* > 0: STFT (fft_plan_create_stft) of the file's
                             complex64 signal of L samples: F = 1 + ceil((L-n)/hop)
                             frames (L <= n: 1), samples past L read as zero;
                             output F*n complex64.  Each chunk reads its frames'
                             samples including the n - hop halo it shares with
                             the next chunk or GPU (re-read, no exchange).  Files
                             only (fft_file_ex, fft_file_range)                 */
    const float *window;  /* STFT window, window_len = n floats (NULL = none)  */
    int64_t window_len;
} fft_stream_opts;

typedef struct fft_stream_stats {
    int64_t records;      /* records transformed (all GPUs)                     */
    int64_t chunks;       /* chunks processed (all GPUs)                        */
    int64_t bytes_in;     /* input bytes moved host->device                     */
    int64_t bytes_out;    /* output bytes moved device->host                    */
    double wall_s;        /* first read to last write                           */
    double read_s;        /* summed per-chunk host read time (file source)      */
    double h2d_s;         /* summed per-chunk H2D copy time (CUDA events)       */
    double fft_s;         /* summed per-chunk kernel time (CUDA events)         */
    double d2h_s;         /* summed per-chunk D2H copy time (CUDA events)       */
    double write_s;       /* summed per-chunk host write time (file sink)       */
    int ngpu;
    int numa_node;        /* NUMA node the pinned slots were bound to (-1: none) */
    int direct_io;        /* 1 if the file I/O used O_DIRECT                      */
    int64_t taps;         /* tapped records filled                              */
} fft_stream_stats;

/*
 * fft_file — the whole method on a file (north_star; §III).
 *   in_path      headerless complex64 little-endian file; size must be a
 *                multiple of 8 bytes (else FFT_E_ARG); empty -> FFT_E_EMPTY.
 *   out_path     written as out_path + ".tmp" then renamed; its
 *                size is R*8*record_len with the final record zero-padded
 *                (SPEC.md:188).  On failure the .tmp is removed and out_path
 *                is untouched.
 *   record_len   N, validated as in fft_plan_create.
 *   ngpu         devices 0..ngpu-1 (1 <= ngpu <= device count, else
 *                FFT_E_DEVICE).  GPU g transforms the contiguous record range
 *                fft_partition(R, ngpu, g) and writes it at byte offset
 *                first*8*N of the output — no merge step, no collective
 *                (PAPER.md:63 zero reducers; reading c5).
 * Forward direction.  Per GPU: pread -> pinned buffer -> H2D (copy stream) ->
 * fft_exec (compute stream) -> D2H (second copy stream) -> pwrite, `depth`
 * chunks in flight so copies overlap compute in both directions
 * (SURVEY.md §8(a) row a8).
 */
int fft_file(const char *in_path, const char *out_path, int64_t record_len, int ngpu);

/* fft_file with direction, options (may be NULL) and stats (may be NULL).
 * dir may also be 0 for the identity kernel (bit-exact copy).  */
int fft_file_ex(const char *in_path, const char *out_path, int64_t record_len, int ngpu,
                int dir, const fft_stream_opts *opts, fft_stream_stats *stats);

/*
 * fft_exec_host — transform `batch` records held in HOST memory on one GPU
 * through the same chunked, overlapped streamer as fft_file (memory source
 * and sink instead of a file).
 *   host_in, host_out  host pointers, batch*8*n bytes each; may be equal.
 *                      Pinned (cudaHostAlloc / registered) buffers are copied
 *                      directly; pageable ones are staged through the
 *                      streamer's pinned ring.
 *   device             CUDA device index.
 *   dir                FFT_FORWARD, FFT_INVERSE, or 0 (identity).
 * Synchronous: returns when host_out holds the result.
 */
int fft_exec_host(int64_t n, int64_t batch, int dir, const void *host_in, void *host_out,
                  int device, const fft_stream_opts *opts, fft_stream_stats *stats);

/*
 * fft_stream_host — the streamer over host-memory RINGS: logical record r
 * (0 <= r < total_records) is read from record r mod in_records of host_in
 * and its transform written to record r mod out_records of host_out.  A
 * capture buffer replayed as an endless signal, a rolling output buffer; with
 * in_records = out_records = total_records it is fft_exec_host.  Pinned
 * (cudaHostAlloc / registered) rings are copied directly; pageable ones are
 * staged.  Synchronous.  Errors as fft_exec_host, plus FFT_E_ARG for ring
 * sizes < 1.  (the 1 TiB logical stream.)
 */
int fft_stream_host(int64_t n, int64_t total_records, int dir, const void *host_in, int64_t in_records,
                    void *host_out, int64_t out_records, int device, const fft_stream_opts *opts,
                    fft_stream_stats *stats);

/*
 * fft_file_range — one GPU's share of fft_file, for launchers that run one
 * process per GPU or per node (the paper's map tasks over a shared file,
 * PAPER.md:53, :111-115): records
 * [first_record, first_record + count) of in_path (R = fft_file_records) are
 * transformed on `device` and written at byte offset first_record*8*n of
 * out_path, which is opened without truncation and never renamed — its owner
 * pre-sizes it to R*8*n bytes and renames it once every range has finished
 * (paper_1407_6915_b200.dist.fan_out).  count = 0 is a no-op.
 * FFT_E_ARG if the range exceeds R; other errors as fft_file_ex.
 */
int fft_file_range(const char *in_path, const char *out_path, int64_t record_len, int dir,
                   int64_t first_record, int64_t count, int device, const fft_stream_opts *opts,
                   fft_stream_stats *stats);

/* NUMA node of a CUDA device from sysfs (-1 if unknown); the node the
 * streamer binds its pinned slots and threads to.                          */
int fft_numa_node(int device);

/* Pinned host memory on `device`'s NUMA node (cudaHostAlloc while the calling
 * thread prefers that node), for sources and sinks of fft_stream_host.  NULL
 * on error (FFT_E_ARG, FFT_E_DEVICE, FFT_E_NOMEM).  Free with fft_host_free. */
void *fft_host_alloc(int64_t bytes, int device);
void fft_host_free(void *p);

/* Host-link roofline of the streamer: copies `bytes`
 * between pinned host buffers and `device`, best of `reps` after a warm-up,
 * timed with CUDA events.  gbs[0] = H2D GB/s alone, gbs[1] = D2H alone,
 * gbs[2] / gbs[3] = H2D / D2H while both directions run at once (best round),
 * gbs[4] = GB/s each way sustained over all `reps` concurrent rounds (gbs
 * holds 5 doubles).  Run it on several GPUs from several threads at the same
 * time for the aggregate roofline.  Returns FFT_OK or FFT_E_ARG /
 * FFT_E_DEVICE / FFT_E_CUDA.                                               */
int fft_link_probe(int device, const void *host_src, void *host_dst, int64_t bytes, int reps, double *gbs);

/* The streamer (fft_file*, fft_exec_host) caches its per-GPU resources
 * (plan, streams, device slots, pinned staging) between calls, keyed by
 * (device, n, dir, variant, chunk records, depth); fft_stream_release frees
 * every cached set not in use and returns how many it freed.              */
int fft_stream_release(void);

/*
 * One transform larger than a GPU (the out-of-card /
 * GPU-cluster FFTs of PAPER.md:41, :43): ONE record of n complex64 points held
 * as ngpu contiguous slabs, GPU g owning points [g n/ngpu, (g+1) n/ngpu).
 * fft_dplan_create: n a power of two, 4 <= n <= 2^44, n = n1 n2 with n1 =
 * 2^ceil(log2(n)/2) <= 2^22 and n1, n2 multiples of ngpu (else FFT_E_SIZE);
 * ngpu a power of two <= device count whose GPUs can all reach each other as
 * peers (NVLink / NVSwitch), else FFT_E_DEVICE; devices = the ngpu CUDA device
 * ids (NULL = 0..ngpu-1); dir FFT_FORWARD / FFT_INVERSE (1/n).  Owns per GPU
 * two scratch slabs (2 n/ngpu complex64), twiddle tables and two batched plans.
 * fft_dplan_exec: slabs_in[g] / slabs_out[g] = device pointers on GPU g of
 * n/ngpu complex64 (16-byte aligned; out may equal in).  Distributed
 * four-step: three transposes, each ONE kernel per GPU that applies the
 * step's twiddle and stores every element straight into the peer GPU's buffer
 * over NVLink (the all-to-all fused with the arithmetic; no NCCL), with the
 * column and row FFTs between them.  Output slabs are in natural order.
 * Synchronous (returns when every output slab is written); not concurrent
 * with itself.  fft_dplan_geometry reports (n1, n2, ngpu).
 */
typedef struct fft_dplan fft_dplan;
fft_dplan *fft_dplan_create(int64_t n, int ngpu, const int *devices, int dir);
int fft_dplan_exec(fft_dplan *plan, void *const *slabs_in, void *const *slabs_out);
int fft_dplan_geometry(const fft_dplan *plan, int64_t *n1, int64_t *n2, int *ngpu);
void fft_dplan_destroy(fft_dplan *plan);

/* Thread-local message describing the last error on this thread ("" if none). */
const char *fft_last_error(void);

/* Thread-local FFT_* status of the last failed call on this thread (FFT_OK if
 * the last call succeeded); lets callers of the pointer-returning
 * fft_plan_create recover the code.                                          */
int fft_last_status(void);

/* BLOCKFFT_VERSION of the loaded library. */
int fft_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKFFT_H */
