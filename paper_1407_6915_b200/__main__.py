"""Command line: the whole method on a file, plus the partition plan.

  python -m paper_1407_6915_b200 fft IN OUT --record-len N [--ngpu G] [--inverse | --identity]
                                  [--real | --hop H [--window hann|none]] [--direct-io]
                                  [--chunk-bytes B] [--force] [--report PATH]
  python -m paper_1407_6915_b200 fan-out IN OUT --record-len N [--inverse] [--real | --hop H ...]
        (one process per GPU under torchrun: every rank transforms its record range,
         rank 0 renames; the multi-node form of fft, paper_1407_6915_b200.dist.fan_out)
  python -m paper_1407_6915_b200 partition --records R --gpus G

`fft` is fft_file_ex (include/blockfft.h): IN is a headerless little-endian
complex64 file (float32 with --real: packed half spectra out; --hop: the STFT
of the file as one signal, frames every H samples, optional Hann window)
split into records of N points (final record zero-padded,
PAPER.md:49 / SURVEY.md §8(c) c6), every record is transformed on the GPUs and
written at its own offset (PAPER.md:63 zero reducers, no merge step).  The
stream statistics go to stdout (or --report) as JSON, messages to stderr.
The chunk size is the paper's one tunable (dfs.block.size):
--chunk-bytes, else the environment variable BLOCKFFT_BLOCK_SIZE.

Exit codes (SPEC.md "Invariants": stable contract for scripting): 0 success,
1 validation error (size, direction, arguments, empty input, existing output
without --force), 2 runtime error (CUDA, memory, devices), 3 I/O error (the
SPEC's "protocol" class).
"""
import argparse
import json
import os
import sys

EXIT_OK, EXIT_VALIDATION, EXIT_RUNTIME, EXIT_IO = 0, 1, 2, 3


def _exit_code(code: int) -> int:
    from . import _abi
    name = _abi.STATUS_NAMES[code] if 0 <= code < len(_abi.STATUS_NAMES) else ""
    if name in ("FFT_E_SIZE", "FFT_E_BATCH", "FFT_E_DIR", "FFT_E_ARG", "FFT_E_EMPTY"):
        return EXIT_VALIDATION
    if name == "FFT_E_IO":
        return EXIT_IO
    return EXIT_RUNTIME


def _cmd_fft(a) -> int:
    import paper_1407_6915_b200 as bf
    if os.path.exists(a.output) and not a.force:
        print(f"output exists (use --force to overwrite): {a.output}", file=sys.stderr)
        return EXIT_VALIDATION
    direction = bf.FFT_INVERSE if a.inverse else (bf.FFT_IDENTITY if a.identity else bf.FFT_FORWARD)
    chunk = a.chunk_bytes
    if chunk is None:
        env = os.environ.get("BLOCKFFT_BLOCK_SIZE")
        try:
            chunk = int(env) if env else 0
        except ValueError:
            print(f"BLOCKFFT_BLOCK_SIZE must be an integer byte count: {env!r}", file=sys.stderr)
            return EXIT_VALIDATION
    try:
        stats = bf.fft_file(a.input, a.output, a.record_len, a.ngpu, direction=direction,
                            options=_stream_options(a, chunk))
    except bf.FFTError as e:
        print(str(e), file=sys.stderr)
        return _exit_code(e.code)
    text = json.dumps({"input": a.input, "output": a.output, "record_len": a.record_len, "ngpu": a.ngpu,
                       "direction": direction, "stats": stats})
    if a.report:
        with open(a.report, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    return EXIT_OK


def _stream_options(a, chunk):
    import numpy as np
    import paper_1407_6915_b200 as bf
    window = None
    if a.hop and a.window == "hann":
        window = 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(a.record_len) / a.record_len)
    return bf.StreamOptions(chunk_bytes=chunk or 0, real=a.real, hop=a.hop or 0, window=window,
                            direct_io=a.direct_io)


def _cmd_fan_out(a) -> int:
    import torch.distributed as dist
    import paper_1407_6915_b200 as bf
    from paper_1407_6915_b200 import dist as bd
    info = bd.rank_info()
    if info.world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    direction = bf.FFT_INVERSE if a.inverse else bf.FFT_FORWARD
    try:
        st = bd.fan_out(a.input, a.output, a.record_len, direction, options=_stream_options(a, a.chunk_bytes))
    except bf.FFTError as e:
        print(str(e), file=sys.stderr)
        return _exit_code(e.code)
    finally:
        if info.world > 1 and dist.is_initialized():
            dist.destroy_process_group()
    print(json.dumps(st))
    return EXIT_OK


def _cmd_partition(a) -> int:
    import paper_1407_6915_b200 as bf
    try:
        ranges = [bf.partition(a.records, a.gpus, g) for g in range(a.gpus)]
    except bf.FFTError as e:
        print(str(e), file=sys.stderr)
        return _exit_code(e.code)
    print(json.dumps({"records": a.records, "gpus": a.gpus,
                      "ranges": [{"gpu": g, "first": f, "count": c} for g, (f, c) in enumerate(ranges)]}))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1407_6915_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("fft", help="transform every record of a complex64 file")
    f.add_argument("input")
    f.add_argument("output")
    f.add_argument("--record-len", type=int, required=True)
    f.add_argument("--ngpu", type=int, default=1)
    g = f.add_mutually_exclusive_group()
    g.add_argument("--inverse", action="store_true")
    g.add_argument("--identity", action="store_true", help="copy records unchanged (pipeline check)")
    f.add_argument("--chunk-bytes", type=int, default=None)
    f.add_argument("--force", action="store_true")
    f.add_argument("--report", default=None)
    k = f.add_mutually_exclusive_group()
    k.add_argument("--real", action="store_true", help="records of N float32 samples (packed half spectra)")
    k.add_argument("--hop", type=int, default=0, help="STFT: frames of N samples every HOP samples")
    f.add_argument("--window", choices=["none", "hann"], default="none")
    f.add_argument("--direct-io", action="store_true", help="O_DIRECT file I/O where supported")
    fo = sub.add_parser("fan-out", help="this rank's record range of a file (torchrun: one process per GPU/node)")
    fo.add_argument("input")
    fo.add_argument("output")
    fo.add_argument("--record-len", type=int, required=True)
    fo.add_argument("--inverse", action="store_true")
    fo.add_argument("--chunk-bytes", type=int, default=0)
    k2 = fo.add_mutually_exclusive_group()
    k2.add_argument("--real", action="store_true")
    k2.add_argument("--hop", type=int, default=0)
    fo.add_argument("--window", choices=["none", "hann"], default="none")
    fo.add_argument("--direct-io", action="store_true")
    p = sub.add_parser("partition", help="the contiguous record range of every GPU")
    p.add_argument("--records", type=int, required=True)
    p.add_argument("--gpus", type=int, required=True)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:       # argparse usage errors are validation errors
        return EXIT_VALIDATION if e.code else EXIT_OK
    if a.cmd == "fft":
        if a.identity and (a.real or a.hop):
            print("--identity copies complex64 records: not with --real or --hop", file=sys.stderr)
            return EXIT_VALIDATION
        return _cmd_fft(a)
    return _cmd_fan_out(a) if a.cmd == "fan-out" else _cmd_partition(a)


if __name__ == "__main__":
    sys.exit(main())
