"""Build the in-tree native libraries (no JIT cache; the .so files travel to
the GPU box with the repo snapshot).

  paper_1407_6915_b200/libblockfft.so  — the C-ABI product library
      csrc/plan.cu (plan layer + kernels), csrc/stream.cpp (streamer)
  paper_1407_6915_b200/libblockfft_stress.so — TEST build: the same library with
      the pipelined kernels compiled with -DBFFT_STRESS (random sleeps at the
      protocol's synchronisation points; tests/test_gpu_stress.py)
  synth/libsynth.so                    — seeded CUDA fill kernel (inputs only)

All CUDA code is compiled for sm_100a only:
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo (no fast-math).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
LIB = os.path.join(PKG, "libblockfft.so")
STRESS_LIB = os.path.join(PKG, "libblockfft_stress.so")
STRESS_UNITS = ("kern_pipe.cu", "kern_pipe3.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libsynth.so")


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    print("+", " ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)


def _includes(path, seen=None):
    """Local headers a source includes (recursively, #include "...")."""
    seen = set() if seen is None else seen
    d = os.path.dirname(path)
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith('#include "'):
                h = os.path.normpath(os.path.join(d, line.split('"')[1]))
                if os.path.exists(h) and h not in seen:
                    seen.add(h)
                    _includes(h, seen)
    return sorted(seen)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INC, "blockfft.h"))
    objs, cmds = [], []
    # translation units compile concurrently (each holds its own kernel instantiations)
    stress_objs = []
    units = [(u, k, "") for u, k in (("plan.cu", "cu"), ("kern_rows.cu", "cu"), ("kern_cluster.cu", "cu"),
                                     ("kern_pipe.cu", "cu"), ("kern_pipe3.cu", "cu"), ("real.cu", "cu"), ("dist.cu", "cu"),
                                     ("stream.cpp", "cpp"))]
    units += [(u, "cu", "stress") for u in STRESS_UNITS]
    for src, kind, flavour in units:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + (".stress" if flavour else "") + ".o")
        if flavour:
            stress_objs.append(o)
        else:
            objs.append(o)
        if force or _newer(o, [s] + _includes(s)):
            if kind == "cu":
                cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                       "-I", INC, "-c", s, "-o", o] + (["-DBFFT_STRESS"] if flavour else [])
                if verbose_ptxas:
                    cmd[1:1] = ["-Xptxas", "-v"]
            else:
                cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-I", INC,
                       "-I", os.path.join(CUDA, "include"), "-c", s, "-o", o]
            cmds.append(cmd)
    procs = []
    for cmd in cmds:
        print("+", " ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in procs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart", "-lpthread"])
        os.replace(LIB + ".tmp", LIB)
    sobjs = [o for o in objs if not any(o.endswith(u + ".o") for u in STRESS_UNITS)] + stress_objs
    if force or _newer(STRESS_LIB, sobjs):
        _run([NVCC, *ARCH, "-shared", "-o", STRESS_LIB + ".tmp", *sobjs, "-lcudart", "-lpthread"])
        os.replace(STRESS_LIB + ".tmp", STRESS_LIB)
    ssrc = os.path.join(ROOT, "synth", "csrc", "synth_fill.cu")
    if force or _newer(SYNTH_LIB, [ssrc]):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", ssrc,
              "-o", SYNTH_LIB + ".tmp", "-lcudart"])
        os.replace(SYNTH_LIB + ".tmp", SYNTH_LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
