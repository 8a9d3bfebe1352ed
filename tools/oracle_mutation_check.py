"""Mutation check for the oracle pins.

Applies plausible one-token mistakes to oracle/oracle.c in a scratch copy,
rebuilds, and checks that tests/test_oracle.py fails for every mutant.
Run: python tools/oracle_mutation_check.py   (CPU only, ~1-2 min)
"""
import os, shutil, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTANTS = [
    ("double wr = cos(ang), wi = -sin(ang);", "double wr = cos(ang), wi = sin(ang);", "fft twiddle sign"),
    ("double tr = wr * orr - wi * oi;", "double tr = wr * orr + wi * oi;", "fft complex-mul sign"),
    ("X[2 * (k + h)] = er - tr;", "X[2 * (k + h)] = er + tr;", "fft butterfly sign"),
    ("fft_rec(x + 2 * stride, 2 * stride, X + 2 * h, h);", "fft_rec(x + 4 * stride, 2 * stride, X + 2 * h, h);", "fft odd offset"),
    ("int64_t m = (j * k) % n;", "int64_t m = (j * k + 1) % n;", "dft exponent index"),
    ("double s = (double)dir * sin(ang);", "double s = -(double)dir * sin(ang);", "dft sign"),
    ("if (dir == 1) { sr /= (double)n; si /= (double)n; }", "", "dft inverse scale dropped"),
    ("out[2 * k + 1] = -out[2 * k + 1] / (double)n;", "out[2 * k + 1] = out[2 * k + 1] / (double)n;", "fft inverse conj dropped"),
    ("si += xr * s + xi * c;", "si += xr * s - xi * c;", "dft imag term sign"),
]

def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    survived = []
    for old, new, name in MUTANTS:
        assert old in src, name
        with tempfile.TemporaryDirectory() as d:
            shutil.copytree(ROOT, os.path.join(d, "r"), ignore=shutil.ignore_patterns(".git", "gpurun_out", "*.so", "baseline"))
            r = os.path.join(d, "r")
            open(os.path.join(r, "oracle", "oracle.c"), "w").write(src.replace(old, new, 1))
            p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "tests/test_oracle.py"],
                               cwd=r, capture_output=True, text=True)
            killed = p.returncode != 0
            print(f"{'KILLED ' if killed else 'SURVIVED'} {name}")
            if not killed:
                survived.append(name)
    print("all mutants killed" if not survived else f"survivors: {survived}")
    return 1 if survived else 0

if __name__ == "__main__":
    sys.exit(main())
