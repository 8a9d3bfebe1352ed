"""Numpy prototype of the CUDA kernels' index algebra (design aid, not a test
of the product).  Checks, against numpy.fft:
  * the per-thread mixed-radix Stockham schedule (PPT points per thread,
    first pass radix 2^(k mod 4), then radix-16 passes) used by both engines;
  * the four-step split n = N2*n1 + n2, k = k1 + N1*k2 with twiddle W_N^{n2 k1};
and counts shared-memory bank conflicts of the swizzled layouts."""
import numpy as np

def W(n, e):  # forward root of unity power
    return np.exp(-2j * np.pi * (np.asarray(e) % n) / n)

def radices(L, ppt=16):
    if L <= ppt:
        return [L]
    k = L.bit_length() - 1
    r = []
    b = k % 4
    if b:
        r.append(1 << b)
    r += [16] * (k // 4)
    return r

def stockham(x, ppt=16):
    L = x.size
    rs = radices(L, ppt)
    P = min(ppt, L)
    T = L // P
    Ns = 1
    for R in rs:
        y = np.empty_like(x)
        for t in range(T):
            v = [x[t + s * T] for s in range(P)]
            for m in range(P // R):
                j = t + m * T
                a = np.array([v[m + q * (P // R)] for q in range(R)])
                a = a * W(Ns * R, (j % Ns) * np.arange(R))
                a = np.fft.fft(a)
                for q in range(R):
                    y[(j // Ns) * Ns * R + j % Ns + q * Ns] = a[q]
        x = y
        Ns *= R
    return x

for k in range(1, 13):
    L = 1 << k
    x = np.random.randn(L) + 1j * np.random.randn(L)
    err = np.abs(stockham(x) - np.fft.fft(x)).max() / np.abs(np.fft.fft(x)).max()
    assert err < 1e-12, (L, err)
print("stockham schedule ok for L=2..4096; radices:", {1 << k: radices(1 << k) for k in range(1, 13)})

def fourstep(x, N1, N2):
    N = N1 * N2
    A = x.reshape(N1, N2)                      # A[n1][n2] = x[N2*n1 + n2]
    Y = np.fft.fft(A, axis=0)                  # Y[k1][n2]
    Y = Y * W(N, np.outer(np.arange(N1), np.arange(N2)))   # * W_N^{n2 k1}
    Z = np.fft.fft(Y, axis=1)                  # Z[k1][k2]
    X = np.empty(N, complex)
    for k1 in range(N1):
        for k2 in range(N2):
            X[k1 + N1 * k2] = Z[k1, k2]
    return X

for (N1, N2) in [(4, 8), (32, 32), (256, 256), (128, 256), (512, 256)]:
    x = np.random.randn(N1 * N2) + 1j * np.random.randn(N1 * N2)
    assert np.allclose(fourstep(x, N1, N2), np.fft.fft(x))
print("four-step ok")

def wavefronts(addrs):
    """8-byte elements; per half-warp count max distinct elements per bank."""
    tot = 0
    for h in range(2):
        banks = {}
        for e in set(addrs[16 * h:16 * h + 16]):
            for b in (2 * e % 32, (2 * e + 1) % 32):
                banks.setdefault(b, set()).add(e)
        tot += max(len(s) for s in banks.values())
    return tot

def swz_row(e):      # E1 (contiguous rows) layout: one pad slot per 16 elements
    return e + (e >> 4)

worst = 0
bad = set()
for k in range(5, 15):
    L = 1 << k
    rs = radices(L)
    T = L // 16
    B = max(1, 256 // T)
    Ns = 1
    for pi, R in enumerate(rs):
        # reads x[t + s*T] ; writes (j//Ns)*Ns*R + j%Ns + q*Ns
        for s in range(16):
            for w0 in range(0, B * T, 32):
                lanes = range(w0, w0 + 32)
                ad = [swz_row((l // T) * L + l % T + s * T) for l in lanes]
                worst = max(worst, wavefronts(ad))
        for m in range(16 // R):
            for q in range(R):
                for w0 in range(0, B * T, 32):
                    ad = []
                    for l in range(w0, w0 + 32):
                        t = l % T; j = t + m * T
                        e = (j // Ns) * Ns * R + j % Ns + q * Ns
                        ad.append(swz_row((l // T) * L + e))
                    wf = wavefronts(ad)
                    if wf > 2:
                        bad.add((L, pi, R, Ns, wf))
                    worst = max(worst, wf)
        Ns *= R
print("conflicting (L, pass, R, Ns, wf):", sorted(bad))
print("E1 worst wavefronts per warp access (2 = optimal for 8B):", worst)
