"""Scalar model of the CUDA FFT engine's index arithmetic (csrc/fft_engine.cuh):
in-place radix-2^k DIF passes (natural in -> bit-reversed out) and their DIT
mirrors (bit-reversed in -> natural out). Used only to check the pass/twiddle
bookkeeping against numpy.fft before writing it in CUDA."""
import numpy as np

def bitrev(x, bits):
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1); x >>= 1
    return r

def passes(K, k):
    out = []
    lo = K
    while lo > 0:
        kk = min(k, lo)
        lo -= kk
        out.append((lo, kk))
    return out   # (lo, active bits) from high to low; last has lo = 0

def W(L, e, sigma):
    return np.exp(sigma * 2j * np.pi * e / L)

def positions(t, lo, k):
    tlo = t & ((1 << lo) - 1); thi = t >> lo
    return [(thi << (lo + k)) | (q << lo) | tlo for q in range(1 << k)], tlo

def dif_pass(buf, K, k, lo, ka, sigma):
    L = 1 << K; R = 1 << k
    kloc = k if lo > 0 else k   # local bits [lo, lo+k) ; last pass lo=0
    for t in range(L >> k):
        pos, tlo = positions(t, lo, k)
        v = [buf[p] for p in pos]
        # DFT over active local bits [0, ka) ... for non-last passes ka == k
        for j in range(ka - 1, -1, -1):
            for q in range(R):
                if q & (1 << j): continue
                q2 = q | (1 << j)
                a, b = v[q], v[q2]
                v[q] = a + b
                v[q2] = (a - b) * W(1 << (j + 1), q & ((1 << j) - 1), sigma)
        # post twiddle: Ls = 2^(lo+ka); freq r' = bitrev_ka(q active part)
        if lo > 0:
            for q in range(R):
                rp = bitrev(q, ka)
                v[q] *= W(L, tlo * rp * (1 << (K - lo - ka)), sigma)
        for q, p in enumerate(pos):
            buf[p] = v[q]

def dit_pass(buf, K, k, lo, ka, sigma):
    L = 1 << K; R = 1 << k
    for t in range(L >> k):
        pos, tlo = positions(t, lo, k)
        v = [buf[p] for p in pos]
        if lo > 0:
            for q in range(R):
                rp = bitrev(q, ka)
                v[q] *= W(L, tlo * rp * (1 << (K - lo - ka)), sigma)
        for j in range(0, ka):
            for q in range(R):
                if q & (1 << j): continue
                q2 = q | (1 << j)
                a = v[q]; b = v[q2] * W(1 << (j + 1), q & ((1 << j) - 1), sigma)
                v[q] = a + b; v[q2] = a - b
        for q, p in enumerate(pos):
            buf[p] = v[q]

def dif(x, k, sigma=-1):
    K = int(np.log2(len(x))); buf = np.array(x, dtype=complex)
    for lo, ka in passes(K, k):
        dif_pass(buf, K, k, lo, ka, sigma)
    return buf

def dit(x, k, sigma=-1):
    K = int(np.log2(len(x))); buf = np.array(x, dtype=complex)
    for lo, ka in reversed(passes(K, k)):
        dit_pass(buf, K, k, lo, ka, sigma)
    return buf

if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for K in (3, 5, 8, 9):
        for k in (1, 2, 3, 4):
            if k > K: continue
            L = 1 << K
            x = rng.standard_normal(L) + 1j * rng.standard_normal(L)
            br = np.array([bitrev(i, K) for i in range(L)])
            X = dif(x, k, -1)
            assert np.allclose(X[br], np.fft.fft(x)), (K, k)   # X at bitrev positions
            Xn = np.empty(L, complex); Xn[br] = np.fft.fft(x)   # bitrev-ordered spectrum
            y = dit(Xn, k, +1)
            assert np.allclose(y, L * np.fft.ifft(np.fft.fft(x))), (K, k)
            y2 = dit(Xn, k, -1)          # forward DFT from bitrev input
            Xb = np.empty(L, complex); Xb[br] = x
            assert np.allclose(dit(Xb, k, -1), np.fft.fft(x)), (K, k)
    print("engine model OK")
