"""Characterise tcgen05.mma.kind::f16 fp32 accumulation (the
rollout certificate's hardware model).

    python tools/tc_accum_analyze.py gen  <in.bin>            # seeded test chains
    tools/tc_accum_probe accum <in.bin> <out.bin>              # on the B200
    python tools/tc_accum_analyze.py check <in.bin> <out.bin>

For every instruction d = c + sum_{k<16} a_k b_k (c = the previous read-back, 0
for the first instruction of a chain) the exact value is computed with
math.fsum (correctly rounded fp64 of the exact sum; the fp16 products are exact
in fp64) and the error of the hardware result is reported in units of
  u_M  = 2^(E-23), E = exponent of the largest addend |c|, |a_k b_k|,
  u_S  = 2^-23 (|c| + sum |a_k b_k|)   (the certificate's per-instruction model),
  u_d  = ulp(d) in fp32.
"""
import math
import sys

import numpy as np

M, N, K = 128, 16, 16


def _f16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16)


def _rand_f16(g, shape, emin, emax):
    s = g.choice([-1.0, 1.0], size=shape)
    e = g.integers(emin, emax + 1, size=shape)
    m = 1.0 + g.integers(0, 1024, size=shape) / 1024.0
    return _f16(s * m * np.exp2(e))


def gen(path, seed=0):
    g = np.random.default_rng(seed)
    fams = []
    # F_rand: independent random addends over a wide exponent range, 4 chained instructions
    for _ in range(48):
        fams.append(("rand", [(_rand_f16(g, (M, K), -10, 6), _rand_f16(g, (N, K), -10, 6)) for _ in range(4)]))
    # F_bigc: a large accumulator c (one product) then 16 small products of one sign near ulp(c)
    for _ in range(48):
        A0 = np.zeros((M, K)); B0 = np.zeros((N, K))
        sr = g.integers(-3, 4, size=M)
        A0[:, 0] = (1.0 + g.integers(0, 1024, size=M) / 1024.0) * np.exp2(sr)
        B0[:, 0] = g.choice([-1.0, 1.0], size=N)
        j = g.integers(-3, 10, size=(M, 1))  # products ~ 2^(sr - 23 - j)
        A1 = (1.0 + g.integers(0, 1024, size=(M, K)) / 1024.0) * np.exp2(sr[:, None] - 12 - j)
        sign = g.choice([-1.0, 1.0], size=(N, 1))
        B1 = sign * (1.0 + g.integers(0, 1024, size=(N, K)) / 1024.0) * np.exp2(-11.0)
        if g.random() < 0.5:
            B1 = B1 * g.choice([-1.0, 1.0], size=(N, K))
        fams.append(("bigc", [(_f16(A0), _f16(B0)), (_f16(A1), _f16(B1))]))
    # F_real: the rollout's split GEMM (L2: h0 * 2^14 hi/lo x W * 2^e hi/lo, K = 128 as 8 chunks x 3 products)
    for _ in range(24):
        h = np.tanh(g.normal(0, 1.2, size=(M, 128))) * 16384.0
        W = g.normal(0, 1 / math.sqrt(128), size=(N, 128))
        e = 14 - math.frexp(np.abs(W).max())[1]
        W = W * 2.0 ** e
        ahi = _f16(h); alo = _f16(h - ahi.astype(np.float64))
        bhi = _f16(W); blo = _f16(W - bhi.astype(np.float64))
        ch = []
        for kb in range(8):
            s = slice(16 * kb, 16 * kb + 16)
            ch += [(ahi[:, s], bhi[:, s]), (ahi[:, s], blo[:, s]), (alo[:, s], bhi[:, s])]
        fams.append(("real", ch))
    nm = max(len(c) for _, c in fams)
    with open(path, "wb") as f:
        np.array([len(fams), nm], dtype=np.int32).tofile(f)
        for _, ch in fams:
            ch = ch + [(np.zeros((M, K), np.float16), np.zeros((N, K), np.float16))] * (nm - len(ch))
            for a, b in ch:
                np.ascontiguousarray(a, dtype=np.float16).tofile(f)
                np.ascontiguousarray(b, dtype=np.float16).tofile(f)
    with open(path + ".fams", "w") as f:
        f.write("\n".join(n + " " + str(len(c)) for n, c in fams))


def check(inp, outp):
    with open(inp, "rb") as f:
        nb, nm = np.fromfile(f, dtype=np.int32, count=2)
        raw = np.fromfile(f, dtype=np.float16)
    per = M * K + N * K
    raw = raw.reshape(nb, nm, per)
    A = raw[:, :, : M * K].reshape(nb, nm, M, K).astype(np.float64)
    B = raw[:, :, M * K:].reshape(nb, nm, N, K).astype(np.float64)
    D = np.fromfile(outp, dtype=np.float32).reshape(nb, nm, M, N).astype(np.float64)
    fams = [l.split() for l in open(inp + ".fams").read().splitlines()]
    stats = {}
    for b in range(nb):
        name, nmm = fams[b][0], int(fams[b][1])
        st = stats.setdefault(name, {"n": 0, "uM": 0.0, "uS": 0.0, "ud": 0.0, "rn": 0, "rz": 0, "nz": 0})
        for j in range(nmm):
            P = A[b, j][:, None, :] * B[b, j][None, :, :]  # [M, N, K], exact in fp64
            C = D[b, j - 1] if j > 0 else np.zeros((M, N))
            d = D[b, j]
            for r in range(M):
                for n in range(N):
                    terms = [C[r, n]] + list(P[r, n])
                    S = math.fsum(terms)
                    err = math.fsum([d[r, n]] + [-t for t in terms])
                    mx = max(abs(t) for t in terms)
                    st["n"] += 1
                    if mx == 0.0:
                        continue
                    st["nz"] += 1
                    E = math.frexp(mx)[1] - 1
                    st["uM"] = max(st["uM"], abs(err) / 2.0 ** (E - 23))
                    st["uS"] = max(st["uS"], abs(err) / (2.0 ** -23 * math.fsum(abs(t) for t in terms)))
                    ud = np.spacing(np.float32(abs(d[r, n]))) if d[r, n] != 0 else np.float32(2.0 ** -149)
                    st["ud"] = max(st["ud"], abs(err) / float(ud))
                    s32 = np.float32(S)
                    st["rn"] += int(float(s32) == d[r, n])
                    rz = s32 if abs(float(s32)) <= abs(S) else np.nextafter(s32, np.float32(0))
                    st["rz"] += int(float(rz) == d[r, n])
    for name, st in stats.items():
        print(f"{name:5s} outputs {st['n']:8d} (nonzero {st['nz']}): max|err| = {st['uM']:.3f} u_M, "
              f"{st['uS']:.3f} u_S, {st['ud']:.3f} ulp(d); == RN(S) {st['rn']}, == RZ(S) {st['rz']}")


if __name__ == "__main__":
    if sys.argv[1] == "gen":
        gen(sys.argv[2])
    else:
        check(sys.argv[2], sys.argv[3])
