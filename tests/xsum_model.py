"""Pure-Python model of csrc/exactsum.cuh (test infrastructure): Python floats are IEEE doubles."""
import math, random, struct
def bits(x): return struct.unpack('<Q', struct.pack('<d', x))[0]
def fromb(b): return struct.unpack('<d', struct.pack('<Q', b))[0]
def binade(s): return ((bits(s) >> 52) & 0x7FF) - 1023
SEG = 64
def seg_map(xs, e):
    inv_u = fromb((1023 + 52 - e) << 52)
    f0 = f1 = 0; p0, p1 = 0, 1
    for x in xs:
        v = x * inv_u
        if not v < 2.0**52: return None
        q = math.floor(v); fr = v - q; q = int(q)
        gt = 1 if fr > 0.5 else 0; tie = 1 if fr == 0.5 else 0; qp = q & 1
        d0 = q + gt + (tie & (p0 ^ qp)); d1 = q + gt + (tie & (p1 ^ qp))
        f0 += d0; f1 += d1; p0 ^= d0 & 1; p1 ^= d1 & 1
        if f0 >= 2**53 or f1 >= 2**53: return None
    return (f0, f1, e)
def apply(s, m):
    if m == "zero": return s
    if m is None or not s > 0: return None
    b = bits(s); e = ((b >> 52) & 0x7FF) - 1023
    if e != m[2] or ((b >> 52) & 0x7FF) == 0: return None
    mant = (b & ((1 << 52) - 1)) | (1 << 52)
    nm = mant + (m[1] if mant & 1 else m[0])
    if nm >= 2**53: return None
    return fromb((b & 0xFFF0000000000000) | (nm - (1 << 52)))
def exact(xs):
    segs = [xs[i:i+SEG] for i in range(0, len(xs), SEG)]
    approx = [sum(sg) for sg in segs]; pre = []; run = 0.0
    for a in approx: pre.append(run); run += a
    maps = [seg_map(sg, binade(p)) if p > 0 else ("zero" if all(x == 0 for x in sg) else None)
            for sg, p in zip(segs, pre)]
    s = 0.0; nseq = 0
    for sg, m in zip(segs, maps):
        r = apply(s, m)
        if r is None:
            nseq += 1
            for x in sg: s = s + x
        else: s = r
    return s, nseq
def seq(xs):
    s = 0.0
    for x in xs: s = s + x
    return s
if __name__ == "__main__":
    random.seed(1)
    bad = tot = nseqs = 0
    for trial in range(400):
        n = random.randint(1, 6000)
        xs = [random.random() for _ in range(n)]
        a, ns = exact(xs)
        tot += 1
        nseqs += ns
        bad += a != seq(xs)
    print("trials", tot, "mismatches", bad, "avg sequential segments", nseqs / tot)
