"""Oracle side of the Ω generator (TEST INFRASTRUCTURE; see oracle/__init__.py).

The paper only says Ω_i = randn(n, b) (Fig. 2 line (2); :866 Fig. 4 line (2)),
slices of one n x ℓ Gaussian matrix Ω = [Ω_1 ... Ω_s] (eq. (OmegaBlock)).
Reading R14/R15: column c of Ω is a pure function of (seed, c), drawn by a
counter-based generator so that the blocked and unblocked algorithms, every block size
and every sharding see the same Ω.  This file implements the generator specification of
DESIGN.md §3.3 with numpy, independently of the CUDA kernel (which implements the same
specification in paper_1503_07157_b200/csrc/omega.cuh).  Only IEEE-754 correctly rounded
+, -, *, /, sqrt are used (no fma, no libm), evaluated in the order written, so the two
sides agree bit for bit.

Pins (tests/test_oracle_omega.py): Random123 Philox4x32-10 known-answer vectors;
``spec_log`` and ``spec_sincospi`` within 2 ulp of correctly rounded values (mpmath);
Gaussian moments and a KS test; the literals below re-derived with mpmath.
"""
import numpy as np

# --- Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11)
PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 arrays (broadcasting).  Returns 4 uint32 arrays.

    Round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2,
           c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by (W0, W1)
    before every round but the first.
    """
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32)
    k1 = np.asarray(k1, dtype=np.uint32)
    with np.errstate(over="ignore"):
        for rnd in range(10):
            if rnd > 0:
                k0 = (k0 + PHILOX_W0).astype(np.uint32)
                k1 = (k1 + PHILOX_W1).astype(np.uint32)
            p0 = PHILOX_M0 * c0.astype(np.uint64)
            p1 = PHILOX_M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


# --- spec_log: natural log on (0, 1], DESIGN.md §3.3 step 4 -------------------------------
SQRT2 = float.fromhex("0x1.6a09e667f3bcdp+0")
LN2_HI = float.fromhex("0x1.62e42fefa3800p-1")   # 43 significant bits: e*LN2_HI exact
LN2_LO = float.fromhex("0x1.ef35793c76730p-45")


def spec_log(x):
    """ln(x) for x in (0, 1]: x = f 2^e, f in (sqrt2/2, sqrt2]; s = (f-1)/(f+1);
    ln f = 2 atanh(s) = 2s + s z (2/3 + 2z/5 + ... + 2z^11/25), z = s^2."""
    x = np.asarray(x, dtype=np.float64)
    mant, ex = np.frexp(x)                 # x = mant 2^ex, mant in [0.5, 1): exact
    f = mant * 2.0
    e = (ex - 1).astype(np.float64)
    big = f > SQRT2
    f = np.where(big, f * 0.5, f)
    e = np.where(big, e + 1.0, e)
    s = (f - 1.0) / (f + 1.0)
    z = s * s
    p = np.full_like(s, 2.0 / 25.0)
    for k in range(11, 0, -1):
        p = p * z + 2.0 / (2 * k + 1)
    t = s * z
    t = t * p
    lf = 2.0 * s + t
    return e * LN2_HI + (e * LN2_LO + lf)


# --- spec_sincospi: (sin(pi t), cos(pi t)) for t in [0, 2), DESIGN.md §3.3 step 5 ----------
# cs[k] = RN((-1)^k pi^(2k+1)/(2k+1)!), cc[k] = RN((-1)^k pi^(2k)/(2k)!)  (tools/gen_sincospi_coeffs.py)
SINPI_C = [float.fromhex(h) for h in (
    "0x1.921fb54442d18p+1", "-0x1.4abbce625be53p+2", "0x1.466bc6775aae2p+1",
    "-0x1.32d2cce62bd86p-1", "0x1.50783487ee782p-4", "-0x1.e3074fde8871fp-8",
    "0x1.e8f434d018d63p-12", "-0x1.6fadb9f155744p-16", "0x1.aaec32af93359p-21",
    "-0x1.8a404211f9547p-26", "0x1.2877020d52cf0p-31")]
COSPI_C = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "-0x1.3bd3cc9be45dep+2", "0x1.03c1f081b5ac4p+2",
    "-0x1.55d3c7e3cbffap+0", "0x1.e1f506891babbp-3", "-0x1.a6d1f2a204a8cp-6",
    "0x1.f9d38a3763cc3p-10", "-0x1.b6e24f44b128fp-14", "0x1.20c62c2f2d7f5p-18",
    "-0x1.2a0c591af8314p-23", "0x1.ef6e308d6d1c4p-29")]


def spec_sincospi(t):
    """Return (sin(pi t), cos(pi t)) for t in [0, 2): j = rint(2t), r = t - j/2 (exact,
    |r| <= 1/4), Taylor polynomials in r^2 by Horner, then the quadrant j mod 4."""
    t = np.asarray(t, dtype=np.float64)
    j = np.rint(2.0 * t)                   # round half to even
    r = t - 0.5 * j
    r2 = r * r
    S = np.full_like(r, SINPI_C[10])
    C = np.full_like(r, COSPI_C[10])
    for k in range(9, -1, -1):
        S = S * r2 + SINPI_C[k]
        C = C * r2 + COSPI_C[k]
    sn = r * S
    cn = C
    q = j.astype(np.int64) & 3
    sin_out = np.select([q == 0, q == 1, q == 2, q == 3], [sn, cn, -sn, -cn])
    cos_out = np.select([q == 0, q == 1, q == 2, q == 3], [cn, -sn, -cn, sn])
    return sin_out, cos_out


TWO_M53 = float.fromhex("0x1p-53")


def gaussian_pairs(seed, p, c):
    """The two normals of pair p (rows 2p, 2p+1) of column c (broadcast over p, c).

    Counter (lo32 p, hi32 p, lo32 c, hi32 c), key (lo32 seed, hi32 seed);
    U1 = (a + 1) 2^-53 in (0, 1], a = (x:y) >> 11; U2 = b 2^-53 in [0, 1), b = (z:w) >> 11;
    rho = sqrt(-2 ln U1); Ω(2p, c) = rho cos(2 pi U2), Ω(2p+1, c) = rho sin(2 pi U2)."""
    p = np.asarray(p, dtype=np.uint64)
    c = np.asarray(c, dtype=np.uint64)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    x, y, z, w = philox4x32_10(p & _MASK32, p >> np.uint64(32), c & _MASK32, c >> np.uint64(32),
                               np.uint32(seed & 0xFFFFFFFF), np.uint32(seed >> 32))
    a = ((x.astype(np.uint64) << np.uint64(32)) | y.astype(np.uint64)) >> np.uint64(11)
    b = ((z.astype(np.uint64) << np.uint64(32)) | w.astype(np.uint64)) >> np.uint64(11)
    u1 = (a + np.uint64(1)).astype(np.float64) * TWO_M53   # exact: a + 1 <= 2^53
    u2 = b.astype(np.float64) * TWO_M53
    rho = np.sqrt(-2.0 * spec_log(u1))
    sn, cn = spec_sincospi(2.0 * u2)
    return rho * cn, rho * sn


def omega_panel(seed, n, col0, w, row0=0, row1=None):
    """Ω(row0:row1, col0:col0+w) as a float64 array of shape (row1 - row0, w).

    Row r of column c is member r & 1 of pair r >> 1, so any row range (a column shard of A
    owns a row range of Ω) reproduces the full panel bit for bit."""
    if row1 is None:
        row1 = n
    if row1 <= row0 or w <= 0:
        return np.zeros((max(row1 - row0, 0), max(w, 0)))
    p = np.arange(row0 >> 1, ((row1 - 1) >> 1) + 1, dtype=np.uint64)
    c = np.arange(col0, col0 + w, dtype=np.uint64)
    even, odd = gaussian_pairs(seed, p[:, None], c[None, :])
    full = np.empty((2 * len(p), w))
    full[0::2] = even
    full[1::2] = odd
    start = row0 - 2 * int(p[0])
    return full[start:start + (row1 - row0)]
