"""Derivation record for the Ω generator's sin/cos(pi r) Taylor coefficients.

Prints cs_k = RN((-1)^k pi^(2k+1)/(2k+1)!) and cc_k = RN((-1)^k pi^(2k)/(2k)!), k = 0..10,
as C99 hex-float literals, computed at 200 bits with mpmath.  The generator specification in
DESIGN.md lists these values; the oracle (oracle/omega.py) and the CUDA kernel
(paper_1503_07157_b200/csrc/omega.cuh) each carry their own copy typed from that list, and
tests/test_oracle_omega.py re-derives them with mpmath to pin the oracle's copy.  This script
writes no file: it is not a shared constant generator, only the record of where the
numbers come from.
"""
import mpmath

mpmath.mp.prec = 200


def coeffs():
    cs, cc = [], []
    for k in range(11):
        s = (-1) ** k * mpmath.pi ** (2 * k + 1) / mpmath.factorial(2 * k + 1)
        c = (-1) ** k * mpmath.pi ** (2 * k) / mpmath.factorial(2 * k)
        cs.append(float(s))  # mpf -> float rounds to nearest
        cc.append(float(c))
    return cs, cc


if __name__ == "__main__":
    cs, cc = coeffs()
    for k, v in enumerate(cs):
        print(f"cs[{k:2d}] = {v.hex()}")
    for k, v in enumerate(cc):
        print(f"cc[{k:2d}] = {v.hex()}")
