"""Helper for test_gpu_pivoted_qr.py: one pivoted-QR case against the oracle in a fresh process, so
that the schedule-selecting environment variables (read once per process by the library) take effect.
Exit status 0 = same permutation and R within 1e-12 ||B||."""
import sys

import numpy as np
import torch

import synth
from oracle import qb as oqb
import paper_1503_07157_b200 as qbp

m, n, kind, eps, b = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4]), int(sys.argv[5])
A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 91 + n)
c = qbp.QB(0)
g = c.factor(torch.from_numpy(np.asfortranarray(A)).cuda(), eps, b, 0, seed=2)
Q, B = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
r = c.pivoted_qr()
perm, Qh, R = r["perm"], r["Qh"].cpu().numpy(), r["R"].cpu().numpy()
Po, Qo, Ro = oqb.pivoted_qr(B)
ok = np.array_equal(perm, Po) and np.abs(R - Ro).max() <= 1e-12 * np.linalg.norm(B)
ok = ok and np.linalg.norm(Qh - Q @ Qo) <= 1e-11 * np.sqrt(g["k"])
print("k", g["k"], "ok", ok)
sys.exit(0 if ok else 1)
