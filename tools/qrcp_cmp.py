"""Debug: first diverging pivot step of qb_pivoted_qr against the oracle (the test's first case)."""
import sys
import numpy as np
import torch
import synth
from oracle import qb as oqb
import paper_1503_07157_b200 as qbp

CASES = [(600, 400, "exp10_20", 1e-6, 16), (1500, 900, "poly2", 1e-4, 64), (800, 2000, "exp_100", 1e-3, 100)]
m, n, kind, eps, b = CASES[int(sys.argv[1]) if len(sys.argv) > 1 else 0]
A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 91 + n)
c = qbp.QB(0)
g = c.factor(torch.from_numpy(np.asfortranarray(A)).cuda(), eps, b, 0, seed=2)
B = g["B"].cpu().numpy()
r = c.pivoted_qr()
perm, R = r["perm"], r["R"].cpu().numpy()
Po, Qo, Ro = oqb.pivoted_qr(B)
d = np.nonzero(perm != Po)[0]
print("k", g["k"], "first perm diff", d[:5])
rd = np.abs(R - Ro).max(axis=1)
bad = np.nonzero(rd > 1e-12)[0]
print("rows with R diff > 1e-12:", bad[:10], "max", rd.max())
for i in list(bad[:3]):
    print(i, "R diag", R[i, i], Ro[i, i], "row diff", rd[i], "cols", np.nonzero(np.abs(R[i] - Ro[i]) > 1e-12)[0][:10])
nrm = np.linalg.norm(B, axis=0)
print("B col norms of gpu perm[1], oracle Po[1]:", perm[1], Po[1])
