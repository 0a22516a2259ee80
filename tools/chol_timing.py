"""Phase timestamps of the cluster Cholesky (needs a -DQB_CHOL_TIMING build in QB_LIB_PATH)."""
import ctypes

import numpy as np
import torch

import paper_1503_07157_b200 as qbp

L = qbp.lib()
c = qbp.QB(0)
rng = np.random.default_rng(1)
for w in (256, 128):
    X = rng.standard_normal((4 * w + 7, w)) * np.exp(-np.arange(w) / 60.0)[None, :]
    G = X.T @ X
    Gd = torch.from_numpy(G.T.copy()).cuda()
    R = torch.zeros((w, w), dtype=torch.float64, device="cuda")
    for rep in range(3):
        qbp.qb_chol_rinv(c.ctx, Gd.data_ptr(), w, w, X.shape[0], R.data_ptr(), w)
    ts = (ctypes.c_ulonglong * 64)()
    L.qb_debug_chol_ts(ts)
    t = np.array(ts[:64], dtype=np.int64)
    print("w", w, [(i, int(t[i] - t[0])) for i in range(40) if t[i] >= t[0]])
