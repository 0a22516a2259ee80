"""Write tests/golden/c5_oracle.json: the ORACLE's k and per-block residual history for BASELINE
configs[4] (C5: 50000 x 50000 FP64, sigma_j = e^(-j/150), rank 3584, eps = 1e-6, b = 256, q = 1),
next to the SHA-256 of the A bytes it factored.

Calls only synth/ (the seeded input generator; on a GPU box it builds A with torch) and oracle/
(randQB_pb, Fig. 4) — nothing from the CUDA path.  The oracle needs ~10-20 min
and ~90 GB of host memory on the 16-core GPU-box host, too long for a test, so the test
(tests/test_gpu_fullsize.py::test_c5_against_stored_oracle_values) compares against these values.

    python tools/c5_oracle_values.py [out.json]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import qb as oqb  # noqa: E402


def main():
    import torch
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c5_oracle.json")
    cfg = synth.CONFIGS["C5"]
    t0 = time.time()
    A_dev = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix)
    A = np.empty((cfg.m, cfg.n), dtype=np.float64, order="F")
    h = hashlib.sha256()
    for j in range(0, cfg.n, 512):
        slab = A_dev[:, j:j + 512].t().contiguous().cpu().numpy()
        h.update(slab.tobytes())
        A[:, j:j + 512] = slab.T
    del A_dev
    torch.cuda.empty_cache()
    t_gen = time.time() - t0
    t0 = time.time()
    o = oqb.randqb_pb(A, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega)
    t_orc = time.time() - t0
    rec = {
        "what": "oracle (oracle/qb.py randqb_pb, Fig. 4 PAPER.md:859-887) on BASELINE configs[4] C5",
        "written_by": "tools/c5_oracle_values.py (calls only synth/ and oracle/)",
        "config": {"m": cfg.m, "n": cfg.n, "spectrum": cfg.spectrum, "rank": cfg.rank, "eps": cfg.eps, "b": cfg.b,
                   "q": cfg.q, "seed_matrix": cfg.seed_matrix, "seed_omega": cfg.seed_omega},
        "a_sha256": h.hexdigest(),
        "a_fro2": float(o.r2_0),
        "status": int(o.status),
        "k": int(o.k),
        "hist": [[int(e), int(w), float(r2), float(ei)] for (e, w, r2, ei) in o.hist],
        "seconds_generate": t_gen,
        "seconds_oracle": t_orc,
        "host_cores": os.cpu_count(),
        "torch": torch.__version__,
    }
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps({k: rec[k] for k in ("k", "status", "seconds_oracle", "a_sha256")}))


if __name__ == "__main__":
    main()
