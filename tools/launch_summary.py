"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py:
per-kernel-class time and share over the LAST factorization (the timed step).

    python tools/launch_summary.py gpurun_out/launches_r01.csv [launches_per_step] > profiles/launches_r01_summary.json
"""
import collections
import csv
import json
import re
import sys


def classify(name, grid):
    if "gemm_f64_kernel" in name:
        m = re.search(r"gemm_f64_kernel<(?:\(int\))?(\d), (?:\(int\))?(\d+), (?:\(int\))?(\d)>", name)
        lay, bn, epi = (int(m.group(1)), int(m.group(2)), int(m.group(3))) if m else (-1, -1, -1)
        return f"gemm_f64<{'NN' if lay == 0 else 'TN'},{bn},{['STORE_COL', 'STORE_ROW', 'SUB_COL'][epi]}>"
    if "gemm_tf32_kernel" in name:
        m = re.search(r"gemm_tf32_kernel<(?:\(int\))?(\d), (?:\(int\))?(\d+), (?:\(int\))?(\d)(?:, (?:\(bool\))?\w+)?>",
                      name)
        lay, bn, epi = (int(m.group(1)), int(m.group(2)), int(m.group(3))) if m else (-1, -1, -1)
        return f"gemm_tf32<{'NN' if lay == 0 else 'TN'},{bn},{['STORE_COL', 'STORE_ROW', 'SUB_COL'][epi]}>"
    m = re.search(r"qbk::(\w+)", name)
    return m.group(1) if m else None


def main():
    path = sys.argv[1]
    per_step = int(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = []
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append(d)
    ours = [(classify(d["Kernel Name"], d["Grid Size"]), float(d["Metric Value"]), d["Metric Unit"], d["Grid Size"])
            for d in rows if "qbk::" in d["Kernel Name"]]
    if per_step:
        ours = ours[-per_step:]
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v, u, g in ours:
        tot[k] += v * scale.get(u, 1e-6)
        cnt[k] += 1
    T = sum(tot.values())
    out = {"source": path, "launches": len(ours), "total_ms": T,
           "note": "ncu launch list: cold-cache, serialised per-launch times; compare shares, not absolutes",
           "kernels": {k: {"launches": cnt[k], "ms": tot[k], "share": tot[k] / T} for k in sorted(tot, key=lambda x: -tot[x])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
