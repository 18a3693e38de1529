"""Golden fixtures for the comparison baselines, produced by running the
REFERENCE's own ``one_pass`` / ``overlap_greedy`` (baselines.py:16-91, via
oracle/_ref built from /root/reference).  Run here:

    python tests/golden/make_baseline_golden.py

baselines.npz — 12 seeded instances (gen.py-style random and layered-SNN
shapes, unit and non-unit node sizes): inputs, limits, and the reference's
assignments and partition counts for both methods.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_loader  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402


def main():
    ref = ref_loader.load()
    out = {}
    rs = np.random.RandomState(2024)
    cases = []
    for t in range(8):
        n = int(rs.randint(20, 900))
        arr = W.random_dhg(n, int(rs.choice([1, 2, 3])) * n, int(rs.choice([3, 5, 8])), seed=3100 + t)
        indeg = int(np.bincount(arr[5], minlength=n).max()) if len(arr[5]) else 0
        sizes = rs.randint(1, 4, size=n).astype(np.int32) if t % 3 == 2 else None
        omega = int(rs.choice([4, 16, 64])) + (3 if sizes is not None else 0)
        cases.append((arr, sizes, omega, max(indeg, 1) + int(rs.randint(0, 40))))
    for t, (layers, width) in enumerate(((4, 150), (6, 200), (3, 400), (5, 100))):
        arr = W.layered_snn(layers, width, fanout=24, window=64, seed=50 + t)
        cases.append((arr, None, int((64, 128, 256, 32)[t]), int((512, 4096, 1024, 256)[t])))
    for i, (arr, sizes, omega, delta) in enumerate(cases):
        n, w, so, sd, do, dd = arr
        g = ref.Hypergraph._from_csr(n, w, ref.CsrSets(so, sd), ref.CsrSets(do, dd), node_size=sizes)
        c = ref.Constraints(omega, delta)
        p1 = ref.one_pass(g, c)
        p2 = ref.overlap_greedy(g, c)
        for k, v in zip(("n", "w", "so", "sd", "do", "dd"), arr):
            out[f"c{i}_in_{k}"] = np.asarray(v)
        out[f"c{i}_size"] = np.asarray(sizes if sizes is not None else np.ones(n, np.int32))
        out[f"c{i}_omega"] = np.int64(omega)
        out[f"c{i}_delta"] = np.int64(delta)
        out[f"c{i}_onepass"] = p1.assign
        out[f"c{i}_onepass_k"] = np.int64(p1.num_parts)
        out[f"c{i}_overlap"] = p2.assign
        out[f"c{i}_overlap_k"] = np.int64(p2.num_parts)
        print(i, n, omega, delta, p1.num_parts, p2.num_parts, flush=True)
    out["cases"] = np.arange(len(cases))
    np.savez_compressed(Path(__file__).resolve().parent / "baselines.npz", **out)


if __name__ == "__main__":
    main()
