"""bigedge.npz: an instance with one h-edge of 8,300 pins (above the 8,192
slots a per-segment sort keeps in shared memory) on top of a gen.py-style
graph, partitioned by the REFERENCE (oracle/_ref).  Stores the inputs and the
reference's assign / num_parts / levels / trace.  Run here (minutes):

    python tests/golden/make_bigedge_golden.py
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_loader  # noqa: E402
from paper_2604_14411_b200 import workloads as W  # noqa: E402


def big_instance(n=9000, big=8300, seed=5):
    N, w, so, sd, do, dd = W.random_dhg(n, int(1.2 * n), 6, seed=seed)
    rs = np.random.RandomState(seed)
    members = np.sort(rs.choice(n, size=big, replace=False)).astype(np.int32)
    so = np.concatenate([so, [so[-1] + 1]]).astype(np.int64)
    sd = np.concatenate([sd, members[:1]]).astype(np.int32)
    do = np.concatenate([do, [do[-1] + big - 1]]).astype(np.int64)
    dd = np.concatenate([dd, members[1:]]).astype(np.int32)
    w = np.concatenate([w, [3.0]])
    return N, w, so, sd, do, dd


def main():
    dp = ref_loader.load()
    arr = big_instance()
    n, w, so, sd, do, dd = arr
    omega = 256
    delta = int(np.bincount(dd, minlength=n).max()) + 8
    g = dp.Hypergraph._from_csr(n, w, dp.CsrSets(so, sd), dp.CsrSets(do, dd))
    t = time.perf_counter()
    part, st = dp.partition(g, dp.Config(dp.Constraints(omega, delta), max_levels=1 << 20))
    secs = time.perf_counter() - t
    out = {f"in_{k}": np.asarray(v) for k, v in zip(("n", "w", "so", "sd", "do", "dd"), arr)}
    out.update(omega=np.int64(omega), delta=np.int64(delta), assign=part.assign, num_parts=np.int64(part.num_parts),
               stats=np.frombuffer(json.dumps({"levels": st.levels, "trace": st.connectivity_trace,
                                               "reference_seconds": secs}).encode(), np.uint8))
    np.savez_compressed(Path(__file__).resolve().parent / "bigedge.npz", **out)
    print("bigedge", round(secs, 1), "s", len(st.levels), "levels", part.num_parts, "parts")


if __name__ == "__main__":
    main()
