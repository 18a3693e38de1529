"""Per-kernel summary of a whole-run ncu launch list (gpu__time_duration.sum only):
launches, total / p50 / p90 / p99 / max microseconds.  Usage:
python tests/launch_summary.py launches.csv [top]"""
import collections
import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402


def summary(path, top=40):
    per, names = load(path)
    by = collections.defaultdict(list)
    for i in sorted(per, key=int):
        by[names[i]].append(per[i].get("gpu__time_duration.sum", 0.0))
    total = sum(sum(v) for v in by.values())
    rows = []
    for k, v in sorted(by.items(), key=lambda x: -sum(x[1]))[:top]:
        a = np.array(v)
        rows.append({"kernel": k, "launches": len(a), "ms": round(a.sum() / 1e3, 2),
                     "share": round(a.sum() / total, 4), "p50_us": round(float(np.median(a)), 1),
                     "p90_us": round(float(np.percentile(a, 90)), 1), "p99_us": round(float(np.percentile(a, 99)), 1),
                     "max_us": round(float(a.max()), 1)})
    return {"launches": sum(len(v) for v in by.values()), "kernel_ms": round(total / 1e3, 1), "kernels": rows}


if __name__ == "__main__":
    r = summary(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
    print(json.dumps(r, indent=1))
