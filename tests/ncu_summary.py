"""Summarise ncu launch lists with time + DRAM bytes per launch (tests/ncu_profile.sh):
per kernel: launches, total / mean microseconds, DRAM bytes per launch, achieved DRAM GB/s."""
import collections
import csv
import io
import json
import sys


def load(path):
    lines = open(path).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[u]
        else:
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        per[r["ID"]][r["Metric Name"]] = v
        names[r["ID"]] = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "").split("<")[0]
    return per, names


def summary(path):
    per, names = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    out = []
    for k, (n, us, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "us_total": round(us, 1), "us_mean": round(us / n, 2),
                    "dram_bytes_per_launch": round(b / n), "dram_gbs": round(b / (us * 1e3), 1) if us else None})
    return out


if __name__ == "__main__":
    res = {p: summary(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
