"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel
count / total / mean microseconds (diagnostics for profiles/)."""
import collections, csv, io, sys

lines = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
tot = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    v = {"ns": v / 1000, "nsecond": v / 1000, "us": v, "usecond": v, "ms": v * 1000, "msecond": v * 1000}[u]
    k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:48]
    tot[k][0] += 1
    tot[k][1] += v
    seq.append((k, round(v, 1), r["Grid Size"]))
s = sum(v[1] for v in tot.values())
n = sum(v[0] for v in tot.values())
print(f"kernels {n}  sum {s:.1f} us  mean {s / max(n, 1):.2f} us")
for k, v in sorted(tot.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{k:48s} {v[0]:6d} {v[1]:10.1f} {v[1] / v[0]:8.2f}")
if len(sys.argv) > 2:
    for x in seq[: int(sys.argv[2])]:
        print(x)
