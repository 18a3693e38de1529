"""Key --set full metrics per captured launch of an .ncu-rep (summaries for
profiles/).  Usage: python tests/ncu_details.py report.ncu-rep > out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    per = {}
    for r in rows:
        i = int(r["ID"])
        d = per.setdefault(i, {"id": i, "kernel": r["Kernel Name"].split("(")[0].replace("void ", "")})
        if r["Metric Name"] in KEYS and r["Metric Name"] not in d:
            d[r["Metric Name"]] = f'{r["Metric Value"]} {r["Metric Unit"]}'.strip()
    return [per[k] for k in sorted(per)]


if __name__ == "__main__":
    print(json.dumps(details(sys.argv[1]), indent=1))
