"""DRAM bytes per launch of the bench's kernel classes (bench.py roofline
`traffic`), from the launch windows of tests/ncu_profile.sh:
score_select = per coarsening level (levels counted by k_inc_base),
propose = per refinement round (rounds counted by k_propose_warp).
Usage: python tests/ncu_traffic.py win_coarsen.csv win_refine.csv > profiles/ncu_traffic.json"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402

CLASSES = {
    "score_select": ("k_inc_base", {"k_inc_base", "k_score_warp", "k_score_heavy", "k_score_block",
                                    "k_inc_tuples_quick", "k_inc_tuples", "k_inc_finalize"}),
    "propose": ("k_propose_warp", {"k_propose_warp", "k_propose_hub", "k_propose_heavy", "k_hub_prefix",
                                   "k_propose_mid", "k_propose_block"}),
}


def per_unit(paths):
    out = {}
    for cls, (unit, members) in CLASSES.items():
        units, dram = 0, 0.0
        for p in paths:
            per, names = load(p)
            for i, m in per.items():
                n = names[i]
                if n == unit:
                    units += 1
                if n in members:
                    dram += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if units:
            out[cls] = int(dram / units)
    return out


if __name__ == "__main__":
    r = per_unit(sys.argv[1:])
    r["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class (all its kernels in "
                  "one coarsening level / refinement round), from the ncu launch windows of tests/ncu_profile.sh: "
                  "score_select = k_inc_base + k_score_{warp,heavy,block} (2 passes) + k_inc_tuples(_quick) + "
                  "k_inc_finalize per level; propose = k_propose_{warp,hub,heavy,mid,block} + k_hub_prefix per round")
    print(json.dumps(r, indent=1))
