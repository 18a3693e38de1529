"""DRAM bytes per launch of the bench's kernel classes (bench.py roofline
`traffic`), from ncu launch windows (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum) of the bench workload:

    python tests/ncu_traffic.py win1.csv [win2.csv ...] > profiles/ncu_traffic.json

A class's launch = all its kernels in one coarsening level or refinement
round; the unit kernel counts the launches.  k_contract_edges runs in both
contraction passes (as do the node-list unions): they belong to `contract`
between k_gamma and k_contract_status and to `contract_write` after it
(kernel names come without template arguments, tests/ncu_summary.py)."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402

CLASSES = {
    "score_select": ("k_inc_base", {"k_inc_base", "k_score_warp", "k_score_mid", "k_score_heavy", "k_score_block",
                                    "k_inc_tuples_quick", "k_inc_tuples", "k_inc_finalize"}),
    "propose": ("k_propose_warp", {"k_propose_warp", "k_propose_hub", "k_propose_heavy", "k_hub_prefix",
                                   "k_propose_mid", "k_propose_block"}),
    "contract": ("k_gamma", {"k_gamma", "k_node_count", "k_node_union_warp@count", "k_node_union@count",
                             "k_edge_count_bulk", "k_marked_list", "k_contract_edges@count", "k_contract_status"}),
    "contract_write": ("k_node_union_warp@write", {"k_contract_edges@write", "k_map_gaps", "k_node_write",
                                        "k_node_union_warp@write", "k_node_union@write"}),
    "seq_gains": ("k_round_moves", {"k_round_edges", "k_round_edges_flat", "k_seq_gains_edge_block",
                                    "k_inbound_events_block", "k_edge_movers_huge", "k_round_moves"}),
    "project": ("k_project_state", {"k_gamma_count", "k_project_state", "k_split_counts", "k_project"}),
    "movers": ("k_mover_compact", {"k_mover_compact", "k_mover_flags"}),
    "apply": ("k_apply_inc", {"k_apply_inc", "k_apply"}),
    "select": ("k_select_small", {"k_select_small"}),
    "runs_update": ("k_runs_update", {"k_runs_update", "k_runs_update_wide"}),
}


def per_unit(paths):
    units = {k: 0 for k in CLASSES}
    dram = {k: 0.0 for k in CLASSES}
    for p in paths:
        per, names = load(p)
        phase = "count"
        for i in sorted(per, key=int):
            n = names[i]
            if n == "k_gamma":
                phase = "count"
            elif n == "k_contract_status":
                phase = "write"
            key = f"{n}@{phase}" if n in ("k_contract_edges", "k_node_union", "k_node_union_warp") else n
            m = per[i]
            b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            for cls, (unit, members) in CLASSES.items():
                if key == unit:
                    units[cls] += 1
                if key in members:
                    dram[cls] += b
    return {cls: int(dram[cls] / units[cls]) for cls in CLASSES if units[cls]}


if __name__ == "__main__":
    r = per_unit(sys.argv[1:])
    r["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class (all its kernels in "
                  "one coarsening level / refinement round), from ncu launch windows: " +
                  "; ".join(f"{c} = {sorted(m)} per {u}" for c, (u, m) in CLASSES.items()))
    print(json.dumps(r, indent=1))
