#!/bin/bash
# Profiling recipe for the round's ncu evidence (run on the GPU box; outputs
# under gpurun_out/, summaries copied into profiles/):
#   1. the whole C2 partition's launch list (gpu__time_duration, warm L2:
#      --cache-control none) -> per-kernel shares (tests/launch_summary.py)
#   2. launch windows with DRAM bytes for a coarsening and a refinement stretch
#      (-> tests/ncu_traffic.py: bytes per level / round of the kernel classes)
#   3. --set full captures of the hot kernels at mid-run levels / rounds
set -x
mkdir -p gpurun_out
O=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file $O/c2_all_launches.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 14000 -c 1500 --csv --log-file $O/win_coarsen.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 60000 -c 1500 --csv --log-file $O/win_refine.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(score_heavy|score_warp|runs_update|contract_edges|propose_warp|propose_hub|node_write|node_union|select_small|round_edges)" \
    -s 2400 -c 20 -o $O/full_hot python tests/prof_run.py C2 > $O/ncu_full_hot.log 2>&1
