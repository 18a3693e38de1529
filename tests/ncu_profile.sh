#!/bin/bash
# Round-1b profiling recipe (run on the GPU box; outputs under gpurun_out/):
#   1. launch lists with per-launch time and DRAM bytes for a coarsening and a
#      refinement window of one C2 partition
#   2. --set full captures of the hot kernels at mid-run levels
set -x
mkdir -p gpurun_out
O=gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -s 14000 -c 1500 --csv --log-file $O/win_coarsen.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 60000 -c 1500 --csv --log-file $O/win_refine.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(score_heavy|score_warp|contract_edges|merge_write|propose_hub|propose_warp|select_small|round_edges|runs_update|inc_tuples_quick)" \
    -s 2400 -c 20 -o $O/full_hot python tests/prof_run.py C2 > $O/ncu_full_hot.log 2>&1
