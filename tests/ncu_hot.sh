#!/bin/bash
# Profiling recipe for the round's ncu evidence (run on the GPU box):
#   1. launch list (gpu__time_duration) for a mid-run window of a C2 partition
#   2. --set full captures of the hot kernels at a mid level of C2
# Outputs go to gpurun_out/; summaries are copied into profiles/ by hand.
set -x
mkdir -p gpurun_out
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 40000 -c 2500 --csv --log-file $OUT/launches_c2_window.csv python tests/prof_run.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(propose_warp|edge_runs_fused|score_warp|score_heavy|score_block|merge_write|merge_count|seg_sort_warp|seq_gains_dn|select_small|propose_heavy|scan_onepass|k_line_pass1)" \
    -s 30000 -c 14 -o $OUT/c2_hot python tests/prof_run.py C2 > $OUT/ncu_c2_hot.log 2>&1
