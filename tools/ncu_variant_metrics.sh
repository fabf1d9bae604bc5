#!/bin/bash
# Per-variant raster metrics (one C2 view each): shared wavefronts / conflicts, issue, LSU pipe.
mkdir -p gpurun_out
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  timeout 600 ncu --metrics $M --clock-control none -k regex:raster_kernel -s 20 -c 1 --csv python bench.py --no-e2e --no-cpu --no-check --steps 1 --warmup 3 > gpurun_out/ncuv_$n.csv 2>/dev/null
  echo "== $n"; grep -E '"(gpu__time|smsp__inst|l1tex|smsp__issue|smsp__average)' gpurun_out/ncuv_$n.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
cp /tmp/lib_orig.so $LIB
