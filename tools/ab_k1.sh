mkdir -p gpurun_out/ab
for v in head cur; do
  if [ $v = head ]; then export PJG_LIB=variants/libpjg_head.so; else unset PJG_LIB; fi
  PJG_NO_REPLAY=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,launch__registers_per_thread,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio --clock-control none -k regex:"k1_sync" --csv --log-file gpurun_out/ab/$v.csv python tools/profile_run.py --config 3 --reps 1 > /dev/null 2>&1
done
