# placement + small-frame inference kernels (round 2 final): per-kernel time, instructions, issue, DRAM
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pp_c1.csv python tools/prof_c1.py > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pp_train.csv python tools/prof_place_train.py > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pp_c0.csv python tools/inf_timing.py > /dev/null 2>&1
echo done
