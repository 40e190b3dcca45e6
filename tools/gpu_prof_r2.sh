# ncu --set full captures of the backward level kernels (c4a-shaped 4 frames:
# bwd_l1 and bwd_l0; c3: bwd_l0) with line-level attribution
TAG=${1:-p2}
mkdir -p gpurun_out
prof() {  # name skip regex args...
  local name=$1 skip=$2 rx=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o gpurun_out/${TAG}_$name -f \
     python tools/prof_case.py "$@" > gpurun_out/${TAG}_${name}_ncu.log 2>&1; echo "ncu $name rc=$?"
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page details > gpurun_out/${TAG}_${name}_details.txt 2>&1
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page raw --csv > gpurun_out/${TAG}_${name}_raw.csv 2>&1
  python tools/ncu_lines.py gpurun_out/${TAG}_$name.ncu-rep $rx 60 > gpurun_out/${TAG}_${name}_lines.txt 2>&1
  python tools/ncu_lines.py gpurun_out/${TAG}_$name.ncu-rep $rx 60 0 --by-stall > gpurun_out/${TAG}_${name}_stall_lines.txt 2>&1
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${name}_sass.csv 2>&1
}
# per iteration: bwd_l1, bwd_l2 (k_pyr_bwd_tma), then bwd_l0: launches 0,1,2 | 3,4,5
prof bwd0_c4a 5 k_pyr_bwd_tma --frames 4 --iters 2
prof bwd1_c4a 3 k_pyr_bwd_tma --frames 4 --iters 2
prof bwd0_c3 7 k_pyr_bwd_tma --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2
rm -f gpurun_out/*.ncu-rep
