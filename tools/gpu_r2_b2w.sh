# B2W (per-part B2 warps) evidence: ncu --set full of bwd_l0 at c3 and c4a shapes,
# source-level SASS dump for the shared-memory wavefront / replay attribution
mkdir -p gpurun_out
cap() {  # tag skip args...
  local tag=$1 skip=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pyr_bwd_tma -s $skip -c 1 -o gpurun_out/$tag -f python tools/prof_case.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>&1
  rm -f gpurun_out/$tag.ncu-rep
}
cap ${TAG:-b2w}_c3 7 --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2
cap ${TAG:-b2w}_c4a 5 --frames 4 --iters 2
