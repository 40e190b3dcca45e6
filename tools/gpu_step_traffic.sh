#!/bin/bash
# DRAM bytes of every kernel of one c4a-shaped and one c3-shaped fwd+bwd step (ncu metrics, cold launches)
TAG=${1:-r01}
python -m paper_2602_08642_b200.build > /dev/null || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/st_c4a.csv python tools/prof_case.py --frames 4 --iters 2 > /dev/null 2>&1; echo "c4a rc=$?"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/st_c3.csv python tools/prof_case.py --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2 > /dev/null 2>&1; echo "c3 rc=$?"
{ echo "# c4a-shaped step (4 x 1920x1080, L3 k5 fp32)"; python tools/step_traffic.py gpurun_out/st_c4a.csv 8294400;
  echo; echo "# c3-shaped step (1 x 3840x2160, L4 k7 bf16 logits)"; python tools/step_traffic.py gpurun_out/st_c3.csv 8294400; } > gpurun_out/${TAG}_step_traffic.txt 2>&1
cat gpurun_out/${TAG}_step_traffic.txt
