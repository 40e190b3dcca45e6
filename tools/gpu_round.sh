# round evidence: full default bench line, launch list of the c4a-shaped step, ncu full summaries of the top kernels
TAG=${1:-r01}
mkdir -p gpurun_out
python -m paper_2602_08642_b200.build > /dev/null || exit 1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/prof_case.py --frames 4 --iters 2 > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_list.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pyr_ -s 9 -c 9 -o gpurun_out/${TAG}_all -f python tools/prof_case.py --frames 4 --iters 2 > gpurun_out/${TAG}_ncu_all.log 2>&1; echo "ncu all rc=$?"
python tools/ncu_summary.py gpurun_out/${TAG}_all.ncu-rep > gpurun_out/${TAG}_all_summary.txt 2>&1
ncu -i gpurun_out/${TAG}_all.ncu-rep --page details > gpurun_out/${TAG}_all_details.txt 2>&1
ncu -i gpurun_out/${TAG}_all.ncu-rep --page raw --csv > gpurun_out/${TAG}_all_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
