# usage: bash tools/gpu_prof.sh TAG  -- launch list + ncu --set full of the level kernels (c4a-shaped 4 frames, and c3)
TAG=${1:-p}
mkdir -p gpurun_out
python -m paper_2602_08642_b200.build > /dev/null
timeout 300 python tools/prof_case.py --frames 4 --iters 2 > gpurun_out/${TAG}_case.log 2>&1 || { echo "case failed"; cat gpurun_out/${TAG}_case.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/prof_case.py --frames 4 --iters 2 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pyr_ -s 6 -c 6 -o gpurun_out/${TAG}_c4a -f python tools/prof_case.py --frames 4 --iters 2 > gpurun_out/${TAG}_ncu_c4a.log 2>&1; echo "ncu c4a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pyr_ -s 8 -c 8 -o gpurun_out/${TAG}_c3 -f python tools/prof_case.py --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2 > gpurun_out/${TAG}_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
# summarise on the box (reports can exceed gpurun's 64 MiB copy-back limit)
for r in c4a c3; do
  python tools/ncu_summary.py gpurun_out/${TAG}_$r.ncu-rep --stalls > gpurun_out/${TAG}_${r}_summary.txt 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page details > gpurun_out/${TAG}_${r}_details.txt 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>&1
done
python tools/launch_list.py gpurun_out/${TAG}_launches.csv --skip 9 > gpurun_out/${TAG}_launches.txt 2>&1
mkdir -p gpurun_out/reps; mv gpurun_out/*.ncu-rep gpurun_out/reps/ 2>/dev/null
du -sh gpurun_out/reps; ls -la gpurun_out/reps
# keep at most ~40 MB of reports
for f in gpurun_out/reps/*.ncu-rep; do s=$(stat -c %s $f); if [ $s -gt 20000000 ]; then rm -f $f; fi; done
