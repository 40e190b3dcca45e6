# one ncu --set full capture of the level-0 backward (level-0-last order: the last k_pyr_bwd_tma launch of the second iteration; SKIP_C4A=3 SKIP_C3=4 for SSB_NO_CHAIN=1) (c4a-shaped, 4 frames) and of c3's; summaries on the box
TAG=${1:-p}
mkdir -p gpurun_out
python -m paper_2602_08642_b200.build > /dev/null || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pyr_bwd_tma -s ${SKIP_C4A:-5} -c 1 -o gpurun_out/${TAG}_bwd_c4a -f python tools/prof_case.py --frames 4 --iters 2 > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu c4a rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pyr_bwd_tma -s ${SKIP_C3:-7} -c 1 -o gpurun_out/${TAG}_bwd_c3 -f python tools/prof_case.py --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2 > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu c3 rc=$?"
for r in bwd_c4a bwd_c3; do
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page details > gpurun_out/${TAG}_${r}_details.txt 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${r}_sass.csv 2>&1
done
python tools/ncu_lines.py gpurun_out/${TAG}_bwd_c4a.ncu-rep k_pyr_bwd_tma 400 8294400 > gpurun_out/${TAG}_bwd_c4a_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/${TAG}_bwd_c3.ncu-rep k_pyr_bwd_tma 400 8294400 > gpurun_out/${TAG}_bwd_c3_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep; du -sh gpurun_out; ls -la gpurun_out/
