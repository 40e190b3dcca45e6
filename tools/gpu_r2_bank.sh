timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_bank_tests.txt 2>&1
ALT=tools/ab/libssb200_base.so WL="c4a c3" ROUNDS=2 bash tools/ab_bench.sh > gpurun_out/r2_bank_ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pyr_bwd_tma -s 7 -c 1 -o gpurun_out/bank_c4a -f python tools/prof_case.py --frames 1 --h 2160 --w 3840 --levels 4 --k 7 --ldt bf16 --iters 2 > /dev/null 2>&1
ncu -i gpurun_out/bank_c4a.ncu-rep --page source --csv --print-source sass > gpurun_out/bank_c4a_sass.csv 2>&1
ncu -i gpurun_out/bank_c4a.ncu-rep --page details > gpurun_out/bank_c4a_details.txt 2>&1
rm -f gpurun_out/bank_c4a.ncu-rep
