# round-2 evidence run: full GPU suite, smoke, the default bench line, the ncu
# launch list of the bench command and the step DRAM bytes, one --set full of
# the dominant kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/r2i_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE --durations=15 > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2i_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2i_ref.json 2> gpurun_out/r2i_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-also > gpurun_out/r2i_ncu_bench.log 2>&1
timeout 900 bash tools/gpu_step_traffic.sh r2i > gpurun_out/r2i_step_traffic.log 2>&1
timeout 900 bash tools/gpu_prof_r2.sh r2i > gpurun_out/r2i_prof.log 2>&1
python tools/bench_shapes.py > gpurun_out/r2i_shapes.json 2>&1
python tools/bench_latency.py > gpurun_out/r2i_latency.json 2>&1
