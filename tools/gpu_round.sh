set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_r1d.txt
cat gpurun_out/pytest_gpu_r1d.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; tail -2 gpurun_out/bench_r1d.err; cat gpurun_out/bench_r1d.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1d.json 2>&1; tail -1 gpurun_out/bench_ref_r1d.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-full > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 7 -o gpurun_out/prof_r1d python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
