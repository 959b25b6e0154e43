# round-end GPU measurements: tests, smoke, bench (both arms), ncu launch list, DRAM metrics of every
# kernel, ncu --set full of the tcgen05 kernels. Usage: bash tools/gpu_round.sh <tag>
T=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$T.txt
cat gpurun_out/pytest_gpu_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -2 gpurun_out/bench_$T.err; cat gpurun_out/bench_$T.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.json 2>&1; tail -1 gpurun_out/bench_ref_$T.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-full --no-window > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hbm_$T.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full --no-window > gpurun_out/ncu_hbm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 7 -o gpurun_out/prof_$T python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full --no-window > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
