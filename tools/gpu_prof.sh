# ncu launch list, per-kernel DRAM bytes, --set full of the tcgen05 kernels (incl. the compressed-key
# KV-outer launch). Usage: bash tools/gpu_prof.sh <tag>
T=${1:-r2}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-full --no-window --no-learned > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hbm_$T.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full --no-window --no-learned > gpurun_out/ncu_hbm.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 8 -o gpurun_out/prof_$T python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full --no-window --no-learned > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/
