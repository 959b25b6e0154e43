T=r1f
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-full --no-window > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hbm_$T.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full --no-window > /dev/null 2>&1
echo done
