timeout 600 python -m pytest tests/test_gpu_learned.py tests/test_gpu_shard.py tests/test_gpu_window.py -q --timeout 300 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/learned_launches.csv python tools/learned_step.py 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/learned_launches.csv 2 | head -14
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config C5 --backend gloo --steps 2 --warmup 3 --no-cpu --no-full --no-window --no-learned > gpurun_out/bench_c5x2_gloo.json 2> gpurun_out/bench_c5x2_gloo.err; tail -2 gpurun_out/bench_c5x2_gloo.err; cut -c1-300 gpurun_out/bench_c5x2_gloo.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config C4 --backend gloo --steps 2 --warmup 3 --no-cpu --no-full --no-window --no-learned > gpurun_out/bench_c4x2_gloo.json 2> gpurun_out/bench_c4x2_gloo.err; tail -2 gpurun_out/bench_c4x2_gloo.err; cut -c1-300 gpurun_out/bench_c4x2_gloo.json
bash tools/gpu_sanitize.sh r2
