# Round-2 measurements. Usage: bash tools/gpu_bench.sh <tag>
T=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -3 gpurun_out/bench_$T.err; cat gpurun_out/bench_$T.json
timeout 900 python bench.py --config C4 --no-cpu --no-learned --no-window > gpurun_out/bench_c4_$T.json 2> gpurun_out/bench_c4_$T.err; tail -3 gpurun_out/bench_c4_$T.err; cut -c1-600 gpurun_out/bench_c4_$T.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.json 2>&1; tail -1 gpurun_out/bench_ref_$T.json | cut -c1-400
# N>1 logic on one GPU (gloo; timing meaningless): mode 2 (C5) and the C4 hybrid placement
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config C5 --backend gloo --steps 2 --warmup 3 --no-cpu --no-full --no-window --no-learned > gpurun_out/bench_c5x2_gloo_$T.json 2> gpurun_out/bench_c5x2_gloo_$T.err; tail -2 gpurun_out/bench_c5x2_gloo_$T.err; cut -c1-400 gpurun_out/bench_c5x2_gloo_$T.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config C4 --backend gloo --steps 2 --warmup 3 --no-cpu --no-full --no-window --no-learned > gpurun_out/bench_c4x2_gloo_$T.json 2> gpurun_out/bench_c4x2_gloo_$T.err; tail -2 gpurun_out/bench_c4x2_gloo_$T.err; cut -c1-400 gpurun_out/bench_c4x2_gloo_$T.json
