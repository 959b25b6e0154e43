# GPU parity suite with the per-tensor parity report. Usage: bash tools/gpu_tests.sh <tag> [pytest args]
T=${1:-r2}; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
SSA_PARITY_REPORT=gpurun_out/parity_$T.json timeout 1500 python -m pytest tests -m gpu -q -rfE --durations=20 --timeout 600 "$@" 2>&1 | tail -60 > gpurun_out/pytest_gpu_$T.txt
tail -40 gpurun_out/pytest_gpu_$T.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
