timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_bf16_full or single_token or c1_fp32" 2>&1 | tail -30
