timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_shard.py -x -q 2>&1 | tail -3
bash tools/gpu_ab.sh A main
for L in A main; do lib=paper_2505_17412_b200/libssa_$L.so; [ $L = main ] && lib=paper_2505_17412_b200/libssa_b200.so
SSA_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --csv -k regex:"k_kv_reduce|k_bwd_final_kv|k_gather_gates" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-full 2>/dev/null | grep -E "k_kv_reduce|k_bwd_final_kv|k_gather_gates" | awk -F'","' '{print "'$L'", $5, $NF}' | sort | uniq -c | head -12; done
