# A/B timing of library variants built with SSA_LIB_OUT (tools: see DESIGN.md §5); args: variant names
for r in 1 2; do
for v in "$@"; do
  lib=paper_2505_17412_b200/libssa_$v.so; [ "$v" = main ] && lib=paper_2505_17412_b200/libssa_b200.so
  SSA_LIB=$lib timeout 600 python bench.py --no-cpu --no-full --no-e2e --no-window --no-learned 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], {k: round(x,3) for k,x in d['kernel_ms'].items()})"
done; done
