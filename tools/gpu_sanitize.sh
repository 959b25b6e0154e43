# compute-sanitizer memcheck / racecheck / synccheck of tools/sanitize_case.py, one case per run (see
# the case list in the script); usage: bash tools/gpu_sanitize.sh <tag> [tools] [cases]
T=${1:-r2}
TOOLS=${2:-"memcheck racecheck synccheck"}
CASES=${3:-"0 1 4 5 2 3"}
for tool in $TOOLS; do
  out=gpurun_out/sanitize_${tool}_$T.txt
  echo "# compute-sanitizer --tool $tool python tools/sanitize_case.py <case> ($T), cases: $CASES" > $out
  for cs in $CASES; do
    echo "## case $cs" >> $out
    timeout 400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $cs >> $out 2>&1
    tail -1 $out
  done
done
