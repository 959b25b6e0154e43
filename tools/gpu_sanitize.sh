# compute-sanitizer memcheck / racecheck / synccheck of tools/sanitize_case.py; usage: bash tools/gpu_sanitize.sh <tag>
T=${1:-r2}
for tool in memcheck racecheck synccheck; do
  echo "# compute-sanitizer --tool $tool python tools/sanitize_case.py ($T)" > gpurun_out/sanitize_${tool}_$T.txt
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_case.py >> gpurun_out/sanitize_${tool}_$T.txt 2>&1
  tail -1 gpurun_out/sanitize_${tool}_$T.txt
done
