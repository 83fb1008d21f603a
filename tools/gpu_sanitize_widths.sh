mkdir -p gpurun_out
SAN_TOOLS="memcheck synccheck racecheck" SAN_TIMEOUT=900 bash tools/gpu_sanitize.sh
for tool in memcheck synccheck; do
  BD_TILE_N=256 timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize256_${tool}.log 2>&1
  echo "$tool (BD_TILE_N=256) rc=$?: $(tail -3 gpurun_out/sanitize256_${tool}.log | tr '\n' ' ')"
done
