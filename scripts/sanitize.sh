# compute-sanitizer over scripts/exp/sanitize_driver.py (every kernel family, small shapes)
# usage (under gpurun): bash scripts/sanitize.sh <outdir>
OUT=${1:-gpurun_out/sanitizer}
mkdir -p $OUT
for tool in memcheck synccheck racecheck; do
  timeout -s KILL 1200 compute-sanitizer --tool $tool --target-processes all python scripts/exp/sanitize_driver.py > $OUT/$tool.log 2>&1
  echo rc=$? >> $OUT/$tool.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=" $OUT/$tool.log | sed "s/^/$tool: /"
done
