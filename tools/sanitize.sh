# compute-sanitizer over tools/sanitize_cases.py (every kernel family); summaries in gpurun_out/sanitize_*.txt
out=gpurun_out; mkdir -p $out
python tools/sanitize_cases.py > $out/sanitize_plain.txt 2>&1; echo "exit $?" >> $out/sanitize_plain.txt
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > $out/sanitize_$tool.txt 2>&1
  echo "exit $?" >> $out/sanitize_$tool.txt
done
