# round 2, call u: compute-sanitizer over tools/sanitize_cases.py (round-2 kernels included) + bench re-run with the
# longer short-kernel warm-up
set -x
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/san_plain.txt 2>&1
for tool in memcheck racecheck initcheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Error|hazard|all cases ran|degenerate cases ran" | head -20
done > gpurun_out/sanitizers_u.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
echo done
