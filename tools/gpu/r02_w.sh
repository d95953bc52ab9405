# round 2, call w: compute-sanitizer over tools/sanitize_cases.py, full output kept (call u's grep hid a failure)
set -x
mkdir -p gpurun_out
which compute-sanitizer; compute-sanitizer --version | head -3
for tool in memcheck racecheck initcheck synccheck; do
  echo "== $tool"; timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ran|degenerate cases ran" gpurun_out/san_$tool.log; tail -5 gpurun_out/san_$tool.log
done > gpurun_out/sanitizers_w.txt 2>&1

for rep in 1 2 3 4 5; do for l in v0 v1; do SASBP_LIB=build_ab/$l.so timeout 300 python tools/k1_bench.py --config 4 --reps 300 | sed "s/^/$l /"; done; done > gpurun_out/ab_k1_w.txt 2>&1
echo done
