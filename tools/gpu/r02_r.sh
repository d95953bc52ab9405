# round 2, call r: source-level ncu of the gated (NEXT-1) K2 on config 2 (tools/prof_gated.py)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdbp -c 1 -o gpurun_out/ncu_gated_r python tools/prof_gated.py > gpurun_out/ncu_gated_r.log 2>&1
echo done
