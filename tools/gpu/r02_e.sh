# round 2, call e: gated K2 A/B (out-of-line fp64 cone masks, with split / prefetch)
set -x
mkdir -p gpurun_out
CFG=2 LIBDIR=build_ab2 timeout 1500 bash tools/ab_gated.sh > gpurun_out/ab_gated_e.txt 2>&1
echo done
