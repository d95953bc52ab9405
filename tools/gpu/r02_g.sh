# round 2, call g: GPU suite (cursor window transform, K0 slack layout), transform A/B dense + gated, K0 A/B
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/gputest_g.txt
timeout 1500 python tools/ab_time.py --libs build_ab3/xf1.so build_ab3/xf0.so --configs 4:150 2:250 --reps 2 > gpurun_out/ab_xf_g.txt 2>&1
CFG=2 LIBDIR=build_ab3 timeout 900 bash tools/ab_gated.sh > gpurun_out/ab_gated_g.txt 2>&1
for rep in 1 2; do for c in 4 2; do for v in 0 1; do SASBP_BB_VEC4=$v timeout 300 python tools/k0_bench.py --config $c; done; done; done > gpurun_out/k0_ab_g.txt 2>&1
echo done
