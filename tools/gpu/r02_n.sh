# round 2, call n: gated K2 A/B -- g1: predicated accumulate (new default), g0: zero-cell address select (old),
# g3: predicated + 3 CTAs/SM for the gated kernels (no spills)
set -x
mkdir -p gpurun_out
SASBP_LIB=build_ab/gate_g1.so timeout 900 python -m pytest tests -m gpu -x -q -k "gate or gated" 2>&1 | tail -3 > gpurun_out/t_n.txt
mkdir -p build_abg && mv build_ab/gate_*.so build_abg/
CFG=2 LIBDIR=build_abg timeout 1500 bash tools/ab_gated.sh > gpurun_out/ab_gated_n.txt 2>&1
echo done
