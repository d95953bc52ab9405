# round 2, call ii: azimuth cone classes on sines (one sqrt) vs two fp64 asin -- gated parity (exact counts, culled ==
# unculled bitwise) and the gated config-2 timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gate or gated or cull or beam or count" 2>&1 | tail -3 > gpurun_out/t_ii.txt
CFG=2 LIBDIR=build_abg timeout 1500 bash tools/ab_gated.sh > gpurun_out/ab_gated_ii.txt 2>&1
echo done
