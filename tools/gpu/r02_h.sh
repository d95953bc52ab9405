# round 2, call h: same-box A/B of the current K2 vs the kernel without the wave-tail split vs round 2's first sepq build;
# gated A/B; K1 packed at 2 CTAs/SM; K0 ncu
set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py --libs build_ab4/cur.so build_ab4/nots.so build_ab4/headb_sepq.so --configs 4:150 2:250 --reps 2 > gpurun_out/ab_h.txt 2>&1
CFG=2 LIBDIR=build_ab4 timeout 900 bash tools/ab_gated.sh > gpurun_out/ab_gated_h.txt 2>&1
for rep in 1 2; do for l in build_ab4/cur.so build_ab4/pack2.so; do for c in 4 2; do SASBP_LIB=$l timeout 300 python tools/k1_bench.py --config $c; done; done; done > gpurun_out/k1_h.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:baseband -s 2 -c 1 -o gpurun_out/ncu_k0_h python tools/k0_bench.py --config 4 --reps 2 > gpurun_out/ncu_k0_h.log 2>&1
echo done
