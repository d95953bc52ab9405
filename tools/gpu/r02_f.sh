# round 2, call f: conditioning tests (K0 float4 staging, swizzled periodogram), whitening + K0 A/B, gated ncu
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next4.py tests/test_gpu_fullsize_conditioning.py tests/test_gpu_random.py -k "baseband or whiten or conditioning or rangecompress" -x -q 2>&1 | tail -5 > gpurun_out/t_f.txt
LIBS="build_ab_wh/wh0.so build_ab_wh/wh1.so" timeout 900 bash tools/wh_ab.sh > gpurun_out/wh_ab_f.txt 2>&1
for rep in 1 2; do for c in 4 2; do for v in 0 1; do SASBP_BB_VEC4=$v timeout 300 python tools/k0_bench.py --config $c; done; done; done > gpurun_out/k0_ab_f.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tdbp -c 1 -o gpurun_out/ncu_gated_f python tools/prof_gated.py > gpurun_out/ncu_gated_f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:baseband -s 2 -c 1 -o gpurun_out/ncu_k0_f python tools/k0_bench.py --config 4 --reps 2 > gpurun_out/ncu_k0_f.log 2>&1
echo done
