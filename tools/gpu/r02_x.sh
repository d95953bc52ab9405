# round 2, call x: 2D dense regression bisect (config 2 was ~1351 Gterm/s on 250-ping slices early in round 2, ~1300 later):
# a = current, b = 2 pi fc/fs and fs/c derived on the device (SASBP_KPH_PARAM=0), c = params without __grid_constant__,
# d = no wave-tail split support compiled in, e = all three
set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py --libs build_ab2/a.so build_ab2/b.so build_ab2/c.so build_ab2/d.so build_ab2/e.so --configs 2:250 4:100 --reps 2 > gpurun_out/ab_x.txt 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2_x.json 2> gpurun_out/bench_cfg2_x.err
echo done
