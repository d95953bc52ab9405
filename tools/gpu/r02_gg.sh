# round 2, call gg: 3D kernel variants (config 4): tile-group size 4 / 16 (launch-order locality) and 24 channels per batch
# vs production; plus the production kernel's DRAM bytes per variant on a 150-ping slice
set -x
mkdir -p gpurun_out
timeout 1800 python tools/abi_time.py --libs paper_2101_05888_b200/libsasbp.so build_ab/tg4.so build_ab/tg16.so build_ab/nb24.so --configs 4:150 --reps 2 > gpurun_out/ab_gg.txt 2>&1
echo done
