# round 2, call pp: 2D plane kernels with 16 pixels per thread (32x64 tiles) at 2 CTAs/SM vs production (8 pixels,
# 4 CTAs/SM), config 2, C ABI
set -x
mkdir -p gpurun_out
timeout 1500 python tools/abi_time.py --libs paper_2101_05888_b200/libsasbp.so build_ab/p16.so --configs 2:250 2:1000 --reps 2 > gpurun_out/ab_pp.txt 2>&1
echo done
