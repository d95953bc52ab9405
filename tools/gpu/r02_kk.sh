# round 2, call kk: 3D tiles with 12 voxels per thread at 3 CTAs/SM (160 registers): 16x12x8 (ky3) and 16x8x12 (kz3)
# vs production 16x8x8 (8 voxels, 4 CTAs/SM, 123 registers), config 4:150, C ABI
set -x
mkdir -p gpurun_out
timeout 1800 python tools/abi_time.py --libs paper_2101_05888_b200/libsasbp.so build_ab/ky3.so build_ab/kz3.so --configs 4:150 --reps 2 > gpurun_out/ab_kk.txt 2>&1
echo done
