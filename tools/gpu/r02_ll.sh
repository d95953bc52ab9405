# round 2, call ll: 3D tiles 16x8x12 (12 voxels/thread, 3 CTAs/SM) vs 16x16x8 and 16x8x16 (16 voxels/thread, 2 CTAs/SM)
# vs production 16x8x8, config 4:150, C ABI
set -x
mkdir -p gpurun_out
timeout 1800 python tools/abi_time.py --libs paper_2101_05888_b200/libsasbp.so build_ab/kz3.so build_ab/ky4.so build_ab/kz4.so --configs 4:150 --reps 2 > gpurun_out/ab_ll.txt 2>&1
echo done
