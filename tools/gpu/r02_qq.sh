# round 2, call qq: 3D tiles 16x12x16 (24 voxels per thread, 2 CTAs/SM, 241 registers) vs production 16x8x16 (16 voxels)
set -x
mkdir -p gpurun_out
timeout 1500 python tools/abi_time.py --libs paper_2101_05888_b200/libsasbp.so build_ab/v24.so --configs 4:150 --reps 2 > gpurun_out/ab_qq.txt 2>&1
echo done
