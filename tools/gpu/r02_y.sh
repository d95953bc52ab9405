# round 2, call y: 2D regression hunt -- historical builds (round-1 end 788ec27, ae399ec AXIS, fc88600 prefetch,
# a8e9db7 tail split / host kph / gate_mask, 047e8ae cursor transform) vs HEAD, C ABI only, same box
set -x
mkdir -p gpurun_out
timeout 2000 python tools/abi_time.py --libs build_r1/788ec27.so build_r1/ae399ec.so build_r1/fc88600.so build_r1/a8e9db7.so build_r1/047e8ae.so paper_2101_05888_b200/libsasbp.so --configs 2:250 4:100 --reps 2 > gpurun_out/ab_y.txt 2>&1
echo done
