# round 2, call b: K1 packed-record parity + timing, K2 3D A/B (separable q, exponent-aligned cell index), ubench, gated ncu
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "rangecompress" -x -q 2>&1 | tail -5 > gpurun_out/t_b.txt
timeout 600 python -m pytest tests/test_gpu_random.py -k "conditioning" -x -q 2>&1 | tail -3 >> gpurun_out/t_b.txt
timeout 600 python -m pytest tests/test_gpu_next4.py -k "rangecompress or whiten" -x -q 2>&1 | tail -3 >> gpurun_out/t_b.txt
for c in 4 2; do timeout 300 python tools/k1_bench.py --config $c; SASBP_RC_NOPACK=1 timeout 300 python tools/k1_bench.py --config $c; done > gpurun_out/k1_b.txt 2>&1
timeout 1500 python tools/ab_time.py --libs build_ab/base.so build_ab/sepq.so build_ab/bin.so build_ab/binsepq.so --configs 4:150 2:250 --reps 2 > gpurun_out/ab_b.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes tools/ubench/pipes.cu && /tmp/pipes > gpurun_out/ubench_r02.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tdbp -c 1 -o gpurun_out/ncu_gated_r02 python tools/prof_gated.py > gpurun_out/ncu_gated.log 2>&1
echo done
