# round 2, call i: 2D dense regression bisect (same box), K0 9-float4 staging
set -x
mkdir -p gpurun_out
timeout 1800 python tools/ab_time.py --libs build_ab5/a_cur.so build_ab5/b_nokph.so build_ab5/c_nogc.so build_ab5/d_nokph_nogc.so build_ab5/e_nots_nokph_nogc.so build_ab5/f_headb.so --configs 2:250 4:100 --reps 2 > gpurun_out/ab_i.txt 2>&1
for rep in 1 2; do for c in 4 2; do for v in 0 1; do SASBP_BB_VEC4=$v timeout 300 python tools/k0_bench.py --config $c; done; done; done > gpurun_out/k0_ab_i.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_next4.py -k "baseband" -x -q 2>&1 | tail -3 > gpurun_out/t_i.txt
echo done
