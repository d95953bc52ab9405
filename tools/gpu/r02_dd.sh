# round 2, call dd: K0 complex-tap staging with precomputed store addresses (+ interior fast path) vs the previous build
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "baseband or conditioning or fullsize" 2>&1 | tail -3 > gpurun_out/t_dd.txt
for rep in 1 2 3; do for l in build_ab/k0_old.so paper_2101_05888_b200/libsasbp.so; do SASBP_LIB=$l timeout 300 python tools/k0_bench.py --config 4 --reps 100 | sed "s|^|$l |"; SASBP_LIB=$l timeout 300 python tools/k0_bench.py --config 2 --reps 50 | sed "s|^|$l |"; done; done > gpurun_out/ab_dd.txt 2>&1
echo done
