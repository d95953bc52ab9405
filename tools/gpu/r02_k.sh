# round 2, call k: pipelined K1 (bulk-staged persistent) correctness + A/B vs the legacy kernel
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rangecompress or whiten" 2>&1 | tail -15 > gpurun_out/t_k.txt
for rep in 1 2; do for c in 4 2; do for l in 0 1; do SASBP_RC_LEGACY=$l timeout 300 python tools/k1_bench.py --config $c; done; done; done > gpurun_out/k1_k.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_pipe -s 2 -c 1 -o gpurun_out/ncu_k1_k python tools/k1_bench.py --config 4 --reps 3 > gpurun_out/ncu_k1_k.log 2>&1
echo done
