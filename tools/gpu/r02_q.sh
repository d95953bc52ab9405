# round 2, call q: K0 complex-tap kernel (default) vs the mixed blocked kernel (SASBP_BB_LEGACY=1): parity + timing + ncu
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "baseband or conditioning or fullsize" 2>&1 | tail -4 > gpurun_out/t_q.txt
for rep in 1 2; do for c in 4 2; do for l in 0 1; do SASBP_BB_LEGACY=$l timeout 300 python tools/k0_bench.py --config $c | sed "s/^/legacy=$l /"; done; done; done > gpurun_out/k0_q.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:baseband_ctap -s 2 -c 1 -o gpurun_out/ncu_k0_q python tools/k0_bench.py --config 4 --reps 3 > gpurun_out/ncu_k0_q.log 2>&1
echo done
