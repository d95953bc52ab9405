# round 2, call p: K0 bulk-staged persistent kernel (a: 2 staging buffers, b: 1) vs the blocked kernel (SASBP_BB_LEGACY=1)
set -x
mkdir -p gpurun_out
for l in a b; do SASBP_LIB=build_ab/k0_$l.so timeout 900 python -m pytest tests -m gpu -x -q -k "baseband or conditioning or fullsize" 2>&1 | tail -2; done > gpurun_out/t_p.txt
for rep in 1 2; do for c in 4 2; do for v in "k0_a.so 0" "k0_b.so 0" "k0_a.so 1"; do set -- $v; SASBP_LIB=build_ab/$1 SASBP_BB_LEGACY=$2 timeout 300 python tools/k0_bench.py --config $c | sed "s/^/$1 legacy=$2 /"; done; done; done > gpurun_out/k0_p.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:baseband_pipe -s 2 -c 1 -o gpurun_out/ncu_k0_p python tools/k0_bench.py --config 4 --reps 3 > gpurun_out/ncu_k0_p.log 2>&1
echo done
