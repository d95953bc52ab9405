# round 2, call v: K1 NS=16 passes with table twiddles (RC_TW16) and K0 at 8 CTAs/SM (BB_CTAP_MINB=8): v1 vs v0
set -x
mkdir -p gpurun_out
SASBP_LIB=build_ab/v1.so timeout 900 python -m pytest tests -m gpu -x -q -k "rangecompress or whiten or baseband or fullsize" 2>&1 | tail -3 > gpurun_out/t_v.txt
for rep in 1 2 3; do for l in v0 v1; do SASBP_LIB=build_ab/$l.so timeout 300 python tools/k1_bench.py --config 4 | sed "s/^/$l /"; SASBP_LIB=build_ab/$l.so timeout 300 python tools/k0_bench.py --config 4 | sed "s/^/$l /"; done; done > gpurun_out/ab_v.txt 2>&1
echo done
