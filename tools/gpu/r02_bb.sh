# round 2, call bb: full config 2 (1000 pings) A/B of the 2D plane-kernel settings: previous production (a0) vs new,
# C-ABI timing on device-random echoes and the bench (synthetic scene) with each library; gated/dense bitwise test
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "open_gate or tail_split or cull or gated_stripmap" 2>&1 | tail -3 > gpurun_out/t_bb.txt
timeout 1800 python tools/abi_time.py --libs build_ab3/a0.so paper_2101_05888_b200/libsasbp.so --configs 2:1000 2:250 --reps 2 > gpurun_out/ab_bb.txt 2>&1
for l in build_ab3/a0.so paper_2101_05888_b200/libsasbp.so; do SASBP_LIB=$l timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-k1 --no-next4 --no-gated 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$l', round(d['value'],1), round(d['roofline']['frac'],4))"; done > gpurun_out/bench_ab_bb.txt 2>&1
echo done
