# round 2, call t: two-launch gated K2 (IN pairs through a mask-free kernel, then the edge pairs) -- parity + A/B
set -x
mkdir -p gpurun_out
SASBP_LIB=build_abg/g_two.so timeout 900 python -m pytest tests -m gpu -x -q -k "gate or gated or cull or beam" 2>&1 | tail -3 > gpurun_out/t_t.txt
for rep in 1 2; do for v in "g_two.so 0" "g_two.so 1" "g_two_cur.so 0"; do set -- $v;
  SASBP_LIB=build_abg/$1 SASBP_GATE_ONE=$2 timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-k1 --no-next4 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 one=$2', 'dense', round(d['value'],1), 'gated_ms', round(d['next1_gated']['ms_per_step'],2), 'in-cone', round(d['next1_gated']['in_cone_Gterm_per_s'],1))"
done; done > gpurun_out/ab_gated_t.txt 2>&1
echo done
