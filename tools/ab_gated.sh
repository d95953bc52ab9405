#!/bin/bash
# A/B of library variants in build_ab/*.so on the dense and the gated (NEXT-1) config-2 launch
for rep in 1 2; do
for lib in ${LIBDIR:-build_ab}/*.so; do
  SASBP_LIB=$lib timeout 300 python bench.py --config ${CFG:-2} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-k1 --no-next4 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', 'dense', round(d['value'],1), 'gated_ms', round(d['next1_gated']['ms_per_step'],2), 'in-cone', round(d['next1_gated']['in_cone_Gterm_per_s'],1))"
done
done
