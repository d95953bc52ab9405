#!/bin/bash
# A/B benchmark of library variants in build_ab/*.so (same box, interleaved twice)
for rep in 1 2; do
for lib in ${LIBDIR:-build_ab}/*.so; do
  SASBP_LIB=$lib timeout 300 python bench.py --config ${CFG:-2} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-k1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done
done
