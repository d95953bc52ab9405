#!/bin/bash
# A/B of the whitening periodogram (and K1) across library variants: LIBS="a.so b.so" bash tools/wh_ab.sh
for rep in 1 2; do
for lib in $LIBS; do
  SASBP_LIB=$lib timeout 300 python tools/wh_bench.py
  SASBP_LIB=$lib timeout 300 python tools/k1_bench.py --config 4
done
done
