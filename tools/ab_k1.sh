#!/bin/bash
for rep in 1 2; do for lib in build_ab/*.so; do SASBP_LIB=$lib python tools/k1_bench.py; done; done
