# round 2, call l: K1 pipelined variants (a: 2 staging buffers 2 CTAs/SM, b: 1 buffer 3 CTAs/SM,
# c: 1 buffer + ping-pong exchange (4 barriers) 2 CTAs/SM, d: 1 buffer 2 CTAs/SM)
set -x
mkdir -p gpurun_out
for l in c b; do SASBP_LIB=build_ab/k1_$l.so timeout 600 python -m pytest tests -m gpu -x -q -k "rangecompress or whiten" 2>&1 | tail -2; done > gpurun_out/t_l.txt
for rep in 1 2 3; do for c in 4 2; do for l in a b c d; do SASBP_LIB=build_ab/k1_$l.so timeout 300 python tools/k1_bench.py --config $c; done; done; done > gpurun_out/k1_l.txt 2>&1
echo done
