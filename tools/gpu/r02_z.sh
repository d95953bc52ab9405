# round 2, call z: 2D dense kernel (config 2) compile variants of k2_2d.cu only -- a0 = production, a = lazy channel range,
# f = tail split / grid-constant params / host kph / cursor transform all off (126 registers like round 1),
# g = indexed transform only, h = no tail split + indexed transform (126 registers), i = no grid-constant + device kph + indexed
set -x
mkdir -p gpurun_out
timeout 1800 python tools/abi_time.py --libs build_ab3/a0.so build_ab3/a.so build_ab3/f.so build_ab3/g.so build_ab3/h.so build_ab3/i.so --configs 2:250 --reps 3 > gpurun_out/ab_z.txt 2>&1
echo done
