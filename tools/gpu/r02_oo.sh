# round 2, call oo: final bench of the committed code, launch list, ncu --set full of the 16-voxel 3D kernel
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_oo.json 2> gpurun_out/bench_oo.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_oo.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_oo.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdbp -s 1 -c 1 -o gpurun_out/ncu_k2_oo python tools/prof_tdbp.py --config 4 --pings 64 --random --forms 2 > gpurun_out/ncu_k2_oo.log 2>&1
echo done
