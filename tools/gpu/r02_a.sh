set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputest_r02_a.txt
timeout 900 python bench.py > gpurun_out/bench_r02_a.json 2> gpurun_out/bench_r02_a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02_a.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdbp -s 1 -c 1 -o gpurun_out/ncu_cfg4_r02 python tools/prof_tdbp.py --config 4 --pings 64 --random --forms 2 > gpurun_out/ncu_cfg4.log 2>&1
echo done
