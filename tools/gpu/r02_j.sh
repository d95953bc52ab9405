# round 2, call j (re-entry): GPU suite + bench + launch list on HEAD 047e8ae code
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputest_r02_j.txt
timeout 900 python bench.py > gpurun_out/bench_r02_j.json 2> gpurun_out/bench_r02_j.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02_j.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_j.log 2>&1
echo done
