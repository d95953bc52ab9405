# round 2, call s: final evidence on the round-2 code -- full GPU suite, default bench (config 4), launch list,
# K2 config-4 full-launch DRAM bytes, K1 (final rc_pipe kernel) ncu, all-config dense + gated table
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gputest_s.txt
timeout 900 python bench.py > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_s.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_s.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tdbp -s 1 -c 1 --csv --log-file gpurun_out/k2_cfg4_dram_s.csv python tools/prof_tdbp.py --config 4 --random --forms 2 > gpurun_out/k2dram_s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_pipe -s 2 -c 1 -o gpurun_out/ncu_k1_s python tools/k1_bench.py --config 4 --reps 3 > gpurun_out/ncu_k1_s.log 2>&1
timeout 1500 python tools/bench_configs.py --configs 2 3 4 5 --gated > gpurun_out/configs_s.jsonl 2> gpurun_out/configs_s.err
echo done
