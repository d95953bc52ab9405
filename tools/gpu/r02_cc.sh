# round 2, call cc: evidence on the final round-2 code -- full GPU suite, default bench (config 4), launch list, K0 ncu
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gputest_cc.txt
timeout 900 python bench.py > gpurun_out/bench_cc.json 2> gpurun_out/bench_cc.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cc.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_cc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:baseband_ctap -s 2 -c 1 -o gpurun_out/ncu_k0_cc python tools/k0_bench.py --config 4 --reps 3 > gpurun_out/ncu_k0_cc.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_cc.txt 2>&1
echo done
