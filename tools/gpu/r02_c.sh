# round 2, call c: full GPU suite, gated A/B (split / prefetch), scaling prediction, K1 cfg4 ncu, bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/gputest_c.txt
CFG=2 timeout 1500 bash tools/ab_gated.sh > gpurun_out/ab_gated_c.txt 2>&1
timeout 1200 python tools/predict_scaling.py --configs 4,2 --ns 2,4,8 > gpurun_out/scaling_pred_c.jsonl 2> gpurun_out/scaling_pred_c.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_fft -s 5 -c 1 -o gpurun_out/ncu_k1_cfg4_r02 python tools/k1_bench.py --config 4 --reps 5 > gpurun_out/ncu_k1.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
echo done
