# round 2, call aa: 2D plane kernels with the round-1 register allocation (k2_2d.cu knob settings): full GPU suite,
# same-box A/B vs the previous production build, config-2 bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gputest_aa.txt
timeout 1800 python tools/abi_time.py --libs build_ab3/a0.so paper_2101_05888_b200/libsasbp.so --configs 2:250 4:100 --reps 3 > gpurun_out/ab_aa.txt 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2_aa.json 2> gpurun_out/bench_cfg2_aa.err
echo done
