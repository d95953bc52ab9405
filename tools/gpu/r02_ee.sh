# round 2, call ee: final verification of the committed code -- full GPU suite, smoke, default bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gputest_ee.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ee.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_ee.json 2> gpurun_out/bench_ee.err
echo done
