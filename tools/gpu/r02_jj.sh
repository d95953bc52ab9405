# round 2, call jj: last check of the committed library -- full GPU suite + smoke
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gputest_jj.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_jj.txt 2>&1
echo done
