# round 2, call ff: nav-table tests incl. streamed / cp.async paths
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "nav" 2>&1 | tail -4 > gpurun_out/t_ff.txt
echo done
