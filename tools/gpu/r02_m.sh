# round 2, call m: NEXT-2 tabled trajectories (sas_bp_set_nav) parity + the motion / abi tests
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "nav or motion or abi" 2>&1 | tail -25 > gpurun_out/t_m.txt
echo done
