# round 2, call nn: 16-voxel 3D kernels with the gate masks sized to the thread's pixels -- full GPU suite + smoke
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gputest_nn.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_nn.txt 2>&1
echo done
