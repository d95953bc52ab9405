# round 2, call mm: 3D kernels with 16 voxels per thread (16x8x16 tiles) at 2 CTAs/SM -- full GPU suite, default bench
# (config 4), the config-4 plan, launch list
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gputest_mm.txt
python -c "
import sys; sys.path.insert(0,'.')
import synth, torch, paper_2101_05888_b200 as pkg
s = synth.scenario(4)
bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid)
e = torch.zeros((4, s.E, s.Ns), dtype=torch.complex64, device='cuda')
bp.set_pings_device(e, s.tx[:4], s.rx[:4], s.t0[:4])
img = torch.empty(bp.shape, dtype=torch.complex64, device='cuda'); bp.form_device(img); torch.cuda.synchronize()
print(bp.plan())" > gpurun_out/plan_mm.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_mm.json 2> gpurun_out/bench_mm.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_mm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-next4 > gpurun_out/bench_ncu_mm.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_mm.txt 2>&1
echo done
