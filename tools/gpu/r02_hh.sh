# round 2, call hh: ncu --set full of the final K2 3D kernel (64-ping slice of the full config-4 grid) + smoke of the final lib
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_hh.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tdbp -s 1 -c 1 -o gpurun_out/ncu_k2_hh python tools/prof_tdbp.py --config 4 --pings 64 --random --forms 2 > gpurun_out/ncu_k2_hh.log 2>&1
echo done
