# round 2, call d: GPU suite with the wave-tail split + swizzled periodogram, tail-split A/B, K2 cfg4 full-launch DRAM bytes, whitening ncu
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/gputest_d.txt
timeout 1500 python tools/ab_time.py --libs build_ab/cur.so build_ab/cur.so,SASBP_NO_TAILSPLIT=1 --configs 4:1000 2:1000 --reps 2 --forms 2 > gpurun_out/ab_tail_d.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tdbp -s 1 -c 1 --csv --log-file gpurun_out/k2_cfg4_dram.csv python tools/prof_tdbp.py --config 4 --random --forms 2 > gpurun_out/k2dram.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wh_periodogram|rc_fft" -c 2 -o gpurun_out/ncu_wh_r02 python tools/prof_cond.py > gpurun_out/ncu_wh.log 2>&1
echo done
