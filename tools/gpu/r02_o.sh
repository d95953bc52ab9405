# round 2, call o: gated K2 A/B (config 2): h0 = zero-cell selects at 4 CTAs/SM (default), h3 = 3 CTAs/SM (no spills),
# h3s = + second pixel-loop copy without selects for IN channels, h3c = + cursor window transform, h3p = + hot-constant prefetch
set -x
mkdir -p gpurun_out
CFG=2 LIBDIR=build_abg timeout 2000 bash tools/ab_gated.sh > gpurun_out/ab_gated_o.txt 2>&1
echo done
