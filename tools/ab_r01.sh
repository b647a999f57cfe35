python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  ISING_SR_LIB=build_variants/u2.so $B > gpurun_out/ab_u2_$rep.json 2>/dev/null
  ISING_SR_BATCH=1 ISING_SR_LIB=build_variants/pp00.so $B > gpurun_out/ab_pp00b1_$rep.json 2>/dev/null
  ISING_SR_LIB=build_variants/pp00.so $B > gpurun_out/ab_pp00b4_$rep.json 2>/dev/null
  ISING_SR_BATCH=1 $B > gpurun_out/ab_defb1_$rep.json 2>/dev/null
done
ISING_SR_LIB=build_variants/pp00.so timeout 600 python tools/iter_profile.py --skip 20 --windows 1 > gpurun_out/iter_pp00.json 2>&1
ISING_SR_LIB=build_variants/u2.so timeout 600 python tools/iter_profile.py --skip 20 --windows 1 > gpurun_out/iter_u2.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel_w -c 2 -o gpurun_out/k1warp -f python tools/prof_warp.py --skip 2 --windows 1 > gpurun_out/ncu_warp.log 2>&1
