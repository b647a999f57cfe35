python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in ci2 ci2m6 m6 ci4; do
  ISING_SR_LIB=build_variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 4 -o gpurun_out/k1u2_w20 -f python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/ncu_k1.log 2>&1
