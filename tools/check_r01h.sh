python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 16 20 24 28 32; do
  ISING_SR_REFILL=$r $B > gpurun_out/vh_r$r.json 2>/dev/null
done
ISING_SR_LIB=build_variants/ci2.so $B > gpurun_out/vh_ci2.json 2>/dev/null
ISING_SR_REFILL=20 ISING_SR_LIB=build_variants/ci2.so $B > gpurun_out/vh_ci2r20.json 2>/dev/null
