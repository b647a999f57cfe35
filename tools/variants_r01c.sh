python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/var_default.json 2> gpurun_out/var_default.err
ISING_SR_POOL=0 $B > gpurun_out/var_lane.json 2> gpurun_out/var_lane.err
ISING_SR_BATCH=1 $B > gpurun_out/var_b1.json 2> gpurun_out/var_b1.err
ISING_SR_BATCH=8 $B > gpurun_out/var_b8.json 2> gpurun_out/var_b8.err
for v in p48 p64ci1 p48ci3; do
  ISING_SR_LIB=build_variants/$v.so $B > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
for r in 16 48; do
  ISING_SR_POOL_REFILL=$r $B > gpurun_out/var_p64_r$r.json 2>/dev/null
done
