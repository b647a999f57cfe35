python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/var_default.json 2> gpurun_out/var_default.err
ISING_SR_BATCH=1 $B > gpurun_out/var_b1.json 2> gpurun_out/var_b1.err
ISING_SR_BATCH=8 $B > gpurun_out/var_b8.json 2> gpurun_out/var_b8.err
for v in pp00 pp01 pp10 pp11m5 pp11ci2; do
  ISING_SR_LIB=build_variants/$v.so $B > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
for r in 20 28; do
  ISING_SR_REFILL=$r $B > gpurun_out/var_r$r.json 2>/dev/null
done
