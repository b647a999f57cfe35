# per-variant short bench (c4, windows 3..22) + full GPU parity on the default build
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
for v in base u1 u2; do
  ISING_SR_LIB=build_variants/$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
for r in 8 16 20 28; do
  ISING_SR_REFILL=$r timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_u2_r$r.json 2>/dev/null
done
