python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_m.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for rep in 1 2; do
  $B > gpurun_out/vn_new_$rep.json 2>/dev/null
  ISING_SR_LIB=build_variants/prev.so $B > gpurun_out/vn_prev_$rep.json 2>/dev/null
done
rm -f gpurun_out/vn_big_new.jsonl gpurun_out/vn_big_prev.jsonl
timeout 600 python tools/sweep.py --configs c3 --c5 --only b32_T4.0_W1.0 --out gpurun_out/vn_big_new.jsonl > /dev/null 2>&1
ISING_SR_LIB=build_variants/prev.so timeout 600 python tools/sweep.py --configs c3 --c5 --only b32_T4.0_W1.0 --out gpurun_out/vn_big_prev.jsonl > /dev/null 2>&1
