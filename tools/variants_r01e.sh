python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/ve_default.json 2> gpurun_out/ve_default.err
for v in sa0 m5 sa0m5; do
  ISING_SR_LIB=build_variants/$v.so $B > gpurun_out/ve_$v.json 2> gpurun_out/ve_$v.err
done
ISING_SR_TAIL_BATCH=1 $B > gpurun_out/ve_notail.json 2> /dev/null
rm -f gpurun_out/ve_b8.jsonl
for v in default sa0 m5 sa0m5; do
  if [ $v = default ]; then L=""; else L="ISING_SR_LIB=build_variants/$v.so"; fi
  env $L timeout 300 python tools/sweep.py --c5 --only b8_T2.269_W1.0 --out gpurun_out/ve_b8_$v.jsonl > /dev/null 2>&1
  env $L timeout 300 python tools/sweep.py --c5 --only b1_T1.0_W4.0 --out gpurun_out/ve_b8_$v.jsonl > /dev/null 2>&1
done
