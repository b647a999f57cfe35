# prefetch K1: parity subset, then A/B of ISING_SR_PF=1 (default) against the batched refill
python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py -q -x -k "${QK:-c1 or geometries or window_invariance or capacity or schedules or log_compaction or tie_mode or loopback_bit_exact}" > gpurun_out/pf_tests.log 2>&1
tail -5 gpurun_out/pf_tests.log
for r in 1 2; do
  for pf in 1 0; do
    ISING_SR_PF=$pf python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pf_${pf}_$r.json 2> gpurun_out/pf_${pf}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/pf_${pf}_$r.json'));print('PF $pf', $r, 'VALUE %.4e ms %.2f frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), d.get('parity'))" 2>&1 | tail -1
  done
done
