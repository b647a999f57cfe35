# tile order by predicted length: parity subset, then A/B against worklist order
python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py -q -x -k "${QK:-c1 or geometries or window_invariance or capacity or schedules or log_compaction or tie_mode or loopback_bit_exact}" > gpurun_out/sort_tests.log 2>&1
tail -3 gpurun_out/sort_tests.log
for r in 1 2; do
  for v in 1 0; do
    ISING_SR_SORT=$v python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sort_${v}_$r.json 2> gpurun_out/sort_${v}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/sort_${v}_$r.json'));print('SORT $v', $r, 'VALUE %.4e ms %.2f frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))" 2>&1 | tail -1
  done
done
for v in 1 0; do
  ISING_SR_SORT=$v python tools/iter_profile.py --skip 20 --windows 1 > gpurun_out/sortit_$v.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/sortit_$v.json'))[0]
print('SORT $v', ' '.join('%d:%.2f' % (r['it'], r['ms']) for r in d['iters'][:8]), 'total %.2f' % sum(r['ms'] for r in d['iters']))"
done
