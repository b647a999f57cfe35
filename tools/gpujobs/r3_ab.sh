# parity subset on the given variants, then interleaved A/B of bench (c4, 20 windows)
# usage: VARIANTS="a b" [TESTV="b"] bash tools/gpujobs/r3_ab.sh
for v in ${TESTV:-}; do
  ISING_SR_LIB=build_variants/$v.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py -q -x -k "${QK:-c1 or geometries or window_invariance or capacity or schedules or log_compaction or tie_mode or loopback_bit_exact}" > gpurun_out/ab_tests_$v.log 2>&1
  echo "tests $v: $(tail -1 gpurun_out/ab_tests_$v.log)"
done
for r in 1 2; do
  for v in $VARIANTS; do
    ISING_SR_LIB=build_variants/$v.so python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline ${BENCHARGS:-} > gpurun_out/ab_${v}_$r.json 2> gpurun_out/ab_${v}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$r.json'));print('$v', $r, 'VALUE %.4e ms %.2f frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))" 2>&1 | tail -1
  done
done
