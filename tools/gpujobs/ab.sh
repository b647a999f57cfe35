# A/B timing of library variants in build_variants/ (interleaved, two rounds)
# usage: VARIANTS="a b c" STEPS=20 bash tools/gpujobs/ab.sh
for r in 1 2; do
  for v in $VARIANTS; do
    ISING_SR_LIB=build_variants/$v.so python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline ${BENCHARGS:-} > gpurun_out/ab_${v}_$r.json 2> gpurun_out/ab_${v}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$r.json'));print('$v', $r, 'VALUE %.4e ms %.2f share %.3f compact %.3f' % (d['value'], d['ms_per_step'], d['roofline']['share_of_step'], d['commit_compaction_ms_per_window']))"
  done
done
