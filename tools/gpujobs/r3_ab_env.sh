# interleaved A/B of "variant:ENV=VAL" specs (ENV part optional), c4 bench 20 windows
# usage: SPECS="pk6 pk6:ISING_SR_REFILL=24" bash tools/gpujobs/r3_ab_env.sh
for r in 1 2; do
  for sp in $SPECS; do
    v=${sp%%:*}; e=""; [ "$sp" != "$v" ] && e=${sp#*:}
    tag=$(echo "$sp" | tr ':=' '__')
    env $e ISING_SR_LIB=build_variants/$v.so python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline ${BENCHARGS:-} > gpurun_out/abe_${tag}_$r.json 2> gpurun_out/abe_${tag}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/abe_${tag}_$r.json'));print('$sp', $r, 'VALUE %.4e ms %.2f frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))" 2>&1 | tail -1
  done
done
