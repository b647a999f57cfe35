# A/B of env settings on the default library: ENVS="A=1 B=2" (one per run), interleaved, two rounds
for r in 1 2; do
  for e in $ENVS; do
    env $e python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abe_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abe_$r.json'));print('$e', $r, 'VALUE %.4e ms %.2f' % (d['value'], d['ms_per_step']))"
  done
done
