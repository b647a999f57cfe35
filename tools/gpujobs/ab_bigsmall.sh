for mu in 1e9 8; do
  ISING_SR_LIB=build_variants/bigsmall.so ISING_SR_BIG_MU=$mu python tools/sweep.py --c5 --only _b4_ --golden --out /tmp/s_$mu.jsonl > /dev/null 2>&1
  ISING_SR_LIB=build_variants/bigsmall.so ISING_SR_BIG_MU=$mu python tools/sweep.py --c5 --only _b8_ --golden --out /tmp/s_$mu.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('/tmp/s_$mu.jsonl'):
    r=json.loads(l); print('mu=$mu', r['config'], 'ev/s %.3e'%r['events_per_s'], 'g', r['g_mean'], 'parity', r.get('parity_golden'))
"
done
