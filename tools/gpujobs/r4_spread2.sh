# spread cap (threads = 148 x 64 x CAP): c3 and c5 32x32 points with golden parity
for r in 1 2; do
  for cap in 2 4 7 14 28; do
    ISING_SR_BIG_SPREAD_CAP=$cap python tools/sweep.py --configs c3 --golden --out gpurun_out/sq_c3_${cap}_$r.jsonl > /dev/null 2>&1
    ISING_SR_BIG_SPREAD_CAP=$cap python tools/sweep.py --c5 --only b32_T4.0_W0.25 --golden --out gpurun_out/sq_c5_${cap}_$r.jsonl > /dev/null 2>&1
    python -c "
import json
for f in ('gpurun_out/sq_c3_${cap}_$r.jsonl', 'gpurun_out/sq_c5_${cap}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('cap $cap', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'))"
  done
done
