# big-region K1: small worklists spread to one region per 2^k lanes (ISING_SR_BIG_SPREAD = max k; 0 = off), c3 and c5 32x32 points with golden parity
for r in 1 2; do
  for sp in 0 5 3; do
    ISING_SR_BIG_SPREAD=$sp python tools/sweep.py --configs c3 --golden --out gpurun_out/sp_c3_${sp}_$r.jsonl > /dev/null 2>&1
    ISING_SR_BIG_SPREAD=$sp python tools/sweep.py --c5 --only b32_T2.269_W1.0 --golden --out gpurun_out/sp_c5_${sp}_$r.jsonl > /dev/null 2>&1
    python -c "
import json
for f in ('gpurun_out/sp_c3_${sp}_$r.jsonl', 'gpurun_out/sp_c5_${sp}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('spread $sp', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'))"
  done
done
