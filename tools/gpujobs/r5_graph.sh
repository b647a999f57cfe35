# the device-side window loop (ISING_SR_GRAPH=1) on the iteration-count-bound points: c1, c2 and the c5 T = 1 points of the lane kernel
for r in 1 2; do
  for gr in 0 1; do
    ISING_SR_GRAPH=$gr python tools/sweep.py --configs c1,c2 --oracle --out gpurun_out/gr_c12_${gr}_$r.jsonl > /dev/null 2>&1
    ISING_SR_GRAPH=$gr python tools/sweep.py --c5 --only T1.0_W --golden --out gpurun_out/gr_c5_${gr}_$r.jsonl > /dev/null 2>&1
    python -c "
import json
for f in ('gpurun_out/gr_c12_${gr}_$r.jsonl', 'gpurun_out/gr_c5_${gr}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('graph $gr', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'), 'oracle', d.get('parity_bit_exact'))"
  done
done
