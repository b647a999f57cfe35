# big-region variants: c3 and the c5 32x32 points (golden parity), interleaved
for r in 1 2; do
  for v in $VARIANTS; do
    ISING_SR_LIB=build_variants/$v.so python tools/sweep.py --configs c3 --golden --out gpurun_out/abb_c3_${v}_$r.jsonl > /dev/null 2>&1
    ISING_SR_LIB=build_variants/$v.so python tools/sweep.py --c5 --only ${ONLY:-b32_T4.0_W1.0} --golden --out gpurun_out/abb_c5_${v}_$r.jsonl > /dev/null 2>&1
    python -c "
import json
for f in ('gpurun_out/abb_c3_${v}_$r.jsonl', 'gpurun_out/abb_c5_${v}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('$v', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'))"
  done
done
