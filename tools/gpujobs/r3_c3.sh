# c3 (16x16 regions): golden-checked full runs with the host loop and the device graph loop; per-iteration times of late windows
for gr in 0 1; do
  ISING_SR_GRAPH=$gr python tools/sweep.py --configs c3 --golden --out gpurun_out/c3_graph$gr.jsonl > gpurun_out/c3_graph$gr.log 2>&1
  python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/c3_graph$gr.jsonl')][-1]
print('GRAPH $gr', {k: d.get(k) for k in ('events_per_s','ms','g_mean','A','golden','bit_exact_golden','parity')})" 2>&1 | tail -2
done
python tools/iter_profile.py --config c3 --skip 60 --windows 2 > gpurun_out/c3_iters.json 2>&1
python -c "
import json
for d in json.load(open('gpurun_out/c3_iters.json')):
    print('window', d['window'], 'events', d['events'], ' '.join('%d:%d/%.3f' % (r['it'], r['regions'], r['ms']) for r in d['iters']))"
