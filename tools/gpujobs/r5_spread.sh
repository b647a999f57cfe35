# lane K1: small worklists spread to one region per 2^k lanes (ISING_SR_LANE_SPREAD = max k; 0 = off): parity subset, then c1/c2 (oracle), the c5 T = 1 points (golden) and c4 (20 windows), two interleaved rounds
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py tests/test_gpu_shards.py -q -x -k "not across_a_window_boundary" > gpurun_out/sp_tests.log 2>&1; tail -2 gpurun_out/sp_tests.log
for r in 1 2; do
  for sp in 0 5; do
    ISING_SR_LANE_SPREAD=$sp python tools/sweep.py --configs c1,c2 --oracle --out gpurun_out/lsp_c12_${sp}_$r.jsonl > /dev/null 2>&1
    ISING_SR_LANE_SPREAD=$sp python tools/sweep.py --c5 --only T1.0_ --golden --out gpurun_out/lsp_c5_${sp}_$r.jsonl > /dev/null 2>&1
    ISING_SR_LANE_SPREAD=$sp python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lsp_c4_${sp}_$r.json 2> gpurun_out/lsp_c4_${sp}_$r.err
    python -c "
import json
for f in ('gpurun_out/lsp_c12_${sp}_$r.jsonl', 'gpurun_out/lsp_c5_${sp}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('spread $sp', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'), 'oracle', d.get('parity_bit_exact'))
d = json.load(open('gpurun_out/lsp_c4_${sp}_$r.json')); print('spread $sp', $r, 'c4', '%.4e' % d['value'], d['ms_per_step'])"
  done
done
