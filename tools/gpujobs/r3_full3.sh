# full GPU suite + smoke on the final code
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/K_smoke.log 2>&1; tail -1 gpurun_out/K_smoke.log
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/K_tests.log 2>&1; tail -3 gpurun_out/K_tests.log
# refill threshold per region shape (c5 points, golden parity)
for rf in 20 24 28 31; do
  ISING_SR_REFILL=$rf python tools/sweep.py --c5 --only W1.0 --golden --out gpurun_out/K_rf$rf.jsonl > /dev/null 2>&1
done
python - <<'PY'
import json
rows = {}
for rf in (20, 24, 28, 31):
    for l in open(f'gpurun_out/K_rf{rf}.jsonl'):
        d = json.loads(l)
        rows.setdefault(d['config'], {})[rf] = (d['events_per_s'], d.get('parity_golden'))
for k, v in rows.items():
    print(k, ' '.join(f'{rf}:{v[rf][0]:.3e}{"" if v[rf][1] else "!"}' for rf in sorted(v)))
PY
