# PLAIN K1 + descriptors with strip ghost rows: strip/exchange tests, a parity subset, then c4 with and without the loopback strip
timeout 1200 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_shards.py tests/test_gpu_dist_ranks.py -q -x > gpurun_out/pg_tests.log 2>&1; echo "strip tests rc=$?"; tail -3 gpurun_out/pg_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -q -x -k "c1 or geometries or window_invariance or capacity or schedules or log_compaction or tie_mode" > gpurun_out/pg_par.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pg_par.log
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 1 2; do
python bench.py $B > gpurun_out/pg_none_$r.json 2>/dev/null
ISING_SR_EXCHANGE=peer python bench.py $B --halo-loopback > gpurun_out/pg_peer_$r.json 2>/dev/null
done
for f in gpurun_out/pg_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', 'VALUE %.4e ms %.3f g %.2f kms %.3f' % (d['value'], d['ms_per_step'], d['iterations_per_window']['mean'], d['roofline']['ms_per_launch']))"; done
