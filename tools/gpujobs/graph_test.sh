python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ISING_SR_GRAPH=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py -q -x -k "c1 or geometries or window_invariance or capacity or diverged or determinism or warp_form or spanning or observables_against or log_compaction or tie_mode or glauber or loopback_bit_exact or magnetisation_moments_against or jacobi or stats_active" > gpurun_out/graph_tests.log 2>&1; tail -15 gpurun_out/graph_tests.log
for r in 1 2; do
for gr in 0 1; do
  ISING_SR_GRAPH=$gr python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gb.json 2>gpurun_out/gb.err
  python -c "import json;d=json.load(open('gpurun_out/gb.json'));print('graph=$gr', $r, 'VALUE %.4e ms %.2f share %.3f k1ms %.3f' % (d['value'], d['ms_per_step'], d['roofline']['share_of_step'], d['roofline']['ms_per_launch']))" || tail -3 gpurun_out/gb.err
done
done
