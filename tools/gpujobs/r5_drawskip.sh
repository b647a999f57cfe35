# ISR_DRAWSKIP: no redraw after a break point in spread (small-worklist) blocks; then the bounds-checked build through the GPU tests (with the new spread test)
ISING_SR_LIB=build_variants/drawskip.so python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or geometries or schedules or spread or tie_mode" > gpurun_out/ds_tests.log 2>&1; tail -1 gpurun_out/ds_tests.log
for r in 1 2; do
  for v in base drawskip; do
    ISING_SR_LIB=build_variants/$v.so python tools/sweep.py --configs c1,c2 --oracle --out gpurun_out/ds_c12_${v}_$r.jsonl > /dev/null 2>&1
    ISING_SR_LIB=build_variants/$v.so python tools/sweep.py --c5 --only T1.0_W1.0 --golden --out gpurun_out/ds_c5_${v}_$r.jsonl > /dev/null 2>&1
    ISING_SR_LIB=build_variants/$v.so python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ds_c4_${v}_$r.json 2> gpurun_out/ds_c4_${v}_$r.err
    python -c "
import json
for f in ('gpurun_out/ds_c12_${v}_$r.jsonl', 'gpurun_out/ds_c5_${v}_$r.jsonl'):
    for l in open(f):
        d = json.loads(l); print('$v', $r, d['config'], '%.4e' % d['events_per_s'], 'golden', d.get('parity_golden'), 'oracle', d.get('parity_bit_exact'))
d = json.load(open('gpurun_out/ds_c4_${v}_$r.json')); print('$v', $r, 'c4', '%.4e' % d['value'], d['ms_per_step'])"
  done
done
ISING_SR_LIB=build_variants/checked.so timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py tests/test_gpu_shards.py -q -x -k "not across_a_window_boundary" > gpurun_out/r05_checked_build_tests.log 2>&1
tail -3 gpurun_out/r05_checked_build_tests.log
