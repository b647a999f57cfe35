for r in 1 2; do
for e in 0 2 4 8; do
  ISING_SR_LIB=build_variants/lpc.so ISING_SR_LPC=$e python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abl.json'));print('lpc=$e', $r, 'VALUE %.4e ms %.2f' % (d['value'], d['ms_per_step']))"
done
done
ISING_SR_LIB=build_variants/lpc.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -q -x -k "c1 or geometries or window_invariance or tie_mode or glauber or spanning or fresh or log_compaction or capacity" 2>&1 | tail -2
