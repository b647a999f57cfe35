# final code: the bounds-checked build through the GPU parity / feature / exchange / strip tests, bench variants
ISING_SR_LIB=build_variants/checked.so timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py tests/test_gpu_shards.py -q -x > gpurun_out/r05_checked_build_tests.log 2>&1
tail -3 gpurun_out/r05_checked_build_tests.log
python bench.py --torch-alloc --no-cpu-baseline > gpurun_out/r05_bench_c4_torch_alloc.json 2> gpurun_out/r05_bench_ta.err
python bench.py --no-cpu-baseline > gpurun_out/r05_bench_c4_b.json 2> gpurun_out/r05_bench_b.err
python bench.py --halo-loopback --no-cpu-baseline --no-e2e > gpurun_out/r05_bench_c4_loopback_peer.json 2> gpurun_out/r05_bench_lp.err
ISING_SR_EXCHANGE=sendrecv python bench.py --halo-loopback --no-cpu-baseline --no-e2e > gpurun_out/r05_bench_c4_loopback_sendrecv.json 2> gpurun_out/r05_bench_ls.err
python bench.py --window tmax --no-cpu-baseline --no-e2e --steps 33 > gpurun_out/r05_bench_c4_tmax.json 2> gpurun_out/r05_bench_tm.err
python tools/gscaling.py --out gpurun_out/r05_g_vs_lnN.jsonl > gpurun_out/r05_g_vs_lnN.log 2>&1
for f in gpurun_out/r05_bench_c4_*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', '%.4e'%d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), d['parity'].get('bit_exact'))"; done
