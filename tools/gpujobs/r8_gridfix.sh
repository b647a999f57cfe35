# the spread's grid enlargement only where k > 0 (large worklists keep their tile-sized grid): A/B against the build that launched n/128 blocks always, then the full evidence on the fixed code
for r in 1 2 3; do
  for v in build_variants/base.so paper_cs_0405053_b200/libising_sr.so; do
    ISING_SR_LIB=$v python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gf_$r.json 2> gpurun_out/gf.err
    python -c "import json;d=json.loads([l for l in open('gpurun_out/gf_$r.json') if l.startswith('{')][-1]);print('$v', $r, 'VALUE %.4e ms %.3f' % (d['value'], d['ms_per_step']))"
  done
done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/R8_bench.json 2> gpurun_out/R8_bench.err; tail -c 300 gpurun_out/R8_bench.json
timeout 3000 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/R8_tests.log 2>&1; tail -3 gpurun_out/R8_tests.log
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/R8_configs.jsonl > gpurun_out/R8_configs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/R8_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/R8_launches.csv --md gpurun_out/R8_launches.md
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/R8_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/R8_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/R8_k1.ncu-rep gpurun_out/R8_iterprof.log gpurun_out/R8_k1_traffic.json --md gpurun_out/R8_k1_traffic.md > gpurun_out/R8_traffic.out 2>&1
ncu -i /tmp/R8_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/R8_k1_details.csv
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/R8_c4_iters.json 2>&1
