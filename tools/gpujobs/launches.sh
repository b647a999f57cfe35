# bench (with and without digests) + the ncu launch list of the bench command
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l_bench.json 2>/dev/null
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --digest > gpurun_out/l_bench_dig.json 2>/dev/null
for f in l_bench l_bench_dig; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f VALUE %.4e ms %.2f compact %.3f' % (d['value'], d['ms_per_step'], d['commit_compaction_ms_per_window']))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_launches_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r2_launches.csv
