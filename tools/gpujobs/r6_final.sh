# the code as committed at the end of round 2: smoke, the full GPU suite, the default bench line, c1-c3 with oracle parity, launch list
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/R6_smoke.log 2>&1; tail -1 gpurun_out/R6_smoke.log
python bench.py > gpurun_out/R6_bench.json 2> gpurun_out/R6_bench.err; tail -1 gpurun_out/R6_bench.json | cut -c1-200
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/R6_tests.log 2>&1; tail -3 gpurun_out/R6_tests.log
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/R6_configs.jsonl > gpurun_out/R6_configs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/R6_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/R6_launches.csv --md gpurun_out/R6_launches.md
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/R6_bench_ref.json 2> gpurun_out/R6_bench_ref.err
