# round-2 (final session) evidence on the final code: smoke, the full GPU suite, bench lines, launch list, K1 capture + traffic, c1-c3 with oracle parity
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/R5_smoke.log 2>&1; tail -1 gpurun_out/R5_smoke.log
python bench.py > gpurun_out/R5_bench.json 2> gpurun_out/R5_bench.err; cut -c1-300 gpurun_out/R5_bench.json
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/R5_tests.log 2>&1; tail -3 gpurun_out/R5_tests.log
python bench.py --config cb > gpurun_out/R5_bench_cb.json 2> gpurun_out/R5_bench_cb.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/R5_bench_ref.json 2> gpurun_out/R5_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/R5_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/R5_launches.csv --md gpurun_out/R5_launches.md
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/R5_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/R5_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/R5_k1.ncu-rep gpurun_out/R5_iterprof.log gpurun_out/R5_k1_traffic.json --md gpurun_out/R5_k1_traffic.md > gpurun_out/R5_traffic.out 2>&1
ncu -i /tmp/R5_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/R5_k1_details.csv
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/R5_configs.jsonl > gpurun_out/R5_configs.log 2>&1
ls -la gpurun_out/R5_*
