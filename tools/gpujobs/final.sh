# round-2 final evidence: smoke, the full GPU suite, the bench lines, launch list, K1 traffic capture
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/F_smoke.log 2>&1; tail -1 gpurun_out/F_smoke.log
python -m pytest tests -m gpu -q --durations=30 > gpurun_out/F_tests.log 2>&1; tail -3 gpurun_out/F_tests.log
python bench.py > gpurun_out/F_bench.json 2> gpurun_out/F_bench.err
python bench.py --config cb > gpurun_out/F_bench_cb.json 2> gpurun_out/F_bench_cb.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/F_bench_ref.json 2> gpurun_out/F_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/F_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/F_launches.csv --md gpurun_out/F_launches.md
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/F_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/F_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/F_k1.ncu-rep gpurun_out/F_iterprof.log gpurun_out/F_k1_traffic.json --md gpurun_out/F_k1_traffic.md > /dev/null 2>&1
ncu -i /tmp/F_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/F_k1_details.csv
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/F_c4_iters.json 2>&1
ls -la gpurun_out/F_*
