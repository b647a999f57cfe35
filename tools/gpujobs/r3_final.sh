# round-2 (late session) final evidence on the current code: bench lines, launch list, K1 capture + traffic, sweeps with golden parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py > gpurun_out/G_bench.json 2> gpurun_out/G_bench.err
python bench.py --config cb > gpurun_out/G_bench_cb.json 2> gpurun_out/G_bench_cb.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/G_bench_ref.json 2> gpurun_out/G_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/G_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/G_launches.csv --md gpurun_out/G_launches.md
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/G_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/G_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/G_k1.ncu-rep gpurun_out/G_iterprof.log gpurun_out/G_k1_traffic.json --md gpurun_out/G_k1_traffic.md > gpurun_out/G_traffic.out 2>&1
ncu -i /tmp/G_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/G_k1_details.csv
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/G_c4_iters.json 2>&1
ls -la gpurun_out/G_*
python tools/sweep.py --c5 --golden --out gpurun_out/r03_c5_sweep.jsonl --csv gpurun_out/r03_c5_sweep.csv > gpurun_out/r03_c5_sweep.log 2>&1
python tools/sweep.py --c5 --window tmax --golden --max-iterations 20000 --out gpurun_out/r03_c5_tmax.jsonl --csv gpurun_out/r03_c5_tmax.csv > gpurun_out/r03_c5_tmax.log 2>&1
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/r03_configs.jsonl > gpurun_out/r03_configs.log 2>&1
wc -l gpurun_out/r03_*.jsonl
