# final evidence on the final code (PLAIN K1, descriptors, compare-select mins): bench lines, launch list, K1 capture + traffic, sweeps with golden parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py > gpurun_out/J_bench.json 2> gpurun_out/J_bench.err
python bench.py --config cb > gpurun_out/J_bench_cb.json 2> gpurun_out/J_bench_cb.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/J_bench_ref.json 2> gpurun_out/J_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/J_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/J_launches.csv --md gpurun_out/J_launches.md
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/J_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/J_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/J_k1.ncu-rep gpurun_out/J_iterprof.log gpurun_out/J_k1_traffic.json --md gpurun_out/J_k1_traffic.md > gpurun_out/J_traffic.out 2>&1
ncu -i /tmp/J_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/J_k1_details.csv
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/J_c4_iters.json 2>&1
ls -la gpurun_out/J_*
python tools/sweep.py --c5 --golden --out gpurun_out/r03b_c5_sweep.jsonl --csv gpurun_out/r03b_c5_sweep.csv > gpurun_out/r03b_c5_sweep.log 2>&1
python tools/sweep.py --c5 --window tmax --golden --max-iterations 20000 --out gpurun_out/r03b_c5_tmax.jsonl --csv gpurun_out/r03b_c5_tmax.csv > gpurun_out/r03b_c5_tmax.log 2>&1
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/r03b_configs.jsonl > gpurun_out/r03b_configs.log 2>&1
wc -l gpurun_out/r03_*.jsonl
