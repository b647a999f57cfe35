set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
python -m pytest tests/test_gpu_features.py -q -k "magnetisation" > gpurun_out/r2_gpu_tests3.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "c4_full or c5_full" --durations=10 >> gpurun_out/r2_gpu_tests3.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/r2_k1_c4_w20 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/r2_iterprof.log 2> gpurun_out/r2_ncu.err
python tools/ncu_traffic.py /tmp/r2_k1_c4_w20.ncu-rep gpurun_out/r2_iterprof.log gpurun_out/k1_traffic_r02.json --md gpurun_out/r02_k1_traffic_c4_w20.md > gpurun_out/r2_traffic.out 2>&1
ncu -i /tmp/r2_k1_c4_w20.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null; gzip -c /tmp/raw.csv > gpurun_out/r2_k1_c4_w20_raw.csv.gz
ncu -i /tmp/r2_k1_c4_w20.ncu-rep --page details --csv 2>/dev/null | gzip -c > gpurun_out/r2_k1_c4_w20_details.csv.gz
ls -la gpurun_out/
