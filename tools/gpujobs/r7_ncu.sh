# K1 capture on the committed code (after the lane spread): ncu --set full of every K1 launch of c4 window 20, DRAM traffic table, details
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o /tmp/R7_k1 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/R7_iterprof.log 2>&1
python tools/ncu_traffic.py /tmp/R7_k1.ncu-rep gpurun_out/R7_iterprof.log gpurun_out/R7_k1_traffic.json --md gpurun_out/R7_k1_traffic.md > gpurun_out/R7_traffic.out 2>&1
ncu -i /tmp/R7_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/R7_k1_details.csv
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/R7_c4_iters.json 2>&1
ls -la gpurun_out/R7_*
