python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "warp_form or c3 or c5 or spanning" > gpurun_out/gputests_big.log 2>&1
rm -f gpurun_out/sw_big.jsonl
timeout 600 python tools/sweep.py --configs c3 --c5 --only b32_T4.0_W1.0 --out gpurun_out/sw_big.jsonl > gpurun_out/sw_big.log 2>&1
timeout 600 python tools/sweep.py --c5 --only b32_T2.269_W0.25 --out gpurun_out/sw_big.jsonl >> gpurun_out/sw_big.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel_big -c 2 -o gpurun_out/k1big -f python tools/prof_warp.py --skip 2 --windows 1 > gpurun_out/ncu_big.log 2>&1
