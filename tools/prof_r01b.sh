python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "warp_form or c3 or c5 or c2" > gpurun_out/gputests_w.log 2>&1
rm -f gpurun_out/sw_b32.jsonl
timeout 600 python tools/sweep.py --configs c3 --c5 --only b32_T4.0_W1.0 --out gpurun_out/sw_b32.jsonl > gpurun_out/sw_b32.log 2>&1
timeout 600 python tools/sweep.py --c5 --only b32_T2.269_W0.25 --out gpurun_out/sw_b32.jsonl >> gpurun_out/sw_b32.log 2>&1
ISING_SR_LIB=build_variants/p48.so timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 3 -o gpurun_out/k1pool_w20 -f python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/ncu_pool.log 2>&1
