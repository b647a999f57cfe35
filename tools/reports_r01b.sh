python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
rm -f gpurun_out/r01b_configs.jsonl gpurun_out/r01b_c5_sweep.jsonl
timeout 900 python tools/sweep.py --configs c1,c2,c3 --oracle --out gpurun_out/r01b_configs.jsonl > gpurun_out/sweep_cfg.log 2>&1
timeout 2400 python tools/sweep.py --c5 --out gpurun_out/r01b_c5_sweep.jsonl --csv gpurun_out/r01b_c5_sweep.csv > gpurun_out/sweep_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o gpurun_out/k1_window20 -f python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/ncu_k1w20.log 2>&1
