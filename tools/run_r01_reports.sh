python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_default.json 2> gpurun_out/var_default.err
rm -f gpurun_out/r01_configs.jsonl gpurun_out/r01_c5_sweep.jsonl
timeout 900 python tools/sweep.py --configs c1,c2,c3 --oracle --out gpurun_out/r01_configs.jsonl > gpurun_out/sweep_cfg.log 2>&1
timeout 1500 python tools/sweep.py --c5 --out gpurun_out/r01_c5_sweep.jsonl --csv gpurun_out/r01_c5_sweep.csv > gpurun_out/sweep_c5.log 2>&1
