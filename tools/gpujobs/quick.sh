# quick check: build, a parity subset, the c4 bench (20 windows)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1 || { tail -30 gpurun_out/q_build.log; exit 1; }
python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py -q -x -k "${QK:-c1 or geometries or window_invariance or capacity or warp_form or schedules or log_compaction or tie_mode or loopback_bit_exact}" > gpurun_out/q_tests.log 2>&1
tail -3 gpurun_out/q_tests.log
python bench.py --steps ${QSTEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline ${QBENCH:-} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'A',d['per_region_per_window']['A_recomputations'],'frac',d['roofline']['frac'],'win',d['roofline']['window']['frac'],'compact',d['commit_compaction_ms_per_window'])"
