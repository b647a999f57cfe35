# Round profile: GPU tests, the c4 bench line, the reference arm, the K1 launch list,
# one ncu --set full capture of a whole c4 window, c1-c3 parity reports, the c5 sweep, the
# checkerboard bench line + ncu capture, the Jacobi-schedule bench line.
# Run on the GPU box: gpurun -- bash tools/profile_round.sh (outputs in gpurun_out/).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 40 -o gpurun_out/k1_window20 -f python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/ncu_k1w20.log 2>&1
rm -f gpurun_out/r01c_configs.jsonl gpurun_out/r01c_c5_sweep.jsonl
timeout 900 python tools/sweep.py --configs c1,c2,c3 --oracle --out gpurun_out/r01c_configs.jsonl > gpurun_out/sweep_cfg.log 2>&1
timeout 2400 python tools/sweep.py --c5 --out gpurun_out/r01c_c5_sweep.jsonl --csv gpurun_out/r01c_c5_sweep.csv > gpurun_out/sweep_c5.log 2>&1
timeout 600 python bench.py --config cb --steps 50 --warmup 3 > gpurun_out/bench_cb.json 2> gpurun_out/bench_cb.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:half_sweep -s 6 -c 2 -o gpurun_out/cb -f python bench.py --config cb --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cb.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --jacobi-all > gpurun_out/b_jac.json 2>&1
