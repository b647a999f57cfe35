# the full GPU suite + the default bench line + smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
python -m pytest tests -m gpu -q --durations=25 > gpurun_out/f_tests.log 2>&1; tail -30 gpurun_out/f_tests.log
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; cat gpurun_out/f_bench.json
