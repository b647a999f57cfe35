# full GPU suite + smoke on the current code
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full_smoke.log 2>&1; tail -1 gpurun_out/full_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/full_tests.log 2>&1; tail -25 gpurun_out/full_tests.log
