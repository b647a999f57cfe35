# full GPU suite + smoke + the default bench line on the current code
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/H_smoke.log 2>&1; tail -1 gpurun_out/H_smoke.log
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/H_tests.log 2>&1; tail -3 gpurun_out/H_tests.log
python bench.py > gpurun_out/H_bench.json 2> gpurun_out/H_bench.err
python -c "import json;d=json.load(open('gpurun_out/H_bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac'],'parity',d.get('parity'))"
