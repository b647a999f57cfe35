# baseline bench + one K1 launch (c4 window 20, iteration 2) captured with source for SASS-level counts
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1 || { tail -30 gpurun_out/s_build.log; exit 1; }
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
python -c "import json;d=json.load(open('gpurun_out/s_bench.json'));print('VALUE',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'])"
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'^region_kernel$' -c 1 -o gpurun_out/k1_it2 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/s_iterprof.log 2> gpurun_out/s_ncu.err
ls -la gpurun_out/
