set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/iter_w20.json 2> gpurun_out/iter.err
python tools/iter_profile.py --skip 60 --windows 1 > gpurun_out/iter_w60.json 2>> gpurun_out/iter.err
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel -c 4 -o gpurun_out/k1_w20 -f python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/ncu_k1.log 2>&1
