python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sweep.py --c5 --window tmax --golden --out gpurun_out/r02_c5_tmax.jsonl --csv gpurun_out/r02_c5_tmax.csv > /dev/null 2>gpurun_out/r02_c5_tmax.err
python tools/gscaling.py --out gpurun_out/r02_g_vs_lnN.jsonl --b 4 > /dev/null 2>&1
python tools/gscaling.py --out gpurun_out/r02_g_vs_lnN.jsonl --b 8 --L 128,256,512,1024,2048,4096,8192,16384 > /dev/null 2>&1
python tools/iter_profile.py --skip 20 --windows 2 > gpurun_out/r02_c4_iters.json 2>&1
wc -l gpurun_out/r02_c5_tmax.jsonl gpurun_out/r02_g_vs_lnN.jsonl
