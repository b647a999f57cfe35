python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sweep.py --c5 --golden --out gpurun_out/r02_c5_sweep_final.jsonl --csv gpurun_out/r02_c5_sweep_final.csv > /dev/null 2>&1
python tools/sweep.py --c5 --window tmax --golden --max-iterations 20000 --out gpurun_out/r02_c5_tmax_final.jsonl --csv gpurun_out/r02_c5_tmax_final.csv > /dev/null 2>&1
python tools/sweep.py --configs c1,c2,c3 --golden --oracle --out gpurun_out/r02_configs_final.jsonl > /dev/null 2>&1
wc -l gpurun_out/r02_*final.jsonl
