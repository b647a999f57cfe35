# the committed code: the c5 sweep and the paper's T_max points with golden parity
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sweep.py --c5 --golden --out gpurun_out/r08_c5_sweep.jsonl --csv gpurun_out/r08_c5_sweep.csv > gpurun_out/r08_c5_sweep.log 2>&1
python tools/sweep.py --c5 --window tmax --golden --max-iterations 20000 --out gpurun_out/r08_c5_tmax.jsonl --csv gpurun_out/r08_c5_tmax.csv > gpurun_out/r08_c5_tmax.log 2>&1
wc -l gpurun_out/r08_*.jsonl
