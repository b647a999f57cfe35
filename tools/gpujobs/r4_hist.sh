# K1 time by worklist size: c3 and two c5 32x32 points (where the big-region kernel spends its time)
python tools/iter_hist.py --config c3 > gpurun_out/h_c3.json 2> gpurun_out/h_c3.err; cat gpurun_out/h_c3.json; tail -2 gpurun_out/h_c3.err
python tools/iter_hist.py --config c5 --b 32 --T 4.0 --W 4.0 > gpurun_out/h_c5a.json 2> gpurun_out/h_c5a.err; cat gpurun_out/h_c5a.json; tail -2 gpurun_out/h_c5a.err
python tools/iter_hist.py --config c5 --b 32 --T 2.269 --W 1.0 > gpurun_out/h_c5b.json 2> gpurun_out/h_c5b.err; cat gpurun_out/h_c5b.json; tail -2 gpurun_out/h_c5b.err
