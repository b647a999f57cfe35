python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/vf_default.json 2> gpurun_out/vf_default.err
rm -f gpurun_out/vf_b8.jsonl
timeout 300 python tools/sweep.py --c5 --only b8_T2.269_W1.0 --out gpurun_out/vf_b8.jsonl > /dev/null 2>&1
timeout 300 python tools/sweep.py --c5 --only b1_T1.0_W4.0 --out gpurun_out/vf_b8.jsonl > /dev/null 2>&1
