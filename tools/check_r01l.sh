python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "warp_form or c3 or c5 or spanning or schedules or fresh or checkpoint" > gpurun_out/gputests_l.log 2>&1
rm -f gpurun_out/res2.jsonl
timeout 600 python tools/sweep.py --configs c3 --c5 --only b32_T4.0_W1.0 --out gpurun_out/res2.jsonl > /dev/null 2>&1
