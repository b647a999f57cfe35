python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "warp_form or c3 or c5 or spanning or schedules or fresh or checkpoint" > gpurun_out/gputests_res.log 2>&1
rm -f gpurun_out/res_on.jsonl gpurun_out/res_off.jsonl
for p in b32_T4.0_W1.0 b32_T2.269_W0.25 b32_T1.0_W4.0; do
  timeout 600 python tools/sweep.py --c5 --only $p --out gpurun_out/res_on.jsonl > /dev/null 2>&1
  ISING_SR_RESUME=0 timeout 600 python tools/sweep.py --c5 --only $p --out gpurun_out/res_off.jsonl > /dev/null 2>&1
done
timeout 300 python tools/sweep.py --configs c3 --out gpurun_out/res_on.jsonl > /dev/null 2>&1
ISING_SR_RESUME=0 timeout 300 python tools/sweep.py --configs c3 --out gpurun_out/res_off.jsonl > /dev/null 2>&1
