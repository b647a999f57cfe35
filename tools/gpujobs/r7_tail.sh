# where a tiny-worklist iteration's time goes: kernel durations (ncu launch list) of c2 against its wall time per iteration, with and without the pipelined loop
for p in 1 0; do
  ISING_SR_PIPELINE=$p python tools/sweep.py --configs c2 --out gpurun_out/tail_c2_p$p.jsonl > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/tail_c2_p$p.jsonl').readline())
it = d['g_mean']*d['windows']; print('pipeline $p c2 events/s %.4e' % d['events_per_s'], 'device_s', d['device_s'], 'iterations', it, 'us/iteration', 1e6*d['device_s']/it)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/tail_c2_launches.csv python tools/sweep.py --configs c2 --out gpurun_out/tail_c2_ncu.jsonl > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/tail_c2_launches.csv --md gpurun_out/tail_c2_launches.md; cat gpurun_out/tail_c2_launches.md
