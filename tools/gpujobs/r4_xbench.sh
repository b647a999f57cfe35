# c4 (20 windows) without strips, and one strip through the exchange to itself with each transport: the per-iteration exchange cost
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 1 2; do
python bench.py $B > gpurun_out/xb_none_$r.json 2> gpurun_out/xb_none_$r.err
ISING_SR_EXCHANGE=peer python bench.py $B --halo-loopback > gpurun_out/xb_peer_$r.json 2> gpurun_out/xb_peer_$r.err
ISING_SR_EXCHANGE=sendrecv python bench.py $B --halo-loopback > gpurun_out/xb_sr_$r.json 2> gpurun_out/xb_sr_$r.err
ISING_SR_EXCHANGE=peer ISING_SR_GRAPH=1 python bench.py $B --halo-loopback > gpurun_out/xb_peergraph_$r.json 2> gpurun_out/xb_peergraph_$r.err
done
for f in gpurun_out/xb_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', 'VALUE %.4e ms %.3f g %.2f exch %s' % (d['value'], d['ms_per_step'], d['iterations_per_window']['mean'], d['config'].get('exchange')))" 2>&1 | tail -1; done
