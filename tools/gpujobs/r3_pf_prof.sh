# per-iteration K1 times of c4 window 20 with and without prefetch; ncu of the prefetch K1, iteration 2
for pf in 1 0; do
  ISING_SR_PF=$pf python tools/iter_profile.py --skip 20 --windows 1 > gpurun_out/pfit_$pf.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/pfit_$pf.json'))[0]
print('PF $pf', ' '.join('%d:%d/%.2f' % (r['it'], r['regions'], r['ms']) for r in d['iters'][:8]), 'total %.2f' % sum(r['ms'] for r in d['iters']))"
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'region_kernel_pf$' -c 1 -o gpurun_out/k1pf_it2 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/s_iterprof.log 2> gpurun_out/s_ncu.err
ls -la gpurun_out/k1pf_it2*
