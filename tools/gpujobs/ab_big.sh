# big-region kernel A/B: c3 (full, golden parity) and c5 32x32 T=4 W=4 (1 window) per variant
for v in big_old big_new; do
  for pc in 1 0; do
    ISING_SR_LIB=build_variants/$v.so ISING_SR_PCACHE=$pc python tools/sweep.py --configs c3 --golden --out /tmp/c3_$v_$pc.jsonl 2>/dev/null | python -c "import json,sys;[print('$v pcache=$pc', r['config'], 'ev/s %.4e'%r['events_per_s'], 'parity', r.get('parity_golden')) for r in map(json.loads, sys.stdin)]"
    ISING_SR_LIB=build_variants/$v.so ISING_SR_PCACHE=$pc python tools/run_point.py c5_b32_T4.0_W4.0 --windows 1 | sed "s/^/$v pcache=$pc c5b32W4 /"
    ISING_SR_LIB=build_variants/$v.so ISING_SR_PCACHE=$pc python tools/run_point.py c5_b32_T2.269_W1.0 --windows 3 | sed "s/^/$v pcache=$pc c5b32W1 /"
  done
done
