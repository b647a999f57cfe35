for r in 1 2; do
for v in ${VARIANTS:-big_old pc_only big_new}; do
    ISING_SR_LIB=build_variants/$v.so python tools/sweep.py --configs c3 --out /tmp/c3_$v.jsonl 2>/dev/null | python -c "import json,sys;[print('$v', r['config'], 'ev/s %.4e'%r['events_per_s']) for r in map(json.loads, sys.stdin)]"
    ISING_SR_LIB=build_variants/$v.so python tools/run_point.py c5_b32_T4.0_W4.0 --windows 1 | sed "s/^/$v c5b32W4 /"
    ISING_SR_LIB=build_variants/$v.so python tools/run_point.py c5_b32_T2.269_W0.25 --windows 8 | tail -1 | sed "s/^/$v c5b32W025 /"
done
done
