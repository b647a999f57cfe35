# launch lists (ncu, per-kernel durations) of c4 through the strip exchange to itself, both transports
for x in peer sendrecv; do
ISING_SR_EXCHANGE=$x timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xncu_$x.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --halo-loopback > gpurun_out/xncu_$x.log 2>&1
echo "$x rc=$?"
done
