# one PLAIN K1 launch (c4 window 20, iteration 2) with source, for SASS-level counts
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'^region_kernel$' -c 1 -o gpurun_out/k1p_it2 python tools/iter_profile.py --skip 20 --windows 1 --profile > gpurun_out/s2_iterprof.log 2> gpurun_out/s2_ncu.err
ls -la gpurun_out/k1p_it2*
