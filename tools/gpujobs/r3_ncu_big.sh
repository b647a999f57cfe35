# ncu (with source) of the big-region K1: c3 window 60, the window's 3rd launch (iteration 3)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'region_kernel_big' -s 2 -c 1 -o gpurun_out/k1big_c3 python tools/iter_profile.py --config c3 --skip 60 --windows 1 --profile > gpurun_out/nb_iterprof.log 2> gpurun_out/nb_ncu.err
ls -la gpurun_out/k1big_c3*
