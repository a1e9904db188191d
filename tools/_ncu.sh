timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'seg_kernel<\(int\)3, \(int\)2' --launch-skip 1 -c 1 -f -o gpurun_out/greedy_v2_r1b python tools/diag_segments.py --config 3 --only 7 > gpurun_out/ncu_g.log 2>&1
tail -2 gpurun_out/ncu_g.log
ls -la gpurun_out/*.ncu-rep
