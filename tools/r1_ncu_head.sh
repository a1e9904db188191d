# ncu --set full of cfg3 GREEDY v = 2 (2 M candidates) on the current code
mkdir -p gpurun_out/r1hn
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'seg_kernel<\(int\)3, \(int\)2' --launch-skip 1 -c 1 -f -o gpurun_out/r1hn/greedy_v2 python tools/diag_segments.py --config 3 --only 7 > gpurun_out/r1hn/ncu_full.log 2>&1; echo "ncu full rc=$?"
