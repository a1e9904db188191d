# DRAM traffic of the bench's dominant launch (cfg3 GREEDY v=2 INT, full segment)
mkdir -p gpurun_out/r1t
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 1500 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'seg_kernel<\(int\)3, \(int\)2' -c 1 -f \
  -o gpurun_out/r1t/dominant python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1t/ncu.log 2>&1
echo "ncu rc=$?"
