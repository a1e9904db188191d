set -u
mkdir -p gpurun_out/r1f
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1f/pytest_gpu.txt 2>&1; tail -2 gpurun_out/r1f/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f/smoke.txt 2>&1; tail -1 gpurun_out/r1f/smoke.txt
timeout 600 python bench.py > gpurun_out/r1f/bench_cfg3.json 2> gpurun_out/r1f/bench_cfg3.err; echo "bench3 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r1f/bench_cfg3_reference.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/r1f/bench_cfg4.json 2>&1; echo "bench4 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r1f/bench_cfg2.json 2>&1; echo "bench2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1f/launches_cfg3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1f/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'seg_kernel<\(int\)3, \(int\)2' --launch-skip 1 -c 1 -f -o gpurun_out/r1f/greedy_v2 python tools/diag_segments.py --config 3 --only 7 > gpurun_out/r1f/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'seg_kernel<\(int\)2, \(int\)2' --launch-skip 1 -c 1 -f -o gpurun_out/r1f/zb_v2 python tools/diag_segments.py --config 3 --only 6 > gpurun_out/r1f/ncu_full_zb.log 2>&1; echo "ncu zb rc=$?"
