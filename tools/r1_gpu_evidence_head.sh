set -u
D=gpurun_out/r1h; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.txt 2>&1; tail -2 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 600 python bench.py > $D/bench_cfg3.json 2> $D/bench_cfg3.err; echo "bench3 rc=$?"
timeout 600 python bench.py --impl reference > $D/bench_cfg3_reference.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_cfg3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $D/ncu_launch.log 2>&1; echo "ncu list rc=$?"
