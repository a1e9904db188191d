set -u
D=gpurun_out/r2a; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt 2>&1
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -3 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > $D/bench_cfg3.json 2> $D/bench_cfg3.err; echo "bench3 rc=$?"
