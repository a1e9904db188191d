# last check of the final tree as committed: GPU tests + smoke + the default bench line
set -u
D=gpurun_out/r2am; mkdir -p $D
timeout 2700 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -2 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 1500 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo "bench rc=$?"
