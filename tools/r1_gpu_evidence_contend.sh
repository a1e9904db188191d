set -u
mkdir -p gpurun_out/r1g
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1g/pytest_gpu.txt 2>&1; tail -2 gpurun_out/r1g/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g/smoke.txt 2>&1; tail -1 gpurun_out/r1g/smoke.txt
timeout 600 python bench.py > gpurun_out/r1g/bench_cfg3.json 2> gpurun_out/r1g/bench_cfg3.err; echo "bench3 rc=$?"
for c in 1 100; do timeout 200 python tools/contend_bench.py 32768 5 $c; done > gpurun_out/r1g/contend_bench.jsonl 2>&1; cat gpurun_out/r1g/contend_bench.jsonl
