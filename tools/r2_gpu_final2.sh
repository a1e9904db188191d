# Final-code confirmation (one B200): GPU tests + smoke, the default bench line, the reference arm, breakdowns.
set -u
D=gpurun_out/r2ai; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -3 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 1500 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo "bench rc=$?"; tail -c 300 $D/bench_default.json
timeout 600 python bench.py --impl reference > $D/bench_reference.json 2>&1; echo "ref rc=$?"
for c in 2 3 4; do timeout 900 python tools/search_breakdown.py $c > $D/breakdown_cfg$c.txt 2>&1; head -3 $D/breakdown_cfg$c.txt; done
