set -u
D=gpurun_out/r2aq; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -2 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; head -6 $D/breakdown_cfg5.txt
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; head -3 $D/breakdown_cfg3.txt
