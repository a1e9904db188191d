set -u
D=gpurun_out/r2o; mkdir -p $D
ADAPTIS_ZB_WFILL_ONE=1 python paper_2509_23722_b200/build.py > $D/build1.txt 2>&1; echo "build one rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_wone.txt 2>&1; grep "ZB\|config" $D/breakdown_cfg3_wone.txt
timeout 600 python tools/search_breakdown.py 4 > $D/breakdown_cfg4_wone.txt 2>&1; grep "ZB\|config" $D/breakdown_cfg4_wone.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random or cfg2 or edges" > $D/pytest_wone.txt 2>&1; tail -2 $D/pytest_wone.txt
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; grep "ZB\|config" $D/breakdown_cfg3.txt
timeout 2400 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -3 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
