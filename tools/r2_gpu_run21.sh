set -u
D=gpurun_out/r2ag; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; grep "1F1B\|ZB\|config" $D/breakdown_cfg5.txt
ADAPTIS_FIXED_MINW=2 timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_minw2.txt 2>&1; grep "ZB\|config" $D/breakdown_cfg5_minw2.txt
timeout 900 python -m pytest tests/test_gpu_fixed.py tests/test_gpu_goldens.py -q -x -rs > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt
