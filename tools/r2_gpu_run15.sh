set -u
D=gpurun_out/r2x; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; cat $D/breakdown_cfg5.txt
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; head -4 $D/breakdown_cfg3.txt
timeout 600 python tools/search_breakdown.py 4 > $D/breakdown_cfg4.txt 2>&1; cat $D/breakdown_cfg4.txt
timeout 900 python -m pytest tests/test_gpu_fixed.py tests/test_gpu_seqg.py -q -x -rs > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt
