set -u
D=gpurun_out/r2ab; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; head -6 $D/breakdown_cfg3.txt
ADAPTIS_SEQ_MAXCTA=8 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_cta8.txt 2>&1; head -3 $D/breakdown_cfg3_cta8.txt
timeout 900 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py -q -x -rs > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt; grep -m3 -B3 Error $D/pytest.txt
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; head -8 $D/breakdown_cfg5.txt
