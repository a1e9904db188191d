set -u
D=gpurun_out/r2al; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/b3_default.txt 2>&1; head -3 $D/b3_default.txt
ADAPTIS_SEQG_REGKEYS=1 python paper_2509_23722_b200/build.py > $D/build_rk.txt 2>&1; echo "build rk rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/b3_regkeys.txt 2>&1; head -3 $D/b3_regkeys.txt
timeout 900 python -m pytest tests/test_gpu_seqg.py -q -x > $D/pytest_rk.txt 2>&1; tail -1 $D/pytest_rk.txt
timeout 900 python tools/search_breakdown.py 5 > $D/b5_regkeys.txt 2>&1; grep "GREEDY\|config" $D/b5_regkeys.txt
python paper_2509_23722_b200/build.py > $D/build_back.txt 2>&1; echo "build back rc=$?"
