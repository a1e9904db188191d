set -u
D=gpurun_out/r2d; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_seqg.py -q -rs -x > $D/pytest_seqg.txt 2>&1; tail -3 $D/pytest_seqg.txt
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; cat $D/breakdown_cfg3.txt
for w in 1 2 3; do ADAPTIS_SEQG_MINW=$w timeout 600 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_w$w.txt 2>&1; head -8 $D/breakdown_cfg5_w$w.txt; done
