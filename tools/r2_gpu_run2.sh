set -u
D=gpurun_out/r2b; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py -q -rs -x > $D/pytest_seqg.txt 2>&1; tail -3 $D/pytest_seqg.txt
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; cat $D/breakdown_cfg3.txt
ADAPTIS_NO_SEQG=1 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_noseq.txt 2>&1; head -3 $D/breakdown_cfg3_noseq.txt
timeout 600 python tools/search_breakdown.py 4 > $D/breakdown_cfg4.txt 2>&1; cat $D/breakdown_cfg4.txt
