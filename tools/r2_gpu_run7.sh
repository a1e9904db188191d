set -u
D=gpurun_out/r2m; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; cp paper_2509_23722_b200/csrc/ptxas.log $D/; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; head -6 $D/breakdown_cfg3.txt
timeout 600 python tools/search_breakdown.py 4 > $D/breakdown_cfg4.txt 2>&1; head -4 $D/breakdown_cfg4.txt
ADAPTIS_SEQ_MINW=4 timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_w4.txt 2>&1; head -8 $D/breakdown_cfg5_w4.txt
timeout 1800 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py tests/test_gpu_memory.py -q -rs -x > $D/pytest.txt 2>&1; tail -3 $D/pytest.txt
timeout 900 python tools/repair_sample.py 3 4 --n 32 > $D/repair_sample.txt 2>&1; cat $D/repair_sample.txt | tail -3
ADAPTIS_SEQG_COMPACT=0 python paper_2509_23722_b200/build.py > $D/build0.txt 2>&1; echo "build0 rc=$?"
ADAPTIS_SEQG_COMPACT=0 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_noncompact.txt 2>&1; head -6 $D/breakdown_cfg3_noncompact.txt
