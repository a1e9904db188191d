set -u
D=gpurun_out/r2t; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"

ADAPTIS_SEQG_H=2 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_h2.txt 2>&1; head -3 $D/breakdown_cfg3_h2.txt; grep "v=1 SEQ  GREEDY" $D/breakdown_cfg3_h2.txt
ADAPTIS_SEQG_H=2 timeout 1500 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py -q -x -rs > $D/pytest_h2.txt 2>&1; tail -3 $D/pytest_h2.txt
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; head -7 $D/breakdown_cfg5.txt
ADAPTIS_SEQG_H2_MAXW=16 python paper_2509_23722_b200/build.py > $D/build16.txt 2>&1; echo "build16 rc=$?"
ADAPTIS_SEQG_H=2 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_h2_w16.txt 2>&1; head -3 $D/breakdown_cfg3_h2_w16.txt
ADAPTIS_SEQG_H2_MAXW=8 python paper_2509_23722_b200/build.py > $D/build8.txt 2>&1; echo "build8 rc=$?"
ADAPTIS_SEQG_H=2 timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3_h2_w8.txt 2>&1; head -3 $D/breakdown_cfg3_h2_w8.txt
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_w8.txt 2>&1; head -4 $D/breakdown_cfg5_w8.txt
