set -u
D=gpurun_out/r2ah; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
ADAPTIS_SEQ_MINW=2 timeout 1200 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_seqminw2.txt 2>&1; grep "GREEDY\|config" $D/breakdown_cfg5_seqminw2.txt
