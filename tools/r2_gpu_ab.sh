set -u
D=gpurun_out/r2j; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; cp paper_2509_23722_b200/csrc/ptxas.log $D/; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/new.txt 2>&1; head -1 $D/new.txt; grep "GREEDY\|ZB\|1F1B" $D/new.txt
ADAPTIS_SEQ_OLD=1 timeout 600 python tools/search_breakdown.py 3 > $D/old.txt 2>&1; grep GREEDY $D/old.txt
timeout 600 python tools/search_breakdown.py 5 > $D/new5.txt 2>&1; cat $D/new5.txt
