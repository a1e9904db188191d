set -u
D=gpurun_out/r2f; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; cp paper_2509_23722_b200/csrc/ptxas.log $D/ptxas.log; echo "build rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:seq_kernel -c 3 -o $D/seq_cfg3 -f python tools/search_breakdown.py 3 > $D/ncu_seq.log 2>&1; echo "ncu rc=$?"; tail -3 $D/ncu_seq.log
