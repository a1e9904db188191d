set -u
D=gpurun_out/r2c; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:seqg_kernel -c 1 -o $D/seqg_v2 -f python tools/search_breakdown.py 3 > $D/ncu_seqg.log 2>&1; echo "ncu rc=$?"; tail -3 $D/ncu_seqg.log
