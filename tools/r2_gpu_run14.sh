set -u
D=gpurun_out/r2w; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_fixed.py tests/test_gpu_goldens.py -q -x -rs > $D/pytest_fixed.txt 2>&1; tail -3 $D/pytest_fixed.txt; grep -m3 -B3 "Error" $D/pytest_fixed.txt
for c in 2 3; do timeout 600 python tools/search_breakdown.py $c > $D/breakdown_cfg$c.txt 2>&1; head -12 $D/breakdown_cfg$c.txt; done
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; cat $D/breakdown_cfg5.txt
ADAPTIS_FIXED_MINW=4 timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_minw4.txt 2>&1; cat $D/breakdown_cfg5_minw4.txt
timeout 600 python tools/search_breakdown.py 3 --prune > $D/breakdown_cfg3_prune.txt 2>&1; head -12 $D/breakdown_cfg3_prune.txt
