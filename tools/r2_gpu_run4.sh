set -u
D=gpurun_out/r2e; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_seqg.py -q -rs -x > $D/pytest_seq.txt 2>&1; tail -3 $D/pytest_seq.txt
for c in 2 3 4; do timeout 600 python tools/search_breakdown.py $c > $D/breakdown_cfg$c.txt 2>&1; cat $D/breakdown_cfg$c.txt; done
ADAPTIS_NO_SEQ=1 timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5_lane.txt 2>&1; cat $D/breakdown_cfg5_lane.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -5 $D/pytest_gpu.txt
