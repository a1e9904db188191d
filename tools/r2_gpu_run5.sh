set -u
D=gpurun_out/r2g; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; cp paper_2509_23722_b200/csrc/ptxas.log $D/; echo "build rc=$?"
for c in 2 3 4; do timeout 600 python tools/search_breakdown.py $c > $D/breakdown_cfg$c.txt 2>&1; cat $D/breakdown_cfg$c.txt; done
timeout 900 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py -q -rs -x > $D/pytest_seq.txt 2>&1; tail -3 $D/pytest_seq.txt
