set -u
D=gpurun_out/r2ac; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_fixed.py tests/test_gpu_parity.py -q -x -rs > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt; grep -m3 -B3 Error $D/pytest.txt
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; head -12 $D/breakdown_cfg3.txt
timeout 600 python tools/search_breakdown.py 2 > $D/breakdown_cfg2.txt 2>&1; head -3 $D/breakdown_cfg2.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:seqg_kernel --launch-skip 2 -c 1 -o $D/seqg_wave -f python tools/search_breakdown.py 3 > $D/ncu_wave.log 2>&1; echo "ncu wave rc=$?"; tail -2 $D/ncu_wave.log
