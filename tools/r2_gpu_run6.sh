set -u
D=gpurun_out/r2l; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; cp paper_2509_23722_b200/csrc/ptxas.log $D/; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/breakdown_cfg3.txt 2>&1; cat $D/breakdown_cfg3.txt | head -4
timeout 1800 python -m pytest tests/test_gpu_seqg.py tests/test_gpu_goldens.py tests/test_gpu_memory.py tests/test_gpu_generator.py -q -rs > $D/pytest.txt 2>&1; tail -3 $D/pytest.txt
timeout 600 python - > $D/gen_timing.txt 2>&1 <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_2509_23722_b200 import adaptis as A, workloads as W
ctx = A.Context(0)
for cid in (3, 4, 5):
    pr, _ = W.config(cid)
    for mode in ("bottleneck", "round-robin"):
        ctx.generate(pr, mode=mode)
        t = time.perf_counter(); g = ctx.generate(pr, mode=mode); dt = time.perf_counter() - t
        print(cid, mode, "wall_ms %.1f kernel_ms %.1f n_eval %d rounds %d steps %s" % (1000 * dt, g["kernel_ms"], g["n_evaluated"], g["rounds"], g["steps"]), flush=True)
PY
cat $D/gen_timing.txt
timeout 900 python tools/repair_sample.py 3 4 --n 32 > $D/repair_sample.txt 2>&1; cat $D/repair_sample.txt
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:seqg_kernel --launch-skip 2 -c 1 -o $D/dominant_wave -f python tools/search_breakdown.py 3 > $D/ncu_full.log 2>&1; echo "ncu full rc=$?"
