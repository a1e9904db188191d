set -u
D=gpurun_out/r2q; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_contended_search.py tests/test_gpu_lists.py tests/test_gpu_goldens.py -q -rs > $D/pytest.txt 2>&1; tail -3 $D/pytest.txt
timeout 900 python - > $D/contended_timing.txt 2>&1 <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_2509_23722_b200 import adaptis as A, workloads as W
ctx = A.Context(0)
for cid, scale in ((2, 1), (2, 100), (3, 1)):
    pr, sp = W.config(cid)
    pr.comm = pr.comm * scale
    prep = ctx.prepare(pr, sp)
    t = time.perf_counter(); b = prep.search_contended(); dt = time.perf_counter() - t
    plain = prep.search()
    print(cid, scale, "contended search %.1f ms (kernel %.1f ms, tasks %d): index %d makespan %d; latency-only winner %d makespan %d"
          % (1000 * dt, b["kernel_ms"], b["n_tasks"], b["index"], b["makespan"], plain["index"], plain["makespan"]), flush=True)
PY
cat $D/contended_timing.txt
timeout 900 python tools/search_breakdown.py 5 > $D/breakdown_cfg5.txt 2>&1; head -9 $D/breakdown_cfg5.txt
