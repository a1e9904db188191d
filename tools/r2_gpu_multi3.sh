# Final code at N = 2 and N = 4 on one box: plain `python bench.py --gpus N` (cfg3 headline + cfg5 leg).
set -u
D=gpurun_out/r2ak; mkdir -p $D
nvidia-smi -L > $D/gpus.txt 2>&1
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
for n in 2 4; do
  timeout 1500 python bench.py --gpus $n > $D/bench_n$n.json 2> $D/bench_n$n.err; echo "bench n$n rc=$?"
  tail -c 400 $D/bench_n$n.json
done
timeout 600 python bench.py --impl reference --gpus 2 > $D/bench_ref_n2.json 2>&1; echo "ref n2 rc=$?"
