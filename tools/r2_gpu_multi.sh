set -u
D=gpurun_out/r2n; mkdir -p $D
nvidia-smi -L > $D/gpus.txt 2>&1
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 1500 python bench.py --gpus 2 --steps 5 --warmup 3 > $D/bench_n2.json 2> $D/bench_n2.err; echo "bench n2 rc=$?"
timeout 600 python bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $D/bench_ref_n2.json 2>&1; echo "ref n2 rc=$?"
tail -c 1500 $D/bench_n2.json
