# cfg5 at N = 4 and 2 on one box, current code (gpurun --gpus 4)
mkdir -p gpurun_out/r1hs5
for n in 4 2; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus $n --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1hs5/bench_cfg5_n$n.json 2>&1; echo "n$n rc=$?"
  tail -c 600 gpurun_out/r1hs5/bench_cfg5_n$n.json
done
