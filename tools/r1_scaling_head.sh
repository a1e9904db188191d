# N = 1, 2, 4 bench lines on one box, current code (run under gpurun --gpus 4); also the reference arm at N = 2
mkdir -p gpurun_out/r1hs
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r1hs/bench_n1.json 2>&1; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --no-cpu-baseline > gpurun_out/r1hs/bench_n$n.json 2>&1; echo "n$n rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k sharded 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 > gpurun_out/r1hs/bench_ref_n2.json 2>&1; echo "ref n2 rc=$?"
