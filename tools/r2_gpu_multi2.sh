# VERDICT r1 item 5 done-criterion: plain `python bench.py --gpus 4 --config 5` on one 4-GPU box
# (4 NCCL ranks, the same winner as N = 1), plus the cfg3 headline at N = 4 with its cfg5 leg.
set -u
D=gpurun_out/r2m4; mkdir -p $D
nvidia-smi -L > $D/gpus.txt 2>&1
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 1500 python bench.py --gpus 4 --config 5 --steps 2 --warmup 3 > $D/bench_cfg5_n4.json 2> $D/bench_cfg5_n4.err; echo "cfg5 n4 rc=$?"
tail -c 1200 $D/bench_cfg5_n4.json
timeout 1500 python bench.py --gpus 4 --steps 5 --warmup 3 > $D/bench_cfg3_n4.json 2> $D/bench_cfg3_n4.err; echo "cfg3 n4 rc=$?"
tail -c 1200 $D/bench_cfg3_n4.json
