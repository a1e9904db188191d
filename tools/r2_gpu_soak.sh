# Round-2 parity soak on the final kernels (eval mode: sequential, static-order and lane kernels)
set -u
D=gpurun_out/r2aj; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 2400 python tools/parity_soak.py --seed 2026 2:all 3:3000000 4:1000000 5:200000 > $D/soak.jsonl 2> $D/soak.err; echo "soak rc=$?"; cat $D/soak.jsonl
