# Round-2 final evidence run (final code) (one B200): GPU tests + smoke, bench (cfg3 headline + cfg5 leg) and
# the reference arm, per-config breakdowns, the launch list of the bench command, ncu --set full
# of the dominant kernel and of the static-order kernel.
set -u
D=gpurun_out/r2ae; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt 2>&1
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"; cp paper_2509_23722_b200/csrc/ptxas.log $D/
timeout 2700 python -m pytest tests -m gpu -q -rs > $D/pytest_gpu.txt 2>&1; tail -3 $D/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -1 $D/smoke.txt
timeout 1500 python bench.py --steps 5 --warmup 3 > $D/bench_cfg3.json 2> $D/bench_cfg3.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_cfg3_reference.json 2>&1; echo "ref rc=$?"
for c in 2 3 4; do timeout 600 python tools/search_breakdown.py $c > $D/breakdown_cfg$c.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_cfg3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --cfg5-steps 0 > $D/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:seqg_kernel --launch-skip 1 -c 1 -o $D/seqg_int -f python tools/search_breakdown.py 3 > $D/ncu_int.log 2>&1; echo "ncu int rc=$?"; python tools/ncu_summary.py $D/seqg_int.ncu-rep > $D/ncu_seqg_int.txt 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:seqg_kernel --launch-skip 2 -c 1 -o $D/seqg_wave -f python tools/search_breakdown.py 3 > $D/ncu_wave.log 2>&1; echo "ncu wave rc=$?"; python tools/ncu_summary.py $D/seqg_wave.ncu-rep > $D/ncu_seqg_wave.txt 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:fixed_kernel --launch-skip 5 -c 1 -o $D/fixed_zb -f python tools/search_breakdown.py 3 > $D/ncu_fixed.log 2>&1; echo "ncu fixed rc=$?"; python tools/ncu_summary.py $D/fixed_zb.ncu-rep > $D/ncu_fixed_zb.txt 2>&1
# keep the returned directory under gpurun's 64 MiB: the summaries stay, the WAVE report (the bench's dominant kernel) stays
rm -f $D/seqg_int.ncu-rep $D/fixed_zb.ncu-rep $D/ptxas.log; du -sh $D
