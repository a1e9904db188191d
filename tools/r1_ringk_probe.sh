# ZB fast-path ring depth probe (DESIGN §9 item 2): per-segment throughput and
# fallback counts of the ZB segments at ADAPTIS_RING_K = 8 / 16 / 32
set -u
D=gpurun_out/r1k; mkdir -p $D
for K in 8 16 32; do
  for spec in "5 6" "5 12" "3 6" "4 6"; do
    set -- $spec
    echo "== K=$K cfg=$1 seg=$2" >> $D/ringk.txt
    ADAPTIS_RING_K=$K timeout 300 python tools/diag_segments.py --config $1 --only $2 --count 4000000 >> $D/ringk.txt 2>&1
  done
done
tail -40 $D/ringk.txt
