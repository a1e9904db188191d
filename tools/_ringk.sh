for k in 8 16 32; do
  echo "== K $k"
  for a in "5 6" "5 5" "5 12" "3 6" "3 5"; do set -- $a
    ADAPTIS_RING_K=$k timeout 300 python tools/diag_segments.py --config $1 --only $2 --count 1000000 2>&1 | tail -1 | cut -c1-170
  done
done
