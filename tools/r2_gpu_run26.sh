# A/B: the lane kernel's GREEDY v <= 2 register budget on cfg5's WAVE v = 2 segment (the only v <= 2 GREEDY lane launch left)
set -u
D=gpurun_out/r2ap; mkdir -p $D
for mb in 4 3; do
  ADAPTIS_GREEDY_MINB=$mb python paper_2509_23722_b200/build.py > $D/build_$mb.txt 2>&1; echo "build $mb rc=$?"
  timeout 900 python tools/search_breakdown.py 5 > $D/b5_minb$mb.txt 2>&1; grep "v=2 WAVE GREEDY\|config" $D/b5_minb$mb.txt
done
python paper_2509_23722_b200/build.py > $D/build_back.txt 2>&1; echo "build back rc=$?"
