# A/B: the lane kernel's GREEDY v >= 3 register budget (CTAs per SM) on cfg5's p = 16 v = 4 segments
set -u
D=gpurun_out/r2an; mkdir -p $D
for mb in 3 2; do
  ADAPTIS_GREEDY_V4_MINB=$mb python paper_2509_23722_b200/build.py > $D/build_$mb.txt 2>&1; echo "build $mb rc=$?"
  timeout 900 python tools/search_breakdown.py 5 > $D/b5_v4minb$mb.txt 2>&1; grep "v=4 .*GREEDY\|config" $D/b5_v4minb$mb.txt
done
python paper_2509_23722_b200/build.py > $D/build_back.txt 2>&1; echo "build back rc=$?"
