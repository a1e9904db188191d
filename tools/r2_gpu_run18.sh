set -u
D=gpurun_out/r2aa; mkdir -p $D
python paper_2509_23722_b200/build.py > $D/build.txt 2>&1; echo "build rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/b3_default.txt 2>&1; head -3 $D/b3_default.txt
ADAPTIS_SEQ_MAXCTA=7 timeout 600 python tools/search_breakdown.py 3 > $D/b3_cta7.txt 2>&1; head -3 $D/b3_cta7.txt
ADAPTIS_SEQ_MAXCTA=6 timeout 600 python tools/search_breakdown.py 3 > $D/b3_cta6.txt 2>&1; head -3 $D/b3_cta6.txt
ADAPTIS_SEQG_WAVE_OVERLAP=1 python paper_2509_23722_b200/build.py > $D/build_wo.txt 2>&1; echo "build wo rc=$?"
timeout 600 python tools/search_breakdown.py 3 > $D/b3_waveoverlap.txt 2>&1; head -3 $D/b3_waveoverlap.txt
ADAPTIS_SEQ_MAXCTA=7 timeout 600 python tools/search_breakdown.py 3 > $D/b3_waveoverlap_cta7.txt 2>&1; head -3 $D/b3_waveoverlap_cta7.txt
python paper_2509_23722_b200/build.py > $D/build2.txt 2>&1; echo "build rc=$?"
ADAPTIS_SEQ_MINW=4 timeout 900 python tools/search_breakdown.py 5 > $D/b5_minw4.txt 2>&1; head -5 $D/b5_minw4.txt
