# T6 substitute (compute-sanitizer is closed on this pool): build with device
# DCHECKs (ADAPTIS_DEBUG=1: ring addresses, stage/cut/index/task ranges, trap on
# failure), run the exhaustive small-space parity tests, then rebuild release.
set -e
ADAPTIS_DEBUG=1 python paper_2509_23722_b200/build.py --force > /dev/null
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q \
  -k "cfg1 or random_small or cap_exactly or edge_shapes or cfg2_blocks or device_resident" 2>&1 | tail -3
python paper_2509_23722_b200/build.py --force > /dev/null
