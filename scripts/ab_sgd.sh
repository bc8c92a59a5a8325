# A/B of libgumap builds (GU_LIB_PATH) on the SGD epoch perf script
for v in "$@"; do
  for c in c5 c3; do
    GU_LIB_PATH=paper_2509_19703_b200/$v/libgumap.so python scripts/perf_sgd.py $c 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
