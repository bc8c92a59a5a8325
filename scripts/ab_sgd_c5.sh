# A/B of libgumap builds on the SGD epoch (perf_sgd.py), interleaved twice
for r in 1 2; do for v in "$@"; do
  GU_LIB_PATH=paper_2509_19703_b200/$v/libgumap.so python scripts/perf_sgd.py ${CFG:-c5} 2>&1 | tail -1 | sed "s/^/$v /"
done; done
