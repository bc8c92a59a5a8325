# A/B of libgumap builds on C1 (smooth_knn_weights, scripts/perf_c1.py), last rep of each
for r in 1 2; do for v in "$@"; do
  GU_LIB_PATH=paper_2509_19703_b200/$v/libgumap.so python scripts/perf_c1.py ${CFG:-c5} 2>&1 | tail -1 | sed "s/^/$v /"
done; done
