# A/B of libgumap builds (GU_LIB_PATH) on the partial BFS and SGD perf scripts
for v in "$@"; do
  for c in c5 c4; do
    GU_LIB_PATH=paper_2509_19703_b200/$v/libgumap.so python scripts/perf_pbfs.py $c 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
