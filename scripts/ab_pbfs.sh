# A/B of libgumap builds (GU_LIB_PATH) on the partial BFS perf script.
#   scripts/ab_pbfs.sh _build_A _build_B ...   (dirs under paper_2509_19703_b200/)
# GU_PBFS_MODE=fast in the environment selects the 32-lane tier F kernel.
for v in "$@"; do
  for c in c5 c4 c3; do
    GU_LIB_PATH=paper_2509_19703_b200/$v/libgumap.so python scripts/perf_pbfs.py $c 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
