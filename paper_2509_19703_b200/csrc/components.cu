// components.cu -- connected components by lock-free union-find on the GPU.
//
// Replaces the connectivity tests of the reference's host paths
// (graph.py Graph.is_connected / largest_connected_component, scipy csgraph),
// used by spectral_init (layout.py:238-239) and LCC extraction.  Every edge
// (v, u > v) hooks the larger root under the smaller one with atomicCAS
// (retrying on races), then a pointer-jumping pass flattens the forest: each
// vertex's label is the smallest vertex id of its component (deterministic).
#include <climits>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

__device__ __forceinline__ int find_root(int* parent, int x) {
  int p = parent[x];
  while (p != x) {
    const int gp = parent[p];
    if (gp != p) parent[x] = gp;  // path halving (benign race: any ancestor)
    x = p;
    p = gp;
  }
  return x;
}

__global__ void cc_init(int n, int* __restrict__ parent) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    parent[v] = v;
}

// 8 lanes per vertex over its adjacency (u > v only: each edge once)
__global__ void cc_hook(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                        int* parent) {
  const int g8 = threadIdx.x & 7;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 3; v < n;
       v += (gridDim.x * blockDim.x) >> 3) {
    const int b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
    for (int p = b + g8; p < e; p += 8) {
      const int u = __ldg(indices + p);
      if (u <= v) continue;
      for (;;) {
        int ru = find_root(parent, u), rv = find_root(parent, v);
        if (ru == rv) break;
        if (ru < rv) {
          const int t = ru;
          ru = rv;
          rv = t;
        }
        // hook the larger root ru under the smaller rv
        if (atomicCAS(parent + ru, ru, rv) == ru) break;
      }
    }
  }
}

__global__ void cc_flatten(int n, int* parent, int* __restrict__ label, int* __restrict__ ncomp) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int r = find_root(parent, v);
    label[v] = r;
    if (r == v) atomicAdd(ncomp, 1);
  }
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" size_t gu_components_workspace_size(int64_t n) { return sizeof(int) * (size_t)n; }

// labels[v] = smallest vertex id in v's component; out_ncomp: device int
extern "C" int gu_connected_components(int64_t n, const int32_t* indptr, const int32_t* indices,
                                       int32_t* labels, int32_t* out_ncomp, void* workspace,
                                       size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n >= INT_MAX) {
    set_error("gu_connected_components: n=%lld", (long long)n);
    return GU_ERR_ARG;
  }
  if (!workspace || ws_bytes < gu_components_workspace_size(n)) {
    set_error("gu_connected_components: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  GU_CHECK(cudaMemsetAsync(out_ncomp, 0, sizeof(int), st));
  if (n == 0) return GU_OK;
  int* parent = (int*)workspace;
  const int N = (int)n;
  cc_init<<<148 * 4, 256, 0, st>>>(N, parent);
  GU_CHECK_LAUNCH("cc_init");
  cc_hook<<<148 * 16, 256, 0, st>>>(N, indptr, indices, parent);
  GU_CHECK_LAUNCH("cc_hook");
  cc_flatten<<<148 * 4, 256, 0, st>>>(N, parent, labels, out_ncomp);
  GU_CHECK_LAUNCH("cc_flatten");
  return GU_OK;
}
