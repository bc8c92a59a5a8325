// Microbenchmark: per-SM throughput of warp collectives used by the partial
// BFS fast tier (MATCH.ANY, VOTE.ANY/ballot, REDUX.OR, SHFL, shared CAS).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_micro_match scripts/micro_match.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void kern(unsigned* out, unsigned seed) {
  __shared__ int tab[8][512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < 512; i += 32) tab[warp][i] = -1;
  __syncwarp();
  unsigned x = seed * (threadIdx.x + 1) + blockIdx.x, acc = 0;
#pragma unroll 8
  for (int i = 0; i < ITERS; i++) {
    unsigned v = x + (unsigned)i * 0x9E3779B1u;
    v = (v >> 27) ^ (lane & 3);  // few distinct values: groups of lanes match
    if (OP == 0) acc += __match_any_sync(0xffffffffu, v);
    if (OP == 1) acc += __ballot_sync(0xffffffffu, v & 1);
    if (OP == 2) acc += __reduce_or_sync(0xffffffffu, v);
    if (OP == 3) acc += __shfl_sync(0xffffffffu, v, (lane + i) & 31);
    if (OP == 4) acc += atomicCAS(&tab[warp][(v * 37u + lane * 13u) & 511], -1, (int)v);
    if (OP == 5) acc += v * 3u;  // ALU baseline
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int OP>
float run(const char* name, unsigned* out, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<OP><<<blocks, 256>>>(out, 1);
  cudaEventRecord(a);
  kern<OP><<<blocks, 256>>>(out, 2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_ops = (double)blocks * 8 * ITERS;
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-10s %8.3f ms  %6.2f warp-ops / SM / cycle (%.1f cycles per op per SM)\n", name, ms,
         warp_ops / sms / cycles, sms * cycles / warp_ops);
  return ms;
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8 * 4;
  run<0>("match.any", out, blocks);
  run<1>("ballot", out, blocks);
  run<2>("redux.or", out, blocks);
  run<3>("shfl", out, blocks);
  run<4>("atoms.cas", out, blocks);
  run<5>("alu", out, blocks);
  return 0;
}
