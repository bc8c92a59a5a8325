// Microbenchmark: which warp-level instructions issue to the ADU pipe on
// sm_100a, and how many per SM per cycle.  Each kernel repeats one construct
// ITERS times; run under ncu with sm__inst_executed_pipe_adu.sum and
// smsp__inst_executed.sum, and timed with events without ncu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_micro_adu scripts/micro_adu.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
__constant__ unsigned ctab[256];

template <int OP>
__global__ void __launch_bounds__(256) kern(unsigned* out, unsigned seed) {
  __shared__ int tab[8][512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < 512; i += 32) tab[warp][i] = -1;
  __syncwarp();
  unsigned x = seed * (threadIdx.x + 1) + blockIdx.x, acc = 0;
#pragma unroll 1
  for (int i = 0; i < ITERS; i++) {
    unsigned v = x + (unsigned)i * 0x9E3779B1u;
    if (OP == 0) acc += __match_any_sync(0xffffffffu, v >> 27);
    if (OP == 1) acc += __ballot_sync(0xffffffffu, v & 1);
    if (OP == 2) acc += __reduce_or_sync(0xffffffffu, v);
    if (OP == 3) acc += __shfl_sync(0xffffffffu, v, (lane + i) & 31);
    if (OP == 4) acc += atomicCAS(&tab[warp][(v * 37u + lane * 13u) & 511], -1, (int)v);
    if (OP == 5) acc = (acc ^ (v * 3u)) * 0x9E3779B1u;  // loop only (uniform back-edge)
    if (OP == 6) {  // lane-divergent branch (a variable-trip loop inside: no predication)
      acc = (acc ^ v) * 0x9E3779B1u;
      if ((v >> 13) & 1) {
#pragma unroll 1
        for (unsigned q = 0; q < (v & 1) + 1; q++) acc = acc * 5u + q;
      }
    }
    if (OP == 12) {  // four independent MATCH per iteration
      acc += __match_any_sync(0xffffffffu, v >> 27) + __match_any_sync(0xffffffffu, v >> 26) +
             __match_any_sync(0xffffffffu, v >> 25) + __match_any_sync(0xffffffffu, v >> 24);
    }
    if (OP == 13) {
      acc += __reduce_or_sync(0xffffffffu, v) + __reduce_or_sync(0xffffffffu, v >> 1) +
             __reduce_or_sync(0xffffffffu, v >> 2) + __reduce_or_sync(0xffffffffu, v >> 3);
    }
    if (OP == 14) {
      acc += ctab[(v >> 24) & 255] + ctab[(v >> 16) & 255] + ctab[(v >> 8) & 255] + ctab[v & 255];
    }
    if (OP == 15) {
      acc += __shfl_sync(0xffffffffu, v, (lane + i) & 31) + __shfl_sync(0xffffffffu, v >> 1, (lane + 3) & 31) +
             __shfl_sync(0xffffffffu, v >> 2, (lane + 5) & 31) + __shfl_sync(0xffffffffu, v >> 3, (lane + 7) & 31);
    }
    if (OP == 16) {  // four MATCH on all-distinct values
      acc += __match_any_sync(0xffffffffu, v) + __match_any_sync(0xffffffffu, v + 1) +
             __match_any_sync(0xffffffffu, v + 2) + __match_any_sync(0xffffffffu, v + 3);
    }
    if (OP == 17) {  // four ballots
      acc += __ballot_sync(0xffffffffu, v & 1) + __ballot_sync(0xffffffffu, v & 2) +
             __ballot_sync(0xffffffffu, v & 4) + __ballot_sync(0xffffffffu, v & 8);
    }
    if (OP == 11) {  // the same with a warp-uniform condition
      acc = (acc ^ v) * 0x9E3779B1u;
      if ((i >> 1) & 1) {
#pragma unroll 1
        for (unsigned q = 0; q < (v & 1) + 1; q++) acc = acc * 5u + q;
      }
    }
    if (OP == 7) acc += __any_sync(0xffffffffu, (v & 7) == 0);
    if (OP == 8) acc += ctab[(v >> 24) & 255];  // dynamic constant index
    if (OP == 9) {
      tab[warp][lane] = (int)v;
      __syncwarp();
      acc += tab[warp][(lane + 1) & 31];
    }
    if (OP == 10) {  // divergent branch followed by a shuffle (BSSY/BSYNC)
      acc = (acc ^ v) * 0x9E3779B1u;
      if ((v >> 13) & 1) {
#pragma unroll 1
        for (unsigned q = 0; q < (v & 1) + 1; q++) acc = acc * 5u + q;
      }
      acc += __shfl_sync(0xffffffffu, acc, 3);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int OP>
void run(const char* name, unsigned* out, int blocks) {
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
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double iters = (double)blocks * 8 * ITERS;
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-12s %8.3f ms  %6.3f cycles per warp-iteration per SM\n", name, ms, sms * cycles / iters);
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
  run<5>("loop", out, blocks);
  run<6>("div-store", out, blocks);
  run<7>("any", out, blocks);
  run<8>("ldc-dyn", out, blocks);
  run<9>("syncwarp", out, blocks);
  run<10>("div+shfl", out, blocks);
  run<11>("uni-branch", out, blocks);
  run<12>("4x match", out, blocks);
  run<13>("4x redux", out, blocks);
  run<14>("4x ldc-dyn", out, blocks);
  run<15>("4x shfl", out, blocks);
  run<16>("4x match-dist", out, blocks);
  run<17>("4x ballot", out, blocks);
  return 0;
}
