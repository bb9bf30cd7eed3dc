// SM-wide throughput of mbarrier operations: W warps each issue 256 try_waits on completed
// barriers (or arrives on their own barrier), aggregate cycles per operation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mbar_tput mbar_tput.cu
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

__global__ void tput(int mode, long long* out) {
  __shared__ uint64_t bar[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x < 32) { mbar_init(&bar[threadIdx.x], 1 << 20); }
  __syncthreads();
  if (threadIdx.x < 32) { mbar_init(&bar[threadIdx.x], 1); }
  fence_mbar_init();
  __syncthreads();
  if (lane == 0 && mode == 0) mbar_arrive(&bar[warp]);   // complete phase 0
  __syncthreads();
  const int N = 256;
  uint32_t acc = 0;
  long long c0 = clock64();
  if (mode == 0) {          // warp-wide try_wait on a completed barrier, results accumulated (no branch)
#pragma unroll 8
    for (int i = 0; i < N; ++i) acc += mbar_try_wait(&bar[warp], 0) ? 1u : 0u;
  } else if (mode == 1) {   // lane-0 try_wait
    if (lane == 0)
#pragma unroll 8
      for (int i = 0; i < N; ++i) acc += mbar_try_wait(&bar[warp], 0) ? 1u : 0u;
  } else if (mode == 2) {   // lane-0 arrive (barrier count 1 -> every arrive completes a phase)
    if (lane == 0)
#pragma unroll 8
      for (int i = 0; i < N; ++i) mbar_arrive(&bar[warp]);
  } else {                  // named barrier among the warp's own 32 threads
#pragma unroll 8
    for (int i = 0; i < N; ++i) asm volatile("bar.sync %0, 32;" ::"r"(1 + (warp & 7)) : "memory");
  }
  long long c1 = clock64();
  __syncthreads();
  if (lane == 0) out[warp] = (c1 - c0) + (acc == 0x7fffffff);
}

int main() {
  long long* d;
  long long h[32];
  cudaMalloc(&d, 256);
  const char* names[4] = {"warp-wide try_wait (complete)", "lane-0 try_wait (complete)", "lane-0 arrive", "bar.sync 32 thr"};
  for (int mode = 0; mode < 4; ++mode)
    for (int w : {1, 4, 8, 16, 32}) {
      if (mode == 3 && w > 8) continue;
      cudaMemset(d, 0, 256);
      tput<<<1, 32 * w>>>(mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8 * w, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-32s warps %2d: %6.2f cycles per op per warp, SM-wide %6.2f cycles per op %s\n", names[mode], w,
             mx / 256.0, mx / (256.0 * w), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
