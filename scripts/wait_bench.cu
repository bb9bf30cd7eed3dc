// Latency of an mbarrier wait on an ALREADY COMPLETED phase: try_wait vs test_wait, and of
// a parity query via the state (debug tool: python scripts/run_microbench.py wait_bench)
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
template <int MODE>
__global__ void k(int iters, long long* out) {
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) { mbar_init(&bar[i], 1); } fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) for (int i = 0; i < 4; ++i) mbar_arrive(&bar[i]);   // phase 0 complete
  __syncthreads();
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) { mbar_wait(&bar[it & 3], 0); }
    else if (MODE == 1) { while (!mbar_test(&bar[it & 3], 0)) {} }
    else { mbar_wait(&bar[it & 3], 0); mbar_wait(&bar[(it + 1) & 3], 0); }
    acc += it;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
}
template <int MODE>
void go(const char* name) {
  long long* d; long long h[2];
  cudaMalloc(&d, 16);
  k<MODE><<<1, 32>>>(4096, d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  printf("%-48s %6.1f cycles per iteration\n", name, h[0] / 4096.0);
}
extern "C" void run_all() {
  go<0>("try_wait loop, completed phase");
  go<1>("test_wait spin, completed phase");
  go<2>("two try_waits (independent), completed");
}
