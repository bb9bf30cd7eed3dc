// mbarrier hand-off latency between two warps (ping-pong), and a named-barrier ping-pong.
// Debug tool: python scripts/run_microbench.py pingpong
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
template <int MODE>
__device__ __forceinline__ void w8(uint64_t* bar, uint32_t ph) {
  if (MODE == 0) mbar_wait(bar, ph);
  else if (MODE == 1) { while (!mbar_test(bar, ph)) {} }
  else {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph), "r"(MODE == 2 ? 10u : 100000u) : "memory");
  }
}
template <int MODE, int LANE0_ARRIVE>
__global__ void pp(int iters, long long* out) {
  __shared__ uint64_t b1, b2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&b1, 1); mbar_init(&b2, 1); fence_mbar_init(); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t ph = it & 1;
    if (warp == 0) {
      if (lane == 0) mbar_arrive(&b1);
      w8<MODE>(&b2, ph);
    } else if (warp == 1) {
      w8<MODE>(&b1, ph);
      if (lane == 0) mbar_arrive(&b2);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void pp_named(int iters, long long* out) {
  const int warp = threadIdx.x / 32;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (warp == 0) { asm volatile("bar.arrive 1, 64;"); asm volatile("bar.sync 2, 64;"); }
    else { asm volatile("bar.sync 1, 64;"); asm volatile("bar.arrive 2, 64;"); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
template <typename K>
void go(K k, const char* name, int threads) {
  long long* d; long long h = 0;
  cudaMalloc(&d, 8);
  k<<<1, threads>>>(2000, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  printf("%-44s %8.1f cycles per round trip %s\n", name, h / 2000.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
extern "C" void run_all() {
  go(pp<0, 1>, "mbarrier ping-pong, try_wait", 64);
  go(pp<1, 1>, "mbarrier ping-pong, test_wait spin", 64);
  go(pp<2, 1>, "mbarrier ping-pong, try_wait hint 10ns", 64);
  go(pp<3, 1>, "mbarrier ping-pong, try_wait hint 100us", 64);
  go(pp_named, "named barrier ping-pong (bar.arrive/bar.sync)", 64);
  go(pp<0, 1>, "mbarrier ping-pong try_wait, +14 idle warps", 512);
}
