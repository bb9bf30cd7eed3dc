// Issue-throughput microbenchmark of tcgen05.mma (A from TMEM) per kind / N, one template
// instantiation per variant so every loop compiles to straight uniform-register code.
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

template <int KIND, int N>  // KIND 0 f16, 1 f8f6f4 (e4m3), 2 i8
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t en) {
  if constexpr (KIND == 0) {
    constexpr uint32_t id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
                 "n"(id), "r"(en));
  } else if constexpr (KIND == 1) {
    constexpr uint32_t id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
                 "n"(id), "r"(en));
  } else {
    constexpr uint32_t id = (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
                 "n"(id), "r"(en));
  }
}

template <int KIND, int N, int PER_COMMIT>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t zs[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < 16384 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  const uint64_t bdesc = smem_desc_kmajor(smem_u32(zs), (N / 8) * 128, 128);
  long long t0 = clock64();
  if (warp == 1) {
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int m = 0; m < 8; ++m) mma<KIND, N>(t + 256, t + 64 * (it & 3) + 8 * m, bdesc, m > 0 ? 1u : 0u);
        if ((it % PER_COMMIT) == PER_COMMIT - 1) mma_commit(&bar);
      }
      __syncwarp();
    }
    mbar_wait(&bar, (iters / PER_COMMIT - 1) & 1);
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 32) out[0] = t1 - t0;
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int KIND, int N, int PC>
void run(const char* name, int iters) {
  long long* d;
  long long h = 0;
  cudaMalloc(&d, 8);
  bench<KIND, N, PC><<<1, 128>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  printf("%-34s %8.1f cycles per 8 MMAs  (%5.1f per MMA) %s\n", name, (double)h / iters, (double)h / iters / 8,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

extern "C" void run_all() {
  const int it = 4000;
  run<0, 16, 1>("f16 K16 N16 commit/8", it);
  run<0, 16, 4>("f16 K16 N16 commit/32", it);
  run<0, 32, 1>("f16 K16 N32", it);
  run<0, 64, 1>("f16 K16 N64", it);
  run<0, 128, 1>("f16 K16 N128", it);
  run<1, 16, 1>("e4m3 K32 N16", it);
  run<1, 32, 1>("e4m3 K32 N32", it);
  run<1, 48, 1>("e4m3 K32 N48", it);
  run<1, 64, 1>("e4m3 K32 N64", it);
  run<1, 128, 1>("e4m3 K32 N128", it);
  run<2, 32, 1>("i8 K32 N32", it);
  run<2, 64, 1>("i8 K32 N64", it);
  run<2, 128, 1>("i8 K32 N128", it);
}
