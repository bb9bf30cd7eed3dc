// Throughput of tcgen05.st shapes (4 KB per warp-instruction each), alone and interleaved
// with the e4m3 expansion ALU work.  Debug tool.
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;

template <int SHAPE>  // 0: 32x32b.x32   1: 16x256b.x8   2: 16x128b.x16   3: 16x64b.x32
__device__ __forceinline__ void st4k(uint32_t ta, const uint32_t (&v)[32]) {
#define R32 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), \
            "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
            "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), \
            "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define L32 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32}"
  if constexpr (SHAPE == 0) asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " L32 ";" ::"r"(ta), R32 : "memory");
  if constexpr (SHAPE == 1) asm volatile("tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], " L32 ";" ::"r"(ta), R32 : "memory");
  if constexpr (SHAPE == 2) asm volatile("tcgen05.st.sync.aligned.16x128b.x16.b32 [%0], " L32 ";" ::"r"(ta), R32 : "memory");
  if constexpr (SHAPE == 3) asm volatile("tcgen05.st.sync.aligned.16x64b.x32.b32 [%0], " L32 ";" ::"r"(ta), R32 : "memory");
}

template <int SHAPE, int EXPAND>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16) + 128 * (warp >> 2);
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1);
  const uint32_t e8 = 0x38383838u ^ (uint32_t)(iters & 0);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t o[32];
    if (EXPAND) {
      expand_e4m3(w, e8, o); expand_e4m3(w ^ 0x55u, e8, o + 8);
      expand_e4m3(w * 3u, e8, o + 16); expand_e4m3(w * 5u, e8, o + 24);
    } else {
      for (int i = 0; i < 32; ++i) o[i] = w + i;
    }
    st4k<SHAPE>(tb + 32 * (it & 3), o);
    w = w * 1664525u + 1013904223u;
  }
  tmem_st_wait();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

template <int SHAPE, int EXPAND>
void run(const char* name, int warps) {
  long long* d; long long h;
  cudaMalloc(&d, 8);
  k<SHAPE, EXPAND><<<1, warps * 32>>>(2048, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  const double per = h / 2048.0;
  printf("%-34s warps %2d: %7.1f cyc/warp-iter -> %6.1f B/clk/SM %s\n", name, warps, per,
         warps * 4096.0 / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

extern "C" void run_all() {
  run<0, 0>("32x32b.x32 store only", 8);
  run<1, 0>("16x256b.x8 store only", 8);
  run<2, 0>("16x128b.x16 store only", 8);
  run<3, 0>("16x64b.x32 store only", 8);
  run<0, 1>("32x32b.x32 + expand", 8);
  run<1, 1>("16x256b.x8 + expand", 8);
  run<2, 1>("16x128b.x16 + expand", 8);
  run<3, 1>("16x64b.x32 + expand", 8);
  run<0, 1>("32x32b.x32 + expand", 16);
  run<1, 1>("16x256b.x8 + expand", 16);
}
