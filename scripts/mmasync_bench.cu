// Legacy warp-level mma.sync throughput on sm_100a (register-fragment MMA), per SM.
// Debug tool: python scripts/run_microbench.py mmasync_bench
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* out, float* sink) {
  uint32_t a0 = threadIdx.x * 0x01010101u, a1 = a0 ^ 0x38383838u, a2 = a0 + 7, a3 = a1 + 9;
  uint32_t b0 = a0 ^ 0x12345678u, b1 = b0 + 3;
  float c[4][4] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {   // 4 independent accumulators
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(*reinterpret_cast<int*>(&c[j][0])), "+r"(*reinterpret_cast<int*>(&c[j][1])),
                       "+r"(*reinterpret_cast<int*>(&c[j][2])), "+r"(*reinterpret_cast<int*>(&c[j][3]))
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 4; ++j) for (int e = 0; e < 4; ++e) s += c[j][e];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
template <int KIND>
void go(const char* name, int warps, int macs_per_mma) {
  long long* d; float* sink; long long h;
  cudaMalloc(&d, 8); cudaMalloc(&sink, 4096);
  const int iters = 4096;
  k<KIND><<<1, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d); cudaFree(sink);
  const double mmas = (double)iters * 4 * warps;
  printf("%-36s warps %2d: %6.2f cycles per warp-mma, %7.0f MAC/clk/SM %s\n", name, warps, h / ((double)iters * 4),
         mmas * macs_per_mma / h, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
extern "C" void run_all() {
  for (int w : {4, 8, 16}) go<0>("mma.sync m16n8k32 e4m3 -> f32", w, 16 * 8 * 32);
  for (int w : {4, 8, 16}) go<1>("mma.sync m16n8k16 f16 -> f32", w, 16 * 8 * 16);
  for (int w : {4, 16}) go<2>("mma.sync m16n8k32 s8 -> s32", w, 16 * 8 * 32);
}
