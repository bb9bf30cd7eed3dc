// HBM -> SMEM streaming rate of 1D bulk copies (cp.async.bulk) through a STAGES-deep mbarrier
// ring, one CTA per SM and a consumer warp that only waits `full` and arrives `empty`, for
// (a) contiguous chunks per CTA and (b) the decode kernel's sign-tile pattern: CTA (g, j) of
// G row groups x J CTAs reads units u in its K range, chunk at u * stride + g * chunk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bench stream_bench.cu
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

template <int STAGES>
__global__ void __launch_bounds__(64, 1) stream(const uint8_t* src, int units, int chunk, long long stride, int G,
                                                int J, long long* out, const uint8_t* zsrc, int zbytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int g = blockIdx.x / J, j = blockIdx.x % J;
  const int u0 = (int)((long long)units * j / J), u1 = (int)((long long)units * (j + 1) / J);
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0; uint32_t ph = 0;
      for (int u = u0; u < u1; ++u) {
        if (u - u0 >= STAGES) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], chunk + zbytes);
        if (zbytes)   // a second copy per unit from an L2-resident buffer (the decode's Zq unit)
          bulk_g2s(smem + STAGES * chunk + s * zbytes, zsrc + (long long)u * zbytes, zbytes, &full[s], pol);
        bulk_g2s(smem + s * chunk, src + (long long)u * stride + (long long)g * chunk, chunk, &full[s], pol);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
}

template <int STAGES>
void go(const char* name, const uint8_t* buf, int units, int chunk, long long stride, int G, int J,
        const uint8_t* zbuf = nullptr, int zbytes = 0) {
  long long* d;
  cudaMalloc(&d, 8 * G * J);
  const int smem = STAGES * (chunk + zbytes);
  cudaFuncSetAttribute(stream<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  stream<STAGES><<<G * J, 64, smem>>>(buf, units, chunk, stride, G, J, d, zbuf, zbytes);   // warm
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) stream<STAGES><<<G * J, 64, smem>>>(buf, units, chunk, stride, G, J, d, zbuf, zbytes);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)units * chunk * G;
  printf("%-34s chunk %6d stages %2d ctas %3d: %7.1f us  %7.1f GB/s %s\n", name, chunk, STAGES, G * J, ms * 1e3 / reps,
         bytes * reps / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  uint8_t* buf;
  const long long total = 400ll << 20;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  // C5 geometry: 12 blocks x 224 subchunks = 2688 units; 16 row groups of 512 rows (8 KB), 9 CTAs each
  go<8>("C5 pattern (stride 128 KB)", buf, 2688, 8192, 131072, 16, 9);
  go<13>("C5 pattern (stride 128 KB)", buf, 2688, 8192, 131072, 16, 9);
  go<24>("C5 pattern (stride 128 KB)", buf, 2688, 8192, 131072, 16, 9);
  go<8>("C5 bytes, contiguous per group", buf, 2688, 8192, 8192, 1, 144);
  go<8>("C5 pattern, 16 KB chunks", buf, 1344, 16384, 262144, 16, 9);
  go<8>("C5 pattern, 4 KB chunks", buf, 5376, 4096, 65536, 16, 9);
  go<8>("C5 pattern 148 CTAs (37 x 4)", buf, 2688, 8192, 131072, 16, 9);
  uint8_t* zq;
  cudaMalloc(&zq, 2688ll * 6656);
  cudaMemset(zq, 2, 2688ll * 6656);
  go<8>("C5 pattern + 6.5 KB Zq copy per unit", buf, 2688, 8192, 131072, 16, 9, zq, 6656);
  go<13>("C5 pattern + 6.5 KB Zq copy per unit", buf, 2688, 8192, 131072, 16, 9, zq, 6656);
  cudaFree(buf);
  return 0;
}
