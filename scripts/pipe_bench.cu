// Core-loop microbenchmark of decode_f8: 8 expander warps (2 warpgroups) expand signs to
// e4m3 in TMEM, one MMA warp issues 4 x kind::f8f6f4 (M128 N48 K32) per tile, pairs of
// tiles per elected region, NBUF A buffers per warpgroup.  No TMA (static smem operands).
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

template <int NBUF, int N, int EXPAND, int WAITS = 1>
__global__ void __launch_bounds__(320, 1) pipe(int tiles, long long* out) {
  __shared__ __align__(1024) uint8_t zs[128 * 48];
  __shared__ uint64_t a_full[8], a_empty[8], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(&a_full[i], 4); mbar_init(&a_empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t kAcc = 2 * NBUF * 32;
  long long t0 = clock64();
  if (warp < 8 && WAITS != 0) {
    const int wg = warp >> 2, qd = warp & 3;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    int ab = 0; uint32_t aph = 0;
    uint32_t w0 = 0x12345678u * (threadIdx.x + 1), w1 = w0 ^ 0x9e3779b9u, w2 = w0 * 3u, w3 = w1 * 5u;
    const uint32_t e8 = 0x38383838u ^ (uint32_t)(tiles & 0);  // runtime-opaque
    for (int t = wg; t < tiles; t += 2) {
      mbar_wait(&a_empty[wg * NBUF + ab], aph ^ 1);
      tc_fence_after();
      const uint32_t a_addr = tbase + lane_base + (uint32_t)(32 * (wg * NBUF + ab));
      uint32_t o[16];
      if (EXPAND) {
        expand_e4m3(w0, e8, o); expand_e4m3(w1, e8, o + 8);
      } else {
        for (int i = 0; i < 16; ++i) o[i] = e8;
      }
      tmem_st16(a_addr, o);
      if (EXPAND) { expand_e4m3(w2, e8, o); expand_e4m3(w3, e8, o + 8); }
      tmem_st16(a_addr + 16, o);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[wg * NBUF + ab]);
      if (++ab == NBUF) { ab = 0; aph ^= 1; }
      w0 = w0 * 1664525u + 1013904223u;
    }
  } else if (warp == 9) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(zs), (N / 8) * 128, 128);
    uint32_t ab0 = 0, ab1 = 0, aph0 = 0, aph1 = 0;
    long long wait_cycles = 0;
    for (int t = 0; t < tiles; t += 2) {
      const uint32_t slot0 = ab0, slot1 = NBUF + ab1;
      long long w0c = clock64();
      if (WAITS == 1 || WAITS == 3) { mbar_wait(&a_full[slot0], aph0); mbar_wait(&a_full[slot1], aph1); }
      if (WAITS == 2) { while (!mbar_test(&a_full[slot0], aph0)) {} while (!mbar_test(&a_full[slot1], aph1)) {} }
      if (lane == 0) wait_cycles += clock64() - w0c;
      tc_fence_after();
      const uint32_t d0 = tbase + kAcc + (uint32_t)((t & 1) * N);
      if (WAITS == 3) {  // dummy consumer: no MMA, release buffers immediately
        if (lane == 0) { mbar_arrive(&a_empty[slot0]); mbar_arrive(&a_empty[slot1]); }
      } else if (elect_one()) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          mma_f8_ts(d0, tbase + 32 * slot0 + 8 * m, bdesc0 + (uint64_t)((m * 2 * (N / 8) * 128) >> 4), idesc, m > 0);
        mma_commit(&a_empty[slot0]);
#pragma unroll
        for (int m = 0; m < 4; ++m)
          mma_f8_ts(d0 + N, tbase + 32 * slot1 + 8 * m, bdesc0 + (uint64_t)((m * 2 * (N / 8) * 128) >> 4), idesc, m > 0);
        mma_commit(&a_empty[slot1]);
        if (t + 2 >= tiles) mma_commit(&done);
      }
      __syncwarp();
      if (++ab0 == NBUF) { ab0 = 0; aph0 ^= 1; }
      if (++ab1 == NBUF) { ab1 = 0; aph1 ^= 1; }
    }
    if (WAITS != 3) mbar_wait(&done, 0);
    if (lane == 0) out[gridDim.x + blockIdx.x] = wait_cycles;
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 288) out[blockIdx.x] = t1 - t0;
  if (warp == 8) tmem_dealloc<512>(tbase);
}

template <int NBUF, int N, int EXPAND, int WAITS = 1>
void run(const char* name, int grid) {
  const int tiles = 4096;
  long long* d;
  cudaMalloc(&d, grid * 16);
  pipe<NBUF, N, EXPAND, WAITS><<<grid, 320>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
  printf("   [MMA warp time in a_full waits: %.1f cycles/tile]\n", (double)h[grid] / tiles);
  cudaFree(d);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-44s grid %3d: %7.1f cycles/tile  (%5.1f sign elements/clk/SM) %s\n", name, grid, mx / tiles,
         128.0 * 128.0 / (mx / tiles), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

extern "C" void run_all() {
  run<4, 48, 1, 0>("no expanders, no waits (MMA warp alone)", 1);
  run<4, 48, 1, 3>("NBUF 4/wg, expanders + dummy consumer (no MMA)", 1);
  run<4, 48, 0, 3>("NBUF 4/wg, STTM only + dummy consumer (no MMA)", 1);
  run<2, 48, 1>("NBUF 2/wg, N48, expand", 1);
  run<2, 48, 1>("NBUF 2/wg, N48, expand", 148);
  run<3, 48, 1>("NBUF 3/wg, N48, expand", 1);
  run<4, 48, 1>("NBUF 4/wg, N48, expand", 1);
  run<4, 48, 0>("NBUF 4/wg, N48, no expand (st only)", 1);
  run<2, 16, 1>("NBUF 2/wg, N16, expand", 1);
  run<4, 16, 1>("NBUF 4/wg, N16, expand", 1);
}
