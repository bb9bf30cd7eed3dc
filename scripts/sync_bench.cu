// Cost breakdown of the expander loop's synchronisation (one warpgroup = 4 warps, 1 CTA).
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;

template <int V, int NW = 4>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* out) {
  __shared__ uint64_t bar_done, bar_free;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar_done, NW); mbar_init(&bar_free, 1); mbar_arrive(&bar_free); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16) + 128 * (warp >> 2);
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1);
  const uint32_t e8 = 0x38383838u ^ (uint32_t)(iters & 0);
  long long t0 = clock64();
  __shared__ __align__(16) uint32_t sbuf[4][4096];
  uint32_t acc13 = 0;
  for (int it = 0; it < iters; ++it) {
    if (V == 13) {  // STTM of constant regs + independent expansion (XOR-reduced, not stored)
      uint32_t c16[16], o32[32];
      for (int i = 0; i < 16; ++i) c16[i] = e8 + i;
      tmem_st16(tb + 32 * (it & 3), c16);
      tmem_st16(tb + 32 * (it & 3) + 16, c16);
      expand_e4m3(w, e8, o32); expand_e4m3(w ^ 0x55u, e8, o32 + 8);
      expand_e4m3(w * 3u, e8, o32 + 16); expand_e4m3(w * 5u, e8, o32 + 24);
      for (int i = 0; i < 32; ++i) acc13 ^= o32[i];
      w = w * 1664525u + 1013904223u + acc13;
      continue;
    }
    if (V == 14) {  // expansion stored to SMEM with STS.128 (SS-mode A operand)
      uint32_t o32[32];
      expand_e4m3(w, e8, o32); expand_e4m3(w ^ 0x55u, e8, o32 + 8);
      expand_e4m3(w * 3u, e8, o32 + 16); expand_e4m3(w * 5u, e8, o32 + 24);
      uint4* dst = reinterpret_cast<uint4*>(&sbuf[it & 3][0]) + (threadIdx.x & 127);
      for (int i = 0; i < 8; ++i) dst[i * 128 % 1024] = make_uint4(o32[4 * i], o32[4 * i + 1], o32[4 * i + 2], o32[4 * i + 3]);
      w = w * 1664525u + 1013904223u;
      continue;
    }
    if (V >= 10) {  // expand all 4 words into 32 registers, one STTM.x32
      uint32_t o32[32];
      expand_e4m3(w, e8, o32); expand_e4m3(w ^ 0x55u, e8, o32 + 8);
      expand_e4m3(w * 3u, e8, o32 + 16); expand_e4m3(w * 5u, e8, o32 + 24);
      tmem_st32(tb + 32 * (it & 3), o32);
      if (V >= 11) tmem_st_wait();
      if (V >= 12) { tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&bar_done); mbar_wait(&bar_free, 0); tc_fence_after(); }
      w = w * 1664525u + 1013904223u;
      continue;
    }
    uint32_t o[16];
    if (V >= 1 && V != 9 || V == 9) { expand_e4m3(w, e8, o); expand_e4m3(w ^ 0x55u, e8, o + 8); }
    else { for (int i = 0; i < 16; ++i) o[i] = w + i; }
    if (V != 9) tmem_st16(tb + 32 * (it & 3), o);
    else { uint32_t acc = 0; for (int i = 0; i < 16; ++i) acc ^= o[i]; w ^= acc; }
    if (V >= 1) { expand_e4m3(w * 3u, e8, o); expand_e4m3(w * 5u, e8, o + 8); }
    if (V != 9) tmem_st16(tb + 32 * (it & 3) + 16, o);
    else { uint32_t acc = 0; for (int i = 0; i < 16; ++i) acc ^= o[i]; w ^= acc; }
    if (V >= 2) tmem_st_wait();
    if (V >= 3) { tc_fence_before(); __syncwarp(); }
    if (V >= 4 && lane == 0) mbar_arrive(&bar_done);              // arrive (phase completes every iteration)
    if (V >= 5) { mbar_wait(&bar_free, 0); tc_fence_after(); }    // wait on an already-complete phase
    w = w * 1664525u + 1013904223u;
  }
  if (V < 2) tmem_st_wait();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0 + (acc13 == 0x12345 ? 1 : 0) + (V == 14 ? (long long)(sbuf[0][5] & 0) : 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

template <int V, int NW = 4>
void run(const char* name) {
  long long* d; long long h;
  cudaMalloc(&d, 8);
  k<V, NW><<<1, NW * 32>>>(4096, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  printf("%-60s %7.1f cycles/iter %s\n", name, h / 4096.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

extern "C" void run_all() {
  run<13, 4>("STTM(const) + independent expand, 4 warps");
  run<13, 8>("STTM(const) + independent expand, 8 warps");
  run<14, 4>("expand + STS.128 to smem, 4 warps");
  run<14, 8>("expand + STS.128 to smem, 8 warps");
  run<10>("x32: expand 32 regs + 1 STTM.x32, 4 warps");
  run<10, 8>("x32: expand 32 regs + 1 STTM.x32, 8 warps");
  run<11, 8>("x32: + wait::st, 8 warps");
  run<12, 8>("x32: + full sync, 8 warps");
  run<12, 16>("x32: + full sync, 16 warps");
  run<0>("2 x STTM.x16 (no expand, no wait)");
  run<0, 8>("8 warps: 2 x STTM.x16 only");
  run<9>("expand only (no STTM), 4 warps");
  run<9, 8>("expand only (no STTM), 8 warps");
  run<1, 8>("8 warps: expand + 2 STTM (per warp-iteration)");
  run<1, 16>("16 warps: expand + 2 STTM (per warp-iteration)");
  run<5, 8>("8 warps: full sync loop");
  run<5, 16>("16 warps: full sync loop");
  run<1>("+ expand 4 words");
  run<2>("+ tcgen05.wait::st");
  run<3>("+ tcgen05.fence::before + syncwarp");
  run<4>("+ mbarrier.arrive");
  run<5>("+ try_wait(complete phase) + fence::after");
}
