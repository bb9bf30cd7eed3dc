// Throughput of the decode core loop without HBM: EWG warpgroups of expander warps write
// e4m3 A tiles into TMEM (tcgen05.st), one MMA warp consumes them in order with 4 x
// kind::f8f6f4 M128 N48 K32 TS MMAs per tile (or a dummy consumer), NBUF slots per warpgroup.
// Answers: is the expand+STTM side, the MMA side, or their TMEM contention the limit?
// Debug tool (scripts/ring_bench.py); not part of the library.
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// WAITMODE 0: every lane spins on try_wait; 1: lane 0 spins on try_wait, then __syncwarp;
// 2: lane 0 test_wait + nanosleep backoff, then __syncwarp
template <int WAITMODE>
__device__ __forceinline__ void wwait(uint64_t* bar, uint32_t parity) {
  if (WAITMODE == 0) {
    mbar_wait(bar, parity);
  } else if (WAITMODE == 1) {
    if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
    __syncwarp();
  } else if (WAITMODE == 2) {
    if ((threadIdx.x & 31) == 0) {
      while (!mbar_test(bar, parity)) __nanosleep(20);
    }
    __syncwarp();
  } else if (WAITMODE == 3) {
    while (!mbar_test(bar, parity)) {}
  } else {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(WAITMODE == 4 ? 20u : 1000u) : "memory");
    }
  }
}

__device__ long long* g_tr = nullptr;
template <int EWG, int NBUF, int EXPAND, int MMA, int WM>
__global__ void __launch_bounds__(32 * (4 * EWG + 1), 1) ring(int tiles, long long* out) {
  long long* tr = g_tr;
  __shared__ __align__(1024) uint8_t zs[128 * 48];
  __shared__ uint64_t a_full[16], a_empty[16], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) { mbar_init(&a_full[i], 4); mbar_init(&a_empty[i], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 4 * EWG) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t kAcc = EWG * NBUF * 32;
  static_assert(kAcc + EWG * 48 <= 512, "TMEM");
  long long t0 = clock64();
  if (warp < 4 * EWG) {
    const int wg = warp >> 2, qd = warp & 3;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    int ab = 0;
    uint32_t aph = 0;
    uint32_t w0 = 0x12345678u * (threadIdx.x + 1), w1 = w0 ^ 0x9e3779b9u, w2 = w0 * 3u, w3 = w1 * 5u;
    const uint32_t e8 = 0x38383838u ^ (uint32_t)(tiles & 0);
    for (int t = wg; t < tiles; t += EWG) {
      const long long c0 = clock64();
      wwait<WM>(&a_empty[wg * NBUF + ab], aph ^ 1);
      const long long c1 = clock64();
      tc_fence_after();
      uint32_t o[32];
      if (EXPAND) {
        expand_e4m3(w0, e8, o); expand_e4m3(w1, e8, o + 8); expand_e4m3(w2, e8, o + 16); expand_e4m3(w3, e8, o + 24);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = e8 + i;
      }
      tmem_st32(tbase + lane_base + (uint32_t)(32 * (wg * NBUF + ab)), o);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[wg * NBUF + ab]);
      const long long c2 = clock64();
      if (tr && lane == 0 && t < 256 && (warp & 3) == 0) {
        tr[t * 8 + 0] = c0 - t0; tr[t * 8 + 1] = c1 - t0; tr[t * 8 + 2] = c2 - t0;
      }
      if (++ab == NBUF) { ab = 0; aph ^= 1; }
      w0 = w0 * 1664525u + 1013904223u;
      w1 ^= w0;
    }
  } else {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(48 >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(zs), (48 / 8) * 128, 128);
    int ab[EWG];
    uint32_t aph[EWG];
    for (int w = 0; w < EWG; ++w) { ab[w] = 0; aph[w] = 0; }
    for (int t = 0; t < tiles; ++t) {
      const int wg = t % EWG;
      const int slot = wg * NBUF + ab[wg];
      const long long c0 = clock64();
      wwait<WM>(&a_full[slot], aph[wg]);
      const long long c1 = clock64();
      if (tr && lane == 0 && t < 256) { tr[t * 8 + 4] = c0 - t0; tr[t * 8 + 5] = c1 - t0; }
      tc_fence_after();
      if (!MMA) {
        if (lane == 0) mbar_arrive(&a_empty[slot]);
      } else if (elect_one()) {
        const uint32_t d0 = tbase + kAcc + (uint32_t)(wg * 48);
#pragma unroll
        for (int m = 0; m < 4; ++m)
          mma_f8_ts(d0, tbase + 32 * slot + 8 * m, bdesc0 + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4), idesc, m > 0);
        mma_commit(&a_empty[slot]);
        if (t + 1 >= tiles) mma_commit(&done);
      }
      __syncwarp();
      if (++ab[wg] == NBUF) { ab[wg] = 0; aph[wg] ^= 1; }
    }
    if (MMA) mbar_wait(&done, 0);
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 32 * 4 * EWG) out[blockIdx.x] = t1 - t0;
  if (warp == 4 * EWG) tmem_dealloc<512>(tbase);
}

// MMA warp alone: back-to-back TS MMAs from fixed slots, commit every 4 (no expanders).
__global__ void __launch_bounds__(32, 1) mma_alone(int tiles, long long* out) {
  __shared__ __align__(1024) uint8_t zs[128 * 48];
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(48 >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(zs), (48 / 8) * 128, 128);
  long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    if (elect_one()) {
#pragma unroll
      for (int m = 0; m < 4; ++m)
        mma_f8_ts(tbase + 256 + (t & 3) * 48, tbase + 32 * (t & 7) + 8 * m,
                  bdesc0 + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4), idesc, m > 0);
      if (t + 1 >= tiles) mma_commit(&done);
    }
    __syncwarp();
  }
  mbar_wait(&done, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncwarp();
  tmem_dealloc<512>(tbase);
}

// 16 warps: expand + STTM x32 (4 KB) per iteration, tcgen05.wait::st every WAIT_EVERY
// iterations (0: only at the end), no mbarriers.
template <int WAIT_EVERY, int EXPAND>
__global__ void __launch_bounds__(512, 1) sttm_loop(int tiles, long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t w0 = 0x12345678u * (threadIdx.x + 1), w1 = w0 ^ 0x9e3779b9u, w2 = w0 * 3u, w3 = w1 * 5u;
  const uint32_t e8 = 0x38383838u ^ (uint32_t)(tiles & 0);
  long long t0 = clock64();
  const int iters = tiles / 4;   // 16 warps x 4 KB = 4 tiles per iteration round
  for (int it = 0; it < iters; ++it) {
    uint32_t o[32];
    if (EXPAND) {
      expand_e4m3(w0, e8, o); expand_e4m3(w1, e8, o + 8); expand_e4m3(w2, e8, o + 16); expand_e4m3(w3, e8, o + 24);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = e8 + i;
    }
    tmem_st32(tbase + lane_base + (uint32_t)(32 * ((warp >> 2) * 4 + (it & 3))), o);
    if (WAIT_EVERY && (it % WAIT_EVERY) == WAIT_EVERY - 1) tmem_st_wait();
    w0 = w0 * 1664525u + 1013904223u;
    w1 ^= w0;
  }
  tmem_st_wait();
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// MMA issue rate with (STW = 1) / without (STW = 0) 16 warps streaming tcgen05.st (+ expansion)
// into other TMEM columns at the same time; no synchronisation between the two sides.
template <int STW, int NMMA>
__global__ void __launch_bounds__(544, 1) mma_vs_sttm(int tiles, long long* out) {
  __shared__ __align__(1024) uint8_t zs[128 * 48];
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  if (warp == 16) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(48 >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(zs), (48 / 8) * 128, 128);
  long long t0 = clock64();
  if (warp == 16) {
    for (int t = 0; t < tiles; ++t) {
      if (elect_one()) {
#pragma unroll
        for (int m = 0; m < NMMA; ++m)
          mma_f8_ts(tbase + 256 + (t & 3) * 48, tbase + 32 * (t & 3) + 8 * m,
                    bdesc0 + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4), idesc, m > 0);
        if (t + 1 >= tiles) mma_commit(&done);
      }
      __syncwarp();
    }
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 512) out[blockIdx.x] = t1 - t0;
  } else if (STW) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t w0 = 0x12345678u * (threadIdx.x + 1), w1 = w0 ^ 0x9e3779b9u, w2 = w0 * 3u, w3 = w1 * 5u;
    const uint32_t e8 = 0x38383838u ^ (uint32_t)(tiles & 0);
    for (int it = 0; it < tiles / 4; ++it) {
      uint32_t o[32];
      expand_e4m3(w0, e8, o); expand_e4m3(w1, e8, o + 8); expand_e4m3(w2, e8, o + 16); expand_e4m3(w3, e8, o + 24);
      tmem_st32(tbase + lane_base + (uint32_t)(128 + 32 * (warp >> 2)), o);   // columns 128..255
      tmem_st_wait();
      w0 = w0 * 1664525u + 1013904223u;
      w1 ^= w0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 16) tmem_dealloc<512>(tbase);
}

template <typename K>
void launch(K k, const char* name, int threads, int grid) {
  const int tiles = 4096;
  long long* d;
  cudaMalloc(&d, grid * 8);
  k<<<grid, threads>>>(tiles, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-58s grid %3d: %7.1f cycles/tile %s\n", name, grid, mx / tiles, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

extern "C" void run_trace() {
  long long* d; long long* tr;
  cudaMalloc(&d, 8);
  cudaMalloc(&tr, 256 * 8 * 8);
  cudaMemset(tr, 0, 256 * 64);
  cudaMemcpyToSymbol(g_tr, &tr, sizeof(tr));
  ring<4, 2, 1, 0, 0><<<1, 32 * 17>>>(1024, d);
  cudaDeviceSynchronize();
  long long h[256 * 8];
  cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tile: expander(wg=t%%4, warp 0): wait_start wait_done arrived | consumer: wait_start wait_done\n");
  for (int t = 100; t < 140; ++t)
    printf("%4d: %7lld %7lld %7lld | %7lld %7lld\n", t, h[t * 8], h[t * 8 + 1], h[t * 8 + 2], h[t * 8 + 4], h[t * 8 + 5]);
  long long z = 0;
  cudaMemcpyToSymbol(g_tr, &z, sizeof(z));
}

// One elected block of 16 MMAs (4 tiles x 4 K-steps) per iteration, alone or with 16 warps
// streaming tcgen05.st; DESC = 0: descriptors recomputed per MMA like the decode kernel
// (slot/stage arithmetic), 1: all 16 (a, b, d) operands precomputed in registers.
template <int STW, int DESC, int NCOMMIT = 0, int FENCE = 0>
__global__ void __launch_bounds__(544, 1) mma16(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t zs[4][128 * 48];
  __shared__ uint64_t done, cb[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < 4 * 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) { mbar_init(&done, 1); for (int c = 0; c < 4; ++c) mbar_init(&cb[c], 1); fence_mbar_init(); }
  if (warp == 16) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(48 >> 3) << 17) | ((128u >> 4) << 24);
  long long t0 = clock64();
  if (warp == 16) {
    uint64_t bd[4];
    for (int u = 0; u < 4; ++u) bd[u] = smem_desc_kmajor(smem_u32(zs[u]), (48 / 8) * 128, 128);
    for (int it = 0; it < iters; ++it) {
      if (FENCE == 1) tc_fence_after();
      if (FENCE == 2) { mbar_wait(&cb[3], 1); tc_fence_after(); }   // completed-phase wait + fence
      if (elect_one()) {
        if (DESC == 0) {
          for (int u = 0; u < 4; ++u) {
            const int st = (it * 4 + u) % 3;
            const uint64_t b0 = smem_desc_kmajor(smem_u32(zs[st]), (48 / 8) * 128, 128);
            const uint32_t a_col = tbase + 32 * ((it + u) & 3);
            const uint32_t d = tbase + 256 + u * 48;
#pragma unroll
            for (int m = 0; m < 4; ++m)
              mma_f8_ts(d, a_col + 8 * m, b0 + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4), idesc, m > 0 || it > 0);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int m = 0; m < 4; ++m)
              mma_f8_ts(tbase + 256 + u * 48, tbase + 32 * u + 8 * m, bd[u] + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4),
                        idesc, 1u);
        }
        for (int c = 0; c < NCOMMIT; ++c) mma_commit(&cb[c]);
        if (it + 1 >= iters) mma_commit(&done);
      }
      __syncwarp();
    }
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 512) out[blockIdx.x] = t1 - t0;
  } else if (STW) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t w0 = 0x12345678u * (threadIdx.x + 1), w1 = w0 ^ 0x9e3779b9u, w2 = w0 * 3u, w3 = w1 * 5u;
    const uint32_t e8 = 0x38383838u ^ (uint32_t)(iters & 0);
    for (int it = 0; it < iters; ++it) {
      if (STW == 2) {   // + a 16-byte LDS per thread per iteration from the operand area (signs)
        const uint4 v = reinterpret_cast<const uint4*>(&zs[0][0])[(threadIdx.x + it * 37) & 1535];
        w0 ^= v.x; w1 ^= v.y; w2 ^= v.z; w3 ^= v.w;
      }
      uint32_t o[32];
      expand_e4m3(w0, e8, o); expand_e4m3(w1, e8, o + 8); expand_e4m3(w2, e8, o + 16); expand_e4m3(w3, e8, o + 24);
      tmem_st32(tbase + lane_base + (uint32_t)(128 + 32 * (warp >> 2)), o);
      tmem_st_wait();
      w0 = w0 * 1664525u + 1013904223u;
      w1 ^= w0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 16) tmem_dealloc<512>(tbase);
}

// Does writing an A slot with tcgen05.st right before the MMAs that read it slow the MMAs?
// 4 warps (one per lane quadrant) write slot (it % NS) each iteration, sync on a named barrier,
// warp 0 issues 4 MMAs from that slot (SAME = 1) or from a never-written slot (SAME = 0).
template <int SAME, int NS>
__global__ void __launch_bounds__(128, 1) st_then_mma(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t zs[128 * 48];
  __shared__ uint64_t done, slot_free[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < 128 * 48 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) { mbar_init(&done, 1); for (int i = 0; i < 8; ++i) mbar_init(&slot_free[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(48 >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t bd = smem_desc_kmajor(smem_u32(zs), (48 / 8) * 128, 128);
  uint32_t o[32];
  for (int e = 0; e < 32; ++e) o[e] = 0x38383838u + e;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int sl = it % NS;
    if (it >= NS) mbar_wait(&slot_free[sl], (uint32_t)(((it / NS) - 1) & 1));
    tc_fence_after();
    tmem_st32(tbase + 32 * sl + lane_base, o);
    tmem_st_wait();
    tc_fence_before();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a = SAME ? tbase + 32 * sl : tbase + 32 * 7;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          mma_f8_ts(tbase + 256, a + 8 * m, bd + (uint64_t)((m * 2 * (48 / 8) * 128) >> 4), idesc, 1u);
        mma_commit(&slot_free[sl]);
        if (it + 1 >= iters) mma_commit(&done);
      }
      __syncwarp();
    }
  }
  if (warp == 0) mbar_wait(&done, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

extern "C" void run_stmma() {
  const int iters = 2048;
  auto go = [&](auto k, const char* name) {
    long long* d; long long h;
    cudaMalloc(&d, 8);
    k<<<1, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    printf("%-58s %7.1f cycles per iteration (4 MMAs) %s\n", name, h / (double)iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  go(st_then_mma<1, 2>, "STTM slot -> MMAs read it (2 slots)");
  go(st_then_mma<0, 2>, "STTM slot, MMAs read another slot (2 slots)");
  go(st_then_mma<1, 4>, "STTM slot -> MMAs read it (4 slots)");
  go(st_then_mma<0, 4>, "STTM slot, MMAs read another slot (4 slots)");
}

extern "C" void run_mma16() {
  const int iters = 1024;
  auto go = [&](auto k, const char* name) {
    long long* d; long long h;
    cudaMalloc(&d, 8);
    k<<<1, 544>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    printf("%-60s %7.1f cycles per 16-MMA block (%5.1f per MMA) %s\n", name, h / (double)iters, h / (16.0 * iters),
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  go(mma16<0, 0>, "16 MMAs/block, per-MMA descriptor math, alone");
  go(mma16<0, 1>, "16 MMAs/block, precomputed descriptors, alone");
  go(mma16<1, 0>, "16 MMAs/block, per-MMA descriptor math, + 16 STTM warps");
  go(mma16<1, 1>, "16 MMAs/block, precomputed descriptors, + 16 STTM warps");
  go(mma16<1, 1, 1>, "  ... + 1 commit per block");
  go(mma16<1, 1, 3>, "  ... + 3 commits per block");
  go(mma16<0, 1, 3>, "16 MMAs/block, precomputed, alone, 3 commits per block");
  go(mma16<0, 1, 3, 1>, "  alone, 3 commits + fence::after_thread_sync per block");
  go(mma16<0, 1, 3, 2>, "  alone, 3 commits + completed mbar wait + fence per block");
  go(mma16<1, 1, 3, 1>, "  + STTM warps, 3 commits + fence per block");
  go(mma16<2, 1, 3, 1>, "  + STTM warps with LDS.128, 3 commits + fence per block");
}

extern "C" void run_contention() {
  launch(mma_vs_sttm<0, 4>, "MMA warp alone (4 MMAs/tile)", 544, 1);
  launch(mma_vs_sttm<1, 4>, "MMA warp + 16 warps expand+STTM (no sync)", 544, 1);
  launch(mma_vs_sttm<0, 1>, "MMA warp alone (1 MMA/tile)", 544, 1);
  launch(mma_vs_sttm<1, 1>, "1 MMA/tile + 16 warps expand+STTM", 544, 1);
}

extern "C" void run_all() {
  launch(mma_alone, "MMA warp alone (4 TS MMAs/tile, N48)", 32, 1);
  launch(ring<4, 2, 1, 0, 0>, "16 exp, dummy consumer, all-lane try_wait", 32 * 17, 1);
  launch(ring<4, 2, 1, 0, 1>, "16 exp, dummy consumer, lane-0 try_wait", 32 * 17, 1);
  launch(ring<4, 2, 1, 0, 2>, "16 exp, dummy consumer, lane-0 test+sleep", 32 * 17, 1);
  launch(ring<4, 2, 1, 1, 0>, "16 exp + MMA, all-lane try_wait", 32 * 17, 1);
  launch(ring<4, 2, 1, 1, 1>, "16 exp + MMA, lane-0 try_wait", 32 * 17, 1);
  launch(ring<4, 2, 1, 1, 2>, "16 exp + MMA, lane-0 test+sleep", 32 * 17, 1);
  launch(ring<4, 2, 0, 1, 1>, "16 STTM-only + MMA, lane-0 try_wait", 32 * 17, 1);
  launch(ring<2, 4, 1, 1, 1>, "8 exp NBUF 4 + MMA, lane-0 try_wait", 32 * 9, 1);
  launch(ring<4, 2, 1, 0, 3>, "16 exp, dummy consumer, all-lane test_wait spin", 32 * 17, 1);
  launch(ring<4, 2, 1, 0, 4>, "16 exp, dummy consumer, try_wait hint 20ns", 32 * 17, 1);
  launch(ring<4, 2, 1, 0, 5>, "16 exp, dummy consumer, try_wait hint 1000ns", 32 * 17, 1);
  launch(ring<4, 2, 1, 1, 3>, "16 exp + MMA, all-lane test_wait spin", 32 * 17, 1);
  launch(ring<4, 2, 1, 1, 4>, "16 exp + MMA, try_wait hint 20ns", 32 * 17, 1);
  launch(sttm_loop<0, 1>, "16 warps expand+STTM, wait::st at end", 512, 1);
  launch(sttm_loop<1, 1>, "16 warps expand+STTM, wait::st every tile", 512, 1);
  launch(sttm_loop<2, 1>, "16 warps expand+STTM, wait::st every 2", 512, 1);
  launch(sttm_loop<4, 1>, "16 warps expand+STTM, wait::st every 4", 512, 1);
  launch(sttm_loop<1, 0>, "16 warps STTM only, wait::st every tile", 512, 1);
  launch(sttm_loop<0, 0>, "16 warps STTM only, wait::st at end", 512, 1);
}
