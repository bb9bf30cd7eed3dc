// Microbenchmarks for the decode-kernel pipeline primitives on sm_100a (debug tool):
//   mode 0: STTM.x16 x4 + wait::st per iteration, 4 warps (one warpgroup)        -> cycles / iter
//   mode 1: 8 x tcgen05.mma (M128 N16 K16, A in TMEM) + commit + wait, 1 thread  -> round-trip cycles
//   mode 2: same as 1 but NGRP groups in flight before waiting                    -> cycles / group
//   mode 3: ping-pong: 4 expander warps (STTM only) <-> MMA warp, NBUF buffers    -> cycles / tile
#include <cuda_fp16.h>
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

__global__ void __launch_bounds__(192, 1) micro(int mode, int iters, int nbuf, long long* out) {
  __shared__ __align__(1024) uint8_t zs[4096];
  __shared__ uint64_t bars[32];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < 4096 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x3C003C00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) mbar_init(&bars[i], i < 8 ? 4 : 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  const uint64_t bdesc = smem_desc_kmajor(smem_u32(zs), 256, 128);
  const uint32_t idesc = idesc_f16_f32(128, 16);
  long long t0 = clock64();
  if (mode == 0) {
    if (warp < 4) {
      uint32_t v[16];
      for (int c = 0; c < 16; ++c) v[c] = 0x3C003C00u ^ (lane + c);
      for (int it = 0; it < iters; ++it) {
        const uint32_t a = t + ((uint32_t)(warp * 32) << 16) + 64 * (it & 3);
        tmem_st16(a, v); tmem_st16(a + 16, v); tmem_st16(a + 32, v); tmem_st16(a + 48, v);
        tmem_st_wait();
      }
    }
  } else if (mode == 1 || mode == 2) {
    if (warp == 4) {
      const int grp = mode == 1 ? 1 : nbuf;
      uint32_t ph = 0;
      for (int it = 0; it < iters; ++it) {
        if (elect_one()) {
          for (int g = 0; g < grp; ++g) {
            for (int m = 0; m < 8; ++m) mma_f16_ts(t + 256 + 16 * g, t + 64 * (g & 3) + 8 * m, bdesc, idesc, m > 0);
          }
          mma_commit(&bars[8]);
        }
        __syncwarp();
        mbar_wait(&bars[8], ph);
        ph ^= 1;
      }
    }
  } else if (mode == 4 || mode == 5) {
    // mode 4: MMA warp: wait(always-complete barrier) + 8 MMA + commit per iteration
    // mode 5: MMA warp: 8 MMA + commit per iteration, no waits (issue throughput); nbuf = N/16
    if (warp == 4) {
      if (threadIdx.x == 128) { mbar_arrive(&bars[9]); }  // bars[9] count 1 -> phase 0 completes
      __syncwarp();
      const uint32_t id = idesc_f16_f32(128, 16 * (nbuf > 0 ? nbuf : 1));
      for (int it = 0; it < iters; ++it) {
        if (mode == 4) mbar_wait(&bars[9], 0);
        tc_fence_after();
        if (elect_one()) {
          for (int m = 0; m < 8; ++m) mma_f16_ts(t + 256, t + 64 * (it & 3) + 8 * m, bdesc, id, m > 0);
          mma_commit(&bars[10]);
        }
        __syncwarp();
      }
      mbar_wait(&bars[10], (iters - 1) & 1);
    }
  } else if (mode == 6) {
    // SS mode: A from SMEM (zs as A too), 8 MMA + commit, no waits; nbuf = N/16
    if (warp == 4) {
      const uint32_t id = idesc_f16_f32(128, 16 * (nbuf > 0 ? nbuf : 1));
      const uint64_t adesc = smem_desc_kmajor(smem_u32(zs), 128 * 16, 128);
      for (int it = 0; it < iters; ++it) {
        if (elect_one()) {
          for (int m = 0; m < 8; ++m) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t + 256),
                         "l"(adesc), "l"(bdesc), "r"(id), "r"((uint32_t)(m > 0)));
          }
          mma_commit(&bars[10]);
        }
        __syncwarp();
      }
      mbar_wait(&bars[10], (iters - 1) & 1);
    }
  } else if (mode == 7 || mode == 8 || mode == 9) {
    // mode 7: kind::f8f6f4 (e4m3 x e4m3 -> f32), K=32, N = 16*nbuf, TS, 8 MMA + commit
    // mode 8: kind::i8 (u8 x s8 -> s32), K=32, N = 16*nbuf, TS, 8 MMA + commit
    // mode 9: kind::f16 N16, commit only every 4 groups
    if (warp == 4) {
      const uint32_t N = 16 * (nbuf > 0 ? nbuf : 1);
      uint32_t id;
      if (mode == 7) id = (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
      else if (mode == 8) id = (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
      else id = idesc_f16_f32(128, 16);
      for (int it = 0; it < iters; ++it) {
        if (elect_one()) {
          for (int m = 0; m < 8; ++m) {
            const uint32_t a = t + 64 * (it & 3) + 8 * m, d = t + 256;
            const uint32_t en = m > 0;
            if (mode == 7)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                           "l"(bdesc), "r"(id), "r"(en));
            else if (mode == 8)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                           "l"(bdesc), "r"(id), "r"(en));
            else
              mma_f16_ts(d, a, bdesc, id, en);
          }
          if (mode != 9 || (it & 3) == 3) mma_commit(&bars[10]);
        }
        __syncwarp();
      }
      if (mode != 9) mbar_wait(&bars[10], (iters - 1) & 1);
      else mbar_wait(&bars[10], (iters / 4 - 1) & 1);
    }
  } else if (mode == 3) {
    // bars[0..nbuf) a_full (count 4), bars[8..8+nbuf) a_empty (count 1)
    if (warp < 4) {
      uint32_t v[16];
      for (int c = 0; c < 16; ++c) v[c] = 0x3C003C00u;
      int ab = 0; uint32_t aph = 0;
      for (int it = 0; it < iters; ++it) {
        mbar_wait(&bars[8 + ab], aph ^ 1);
        tc_fence_after();
        const uint32_t a = t + ((uint32_t)(warp * 32) << 16) + 64 * ab;
        tmem_st16(a, v); tmem_st16(a + 16, v); tmem_st16(a + 32, v); tmem_st16(a + 48, v);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[ab]);
        if (++ab == nbuf) { ab = 0; aph ^= 1; }
      }
    } else if (warp == 4) {
      int ab = 0; uint32_t aph = 0;
      for (int it = 0; it < iters; ++it) {
        mbar_wait(&bars[ab], aph);
        tc_fence_after();
        if (elect_one()) {
          for (int m = 0; m < 8; ++m) mma_f16_ts(t + 448, t + 64 * ab + 8 * m, bdesc, idesc, m > 0);
          mma_commit(&bars[8 + ab]);
        }
        __syncwarp();
        if (++ab == nbuf) { ab = 0; aph ^= 1; }
      }
    }
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 || threadIdx.x == 128) out[blockIdx.x * 2 + (threadIdx.x ? 1 : 0)] = t1 - t0;
  if (warp == 0) tmem_dealloc<512>(t);
}

extern "C" int run_micro(int mode, int iters, int nbuf, int grid, long long* host_out) {
  long long* d;
  cudaMalloc(&d, grid * 2 * sizeof(long long));
  micro<<<grid, 192>>>(mode, iters, nbuf, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(host_out, d, grid * 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return 0;
}
