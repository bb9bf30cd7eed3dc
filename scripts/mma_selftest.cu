// Micro self-test of tcgen05.mma kind::f16 (M=128, N=16, K=16): SS mode (A,B in
// SMEM) and TS mode (A stored to TMEM with tcgen05.st).  Debug tool, not product.
#include <cuda_fp16.h>
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

__global__ void mma_test(int mode, const __half* A, const __half* B, float* D, uint32_t* raw,
                         uint32_t idesc_override, int swap_lbo_sbo) {
  __shared__ __align__(1024) __half sA[128 * 16];
  __shared__ __align__(1024) __half sB[16 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // core-matrix layouts: (row, k) at ((k/8)*(ROWS/8) + row/8)*64 + (row%8)*8 + k%8   (halves)
  for (int e = tid; e < 128 * 16; e += blockDim.x) {
    int row = e / 16, k = e % 16;
    sA[((k / 8) * 16 + row / 8) * 64 + (row % 8) * 8 + k % 8] = A[e];
  }
  for (int e = tid; e < 16 * 16; e += blockDim.x) {
    int row = e / 16, k = e % 16;
    sB[((k / 8) * 2 + row / 8) * 64 + (row % 8) * 8 + k % 8] = B[e];
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  if (mode == 1) {  // TS: row = lane quadrant
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = 0;
    const int row = warp * 32 + lane;
    for (int c = 0; c < 8; ++c) {
      __half2 h = __halves2half2(A[row * 16 + 2 * c], A[row * 16 + 2 * c + 1]);
      v[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st16(t + ((uint32_t)(warp * 32) << 16) + 64, v);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_override ? idesc_override : idesc_f16_f32(128, 16);
    const uint32_t lboB = 2 * 128, sboB = 128;  // B: K-adjacent core matrices 256 B apart
    const uint32_t lboA = 16 * 128, sboA = 128;
    uint64_t bd = swap_lbo_sbo ? smem_desc_kmajor(smem_u32(sB), sboB, lboB) : smem_desc_kmajor(smem_u32(sB), lboB, sboB);
    if (mode == 1) {
      mma_f16_ts(t + 256, t + 64, bd, idesc, 0u);
    } else {
      uint64_t ad = swap_lbo_sbo ? smem_desc_kmajor(smem_u32(sA), sboA, lboA) : smem_desc_kmajor(smem_u32(sA), lboA, sboA);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t + 256),
          "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + 256, v);
    tmem_ld_wait();
    for (int c = 0; c < 16; ++c) D[(warp * 32 + lane) * 16 + c] = __uint_as_float(v[c]);
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + 64, v);
    tmem_ld_wait();
    for (int c = 0; c < 16; ++c) raw[(warp * 32 + lane) * 16 + c] = v[c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

extern "C" int run_mma_test(int mode, const void* A, const void* B, void* D, void* raw, unsigned idesc, int swap) {
  mma_test<<<1, 128>>>(mode, (const __half*)A, (const __half*)B, (float*)D, (uint32_t*)raw, idesc, swap);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
