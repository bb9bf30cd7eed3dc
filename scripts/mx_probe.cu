// Probe of tcgen05.mma kind::mxf8f6f4.block_scale with A read from TMEM (round-2 decode
// operand format): (1) does the TS form run and give A*B*2^(sfa+sfb)?  (2) which TMEM cell
// (lane, column, byte) holds the scale of row m / column n?  (3) does tcgen05.cp
// 32x128b.warpx4 from the CUTLASS SF chunk layout feed it?  (4) random exactness test over
// 4 K-blocks with per-(column, K-block) scales.  (5) throughput vs kind::f8f6f4 / i8, N.
// Standalone (main), build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp8.h>
#include "../paper_2410_23918_b200/csrc/ptx.cuh"
using namespace bs;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__host__ __device__ constexpr uint32_t idesc_mx(uint32_t M, uint32_t N, uint32_t asf, uint32_t bsf) {
  return (bsf << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24) | (asf << 29);
}
__device__ __forceinline__ void mma_mx_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void utccp_32x128b_x4(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// B tile (N x K=128 e4m3, K-major, no swizzle): (n, k) at ((k/16)*(N/8) + n/8)*128 + (n%8)*16 + k%16
__host__ __device__ inline int boff(int n, int k, int N) { return ((k / 16) * (N / 8) + n / 8) * 128 + (n % 8) * 16 + k % 16; }

constexpr int COL_A = 0, COL_SFA = 64, COL_SFB = 72, COL_D = 128;

// mode 0: SFA=SFB=127.  1: SFA cell (L,c) = 40 + L%32 + 32c.  2: SFA cell = 40 + L.  3/4 same for SFB.
// 5: random test: A, B from global (K=128 = 4 K-blocks), scales via tcgen05.cp from the CUTLASS chunk.
template <int N>
__global__ void probe(int mode, const uint8_t* gA, const uint8_t* gB, const uint8_t* gsfa, const uint8_t* gsfb,
                      float* D) {
  __shared__ __align__(1024) uint8_t sB[N * 128];
  __shared__ __align__(128) uint8_t sSFA[512];
  __shared__ __align__(128) uint8_t sSFB[512];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < N * 128; e += blockDim.x) {
    const int n = e / 128, k = e % 128;
    sB[boff(n, k, N)] = gB ? gB[n * 128 + k] : 0x38;
  }
  for (int e = tid; e < 512; e += blockDim.x) {
    sSFA[e] = gsfa ? gsfa[e] : 127;
    sSFB[e] = gsfb ? gsfb[e] : 127;
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  const int row = warp * 32 + lane;
  const uint32_t lq = (uint32_t)(warp * 32) << 16;
  {  // A: 32 columns (K = 128)
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) {
      uint32_t w = 0x38383838u;
      if (gA) w = gA[row * 128 + 4 * c] | (gA[row * 128 + 4 * c + 1] << 8) | (gA[row * 128 + 4 * c + 2] << 16) |
                  ((uint32_t)gA[row * 128 + 4 * c + 3] << 24);
      v[c] = w;
    }
    tmem_st32(t + lq + COL_A, v);
    uint32_t s[16];
    for (int c = 0; c < 4; ++c) {
      uint32_t va = 127, vb = 127;
      if (mode == 1) va = 40 + (row % 32) + 32 * c;
      if (mode == 2) va = 40 + row;
      if (mode == 3) vb = 40 + (row % 32) + 32 * c;
      if (mode == 4) vb = 40 + row;
      s[c] = va * 0x01010101u;
      s[4 + c] = vb * 0x01010101u;
    }
    for (int c = 8; c < 16; ++c) s[c] = 0;
    if (mode != 5) tmem_st16(t + lq + COL_SFA, s);  // cols SFA..SFA+3 = SFA cells, SFB..SFB+3 = SFB cells
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    if (mode == 5) {
      utccp_32x128b_x4(t + COL_SFA, smem_desc_kmajor(smem_u32(sSFA), 128, 128));
      utccp_32x128b_x4(t + COL_SFB, smem_desc_kmajor(smem_u32(sSFB), 128, 128));
    }
    const uint32_t LBO = (N / 8) * 128, SBO = 128;
    const int nkb = mode == 5 ? 4 : 1;
    for (int kb = 0; kb < nkb; ++kb) {
      const uint64_t bd = smem_desc_kmajor(smem_u32(sB + kb * 2 * (N / 8) * 128), LBO, SBO);
      const uint32_t sf = mode == 5 ? (uint32_t)kb : 0u;
      mma_mx_ts(t + COL_D, t + COL_A + 8 * kb, bd, idesc_mx(128, N, sf, sf), t + COL_SFA + (sf << 30),
                t + COL_SFB + (sf << 30), kb > 0 ? 1u : 0u);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c0 = 0; c0 < N; c0 += 32) {
    tmem_ld32(t + lq + COL_D + c0, v);
    tmem_ld_wait();
    for (int c = 0; c < 32 && c0 + c < N; ++c) D[row * N + c0 + c] = __uint_as_float(v[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

static double e4m3_to_double(uint8_t b) {
  const int s = b >> 7, e = (b >> 3) & 15, m = b & 7;
  double v = e == 0 ? ldexp((double)m, -9) : ldexp(1.0 + m / 8.0, e - 7);
  return s ? -v : v;
}

template <int N>
void run_layout() {
  float* dD;
  CK(cudaMalloc(&dD, 128 * N * 4));
  std::vector<float> D(128 * N);
  for (int mode = 0; mode < 0; ++mode) {  // tcgen05.st-written scale probes retired: mode 5 pins the layout
    probe<N><<<1, 128>>>(mode, nullptr, nullptr, nullptr, nullptr, dD);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    printf("N=%d mode %d: D[0,0]=%g D[127,N-1]=%g\n", N, mode, D[0], D[127 * N + N - 1]);
    if (mode == 0) continue;
    // decode exponent per row (mode 1,2) or per column (3,4)
    const bool rows = mode <= 2;
    const int cnt = rows ? 128 : N;
    printf("  %s -> scale value:", rows ? "row m" : "col n");
    for (int i = 0; i < cnt; ++i) {
      const float d = rows ? D[i * N + 0] : D[0 * N + i];
      const int val = (int)lround(log2(d / 32.0)) + 127;
      if (i % 16 == 0) printf("\n   [%3d]", i);
      printf(" %3d", val);
    }
    printf("\n");
    // also: is D constant along the other axis?
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        const float ref = rows ? D[m * N] : D[n];
        if (D[m * N + n] != ref) ++bad;
      }
    printf("  cells differing from the row/col value: %d\n", bad);
  }
  // mode 5: random exactness test
  std::vector<uint8_t> A(128 * 128), B(N * 128), sfa(512), sfb(512);
  srand(1234);
  for (auto& a : A) a = (rand() & 1) ? 0xB8 : 0x38;  // +-1
  for (auto& b : B) {
    uint8_t x;
    do { x = rand() & 0xFF; } while ((x & 0x7F) == 0x7F);  // no NaN
    b = x;
  }
  std::vector<int> SA(128 * 4), SB(N * 4);
  for (int m = 0; m < 128; ++m)
    for (int kb = 0; kb < 4; ++kb) { SA[m * 4 + kb] = 127; }
  for (int n = 0; n < N; ++n)
    for (int kb = 0; kb < 4; ++kb) SB[n * 4 + kb] = 127 - 20 + rand() % 40;
  // CUTLASS chunk: offset(m, kb) = 16 (m%32) + 4 (m/32) + kb
  for (int m = 0; m < 128; ++m)
    for (int kb = 0; kb < 4; ++kb) sfa[16 * (m % 32) + 4 * (m / 32) + kb] = SA[m * 4 + kb];
  for (int i = 0; i < 512; ++i) sfb[i] = 127;
  for (int n = 0; n < N && n < 128; ++n)
    for (int kb = 0; kb < 4; ++kb) sfb[16 * (n % 32) + 4 * (n / 32) + kb] = SB[n * 4 + kb];
  uint8_t *dA, *dB, *dsa, *dsb;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dsa, 512));
  CK(cudaMalloc(&dsb, 512));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsa, sfa.data(), 512, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsb, sfb.data(), 512, cudaMemcpyHostToDevice));
  probe<N><<<1, 128>>>(5, dA, dB, dsa, dsb, dD);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0;
  int nbad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < 128; ++k) {
        const int kb = k / 32;
        const double p = e4m3_to_double(A[m * 128 + k]) * e4m3_to_double(B[n * 128 + k]) *
                         ldexp(1.0, SA[m * 4 + kb] - 127 + SB[n * 4 + kb] - 127);
        ref += p;
        mag += fabs(p);
      }
      const double err = fabs(D[m * N + n] - ref) / (mag > 0 ? mag : 1);
      if (err > maxrel) maxrel = err;
      if (err > 1e-6) ++nbad;
    }
  printf("N=%d mode 5 (tcgen05.cp scales, 4 K-blocks, random B, +-1 A): max |D-ref|/sum|p| = %.3e, bad=%d\n", N,
         maxrel, nbad);
  cudaFree(dA); cudaFree(dB); cudaFree(dsa); cudaFree(dsb); cudaFree(dD);
}

// ---------------------------------------------------------------- throughput
// KIND 0 f8f6f4 e4m3, 1 mxf8f6f4 block_scale, 2 i8.  STALL: warps 4..7 stream tcgen05.st.
template <int KIND, int N, int STALL, int NACC = 1, int DEPTH = 2, int PER = 8>
__global__ void __launch_bounds__(512, 1) thr(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t zs[256 * 32 * 2];
  __shared__ uint64_t bars[DEPTH];
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < (int)sizeof(zs) / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(zs)[e] = 0x38383838u;
  if (threadIdx.x == 0) { for (int b = 0; b < DEPTH; ++b) mbar_init(&bars[b], 1); fence_mbar_init(); done = 0; }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  const uint64_t bdesc = smem_desc_kmajor(smem_u32(zs), (N / 8) * 128, 128);
  long long t0 = clock64();
  long long nst = 0;
  if (warp == 1) {
    for (int it = 0; it < iters; ++it) {
      if (it >= DEPTH) mbar_wait(&bars[it % DEPTH], ((it - DEPTH) / DEPTH) & 1);  // batch it-DEPTH done
      if (elect_one()) {
#pragma unroll
        for (int m = 0; m < PER; ++m) {
          const uint32_t dcol = 256 + (NACC > 1 ? (m % NACC) * N : 0);
          const uint32_t a = t + 8 * ((m / NACC) % 8) + 64 * (m % NACC);
          if constexpr (KIND == 0) {
            constexpr uint32_t id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
            mma_f8_ts(t + dcol, a, bdesc, id, m >= NACC ? 1u : 0u);
          } else if constexpr (KIND == 1) {
            mma_mx_ts(t + dcol, a, bdesc, idesc_mx(128, N, 0, 0), t + 128, t + 136, m >= NACC ? 1u : 0u);
          } else {
            constexpr uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t + dcol), "r"(a),
                         "l"(bdesc), "r"(id), "r"(m >= NACC ? 1u : 0u));
          }
        }
        mma_commit(&bars[it % DEPTH]);
      }
      __syncwarp();
    }
    for (int j = iters - DEPTH; j < iters; ++j) if (j >= 0) mbar_wait(&bars[j % DEPTH], (j / DEPTH) & 1);
    if (threadIdx.x == 32) done = 1;
  } else if (STALL && warp >= 4) {
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = 0x38383838u ^ (threadIdx.x * c);
    const uint32_t lq = (uint32_t)((warp & 3) * 32) << 16;
    while (!done) {
      tmem_st32(t + lq + 448 + 32 * ((int)nst & 1), v);
      tmem_st_wait();
      ++nst;
    }
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 32) out[0] = t1 - t0;
  if (threadIdx.x == 128) out[1] = nst;
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int KIND, int N, int STALL, int NACC = 1, int DEPTH = 2, int PER = 8>
void run_thr(const char* name) {
  long long* d;
  long long h[2] = {0, 0};
  CK(cudaMalloc(&d, 16));
  CK(cudaMemset(d, 0, 16));
  const int iters = 2000;
  thr<KIND, N, STALL, NACC, DEPTH, PER><<<1, STALL == 2 ? 512 : 256>>>(iters, d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  cudaFree(d);
  const double cyc = (double)h[0] / iters / PER;
  printf("%-12s depth=%d per=%2d nacc=%d N=%3d stall=%d: %6.1f cycles/MMA (floor N/2 = %5.1f)  sttm/warp=%lld (%.0f B/cyc/SM)\n", name, DEPTH, PER, NACC, N,
         STALL, cyc, N / 2.0, h[1], STALL ? (double)h[1] * (STALL == 2 ? 12 : 4) * 4096 / h[0] : 0.0);
}

int main() {
  run_thr<1, 48, 0, 1, 1, 8>("mx lat");
  run_thr<1, 48, 0, 1, 1, 1>("mx lat1");
  run_thr<1, 48, 0, 1, 2, 8>("mxf8f6f4");
  run_thr<1, 48, 0, 1, 4, 8>("mxf8f6f4");
  run_thr<1, 48, 0, 1, 8, 8>("mxf8f6f4");
  run_thr<1, 48, 0, 4, 8, 8>("mxf8f6f4");
  run_thr<1, 48, 0, 1, 4, 32>("mxf8f6f4");
  run_thr<1, 32, 0, 1, 8, 8>("mxf8f6f4");
  run_thr<1, 32, 0, 1, 4, 32>("mxf8f6f4");
  run_thr<1, 16, 0, 1, 4, 32>("mxf8f6f4");
  run_thr<1, 96, 0, 1, 4, 32>("mxf8f6f4");
  run_thr<0, 48, 0, 1, 4, 32>("f8f6f4");
  run_thr<2, 32, 0, 1, 4, 32>("i8");
  run_thr<1, 48, 2, 1, 4, 32>("mxf8f6f4");
  run_thr<1, 32, 2, 1, 4, 32>("mxf8f6f4");
  run_thr<1, 96, 2, 1, 4, 32>("mxf8f6f4");
  return 0;
}
