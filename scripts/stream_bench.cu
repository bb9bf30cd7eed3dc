// HBM -> SMEM streaming rate of 1D bulk copies (cp.async.bulk, the decode kernel's producer
// pattern) through a STAGES-deep mbarrier ring, one CTA per SM, a consumer warp that only
// waits `full` and arrives `empty`.  Debug tool: python scripts/run_microbench.py stream_bench
#include <cstdio>
#include "../paper_2410_23918_b200/csrc/decode_f8.cuh"
using namespace bs;

template <int STAGES, int COPIES>
__global__ void __launch_bounds__(64, 1) stream(const uint8_t* src, long long bytes_per_cta, int chunk, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = src + (long long)blockIdx.x * bytes_per_cta;
  const int units = (int)(bytes_per_cta / chunk);
  long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0; uint32_t ph = 0;
      for (int k = 0; k < units; ++k) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], chunk);
        const int part = chunk / COPIES;
        for (int c = 0; c < COPIES; ++c)
          bulk_g2s(smem + s * chunk + c * part, base + (long long)k * chunk + c * part, part, &full[s], pol);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (int k = 0; k < units; ++k) {
      mbar_wait(&full[s], ph);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int STAGES, int COPIES>
void go(const char* name, const uint8_t* buf, int chunk, int sms) {
  const long long per = 4ll << 20;   // 4 MiB per CTA -> 592 MiB total (> 4x L2)
  long long* d;
  cudaMalloc(&d, 8 * sms);
  const int smem = STAGES * chunk;
  cudaFuncSetAttribute(stream<STAGES, COPIES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  stream<STAGES, COPIES><<<sms, 64, smem>>>(buf, per, chunk, d);   // warm
  cudaEventRecord(e0);
  stream<STAGES, COPIES><<<sms, 64, smem>>>(buf, per, chunk, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s chunk %6d x%d stages %2d: %7.1f GB/s %s\n", name, chunk, COPIES, STAGES, per * sms / (ms * 1e-3) / 1e9,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

extern "C" void run_all() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  cudaMalloc(&buf, (4ll << 20) * sms);
  cudaMemset(buf, 1, (4ll << 20) * sms);
  go<12, 1>("1D bulk, decode-like stage", buf, 14336, sms);
  go<12, 2>("1D bulk, 2 copies per stage", buf, 14336, sms);
  go<6, 1>("1D bulk", buf, 32768, sms);
  go<12, 1>("1D bulk", buf, 16384, sms);
  go<24, 1>("1D bulk", buf, 8192, sms);
  go<4, 1>("1D bulk", buf, 16384, sms);
  go<12, 4>("1D bulk, 4 copies per stage", buf, 16384, sms);
  cudaFree(buf);
}
