// W' restore for the prefill with the products in registers:
//   W'[j, c] = sum_i S_i[j, c] * (U'_i V'_i^T)[j, c]      (§2.1 Eq. 4-5, W' = W diag(s))
// written, per (128-row tile, 128-channel unit), as the GEMM's scaled fp16 operand image
// (prefill.cuh img_off layout, row j scaled by 2^-rowexp[j]) -- the same output as rgemv_kernel<16,
// true>, which forms P_i = U'_i V'_i^T with tcgen05 into TMEM and is bound by reading those fp32
// products back (4 B per element and block at 64 B/clk/SM).  Here each warp forms its 32 x 64 part
// of P_i with warp-level mma.sync m16n8k16 (fp16 / bf16 -> fp32, measured 1022 MAC/clk/SM on B200:
// 64 element-blocks per clock per SM at rank 16, 4x the TMEM-read rate), so the accumulator never
// leaves the register file and the restore is bound by its ALU work instead (sign XOR + FADD).
//   producer (lane 0 of warp 0): U'_i tile and V'_i chunk by TMA (box 128 x 16, 32-byte swizzle), the
//                  sign tile by a bulk copy, into a ring of stages (10 KB each);
//   8 warps (row quarter wr x channel half wc): ldmatrix the fragments, 16 mma.sync per
//                  stage, sign application and block sum in fp32; at a unit's last block the row
//                  scale and coalesced fp16 stores (32 lanes = one 128-byte row of the image).
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "rgemv.cuh"

namespace bs {

#ifndef BS_WR_STAGES
#define BS_WR_STAGES 6
#endif
constexpr int kWrStages = BS_WR_STAGES;
constexpr int kWrConsumers = 8;
constexpr int kWrThreads = kWrConsumers * 32;
constexpr int kWrBarOff = kWrStages * kRgStage;
constexpr int kWrSmem = kWrBarOff + 2 * kWrStages * 8 + 1024;   // + alignment slack

template <bool BF16>
__global__ void __launch_bounds__(kWrThreads, 2) wrestore_hmma_kernel(const __grid_constant__ RgParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWrBarOff);
  uint64_t* empty = full + kWrStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // balanced contiguous ranges of the (row tile, unit) pairs, row-tile-major
  const long long W = (long long)p.row_tiles * p.nq;
  const long long w0 = W * blockIdx.x / gridDim.x, w1 = W * (blockIdx.x + 1) / gridDim.x;
  const int U = (int)(w1 - w0), n = p.n, T = U * n;
  const int mt0 = (int)(w0 / p.nq), qa = (int)(w0 % p.nq);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWrStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWrConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // the producer is lane 0 of warp 0 (no separate warp: 8 warps x 2 CTAs per SM keep 128 registers
  // per thread): stage tt = (the CTA's unit tt / n, block tt % n), issued kWrStages - 1 ahead
  const uint64_t pol = policy_evict_first();
  const int dpad = p.nq * 128;
  int pi = 0, pq = qa, pm = mt0, ps = 0, pt = 0;
  uint32_t pph = 0;
  auto issue = [&]() {   // stage pt into slot ps (after every warp released its previous use)
    if (pt >= kWrStages) mbar_wait(&empty[ps], pph ^ 1u);
    uint8_t* st = stages + ps * kRgStage;
    mbar_arrive_expect_tx(&full[ps], 4096 + 4096 + 2048);
    tma_2d(st, &p.tmu, 0, pi * p.rows_pad + pm * 128, &full[ps]);
    tma_2d(st + 4096, &p.tmv, 0, pi * dpad + pq * 128, &full[ps]);
    bulk_g2s(st + 8192, p.signs + ((long long)(pi >> p.ksh) * p.nq + pq) * p.rows_pad + pm * 128, 2048, &full[ps], pol);
    if (++pi == n) {
      pi = 0;
      if (++pq == p.nq) { pq = 0; ++pm; }
    }
    if (++ps == kWrStages) { ps = 0; pph ^= 1u; }
    ++pt;
  };
  const bool producer = threadIdx.x == 0;
  if (producer)
    while (pt < T && pt < kWrStages - 1) issue();

  // ================= consumer warp: rows 32 wr .. +32, channels 64 wc .. +64 of the unit
  const int wr = warp & 3, wc = warp >> 2, g = lane >> 2, t4 = lane & 3;
  // the sign word of row j, channel group (32 channels) q: channel c is bit (c & 3) 8 + (c >> 2); this
  // thread's channels 8 ni + 2 t4 + e sit at bit 8 (2 (t4 & 1) + e) + 2 (ni & 3) + (t4 >> 1)
  const int ssh = 16 * (t4 & 1) + (t4 >> 1);
  // ldmatrix lane addresses (row / channel, 16-byte chunk) inside the stage's U' tile and V' chunk
  // (row + 16 m keeps the swizzle phase, so one offset per operand serves every fragment)
  const uint32_t a_off = sw32_off(32 * wr + (lane & 15), lane >> 4);
  const uint32_t b_off = 4096 + sw32_off(64 * wc + (lane & 7) + 8 * (lane >> 4), (lane >> 3) & 1);
  const uint32_t s_off = 8192 + (32 * wr + g) * 16 + wc * 8;
  float acc[2][8][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.f;
  int s = 0, i = 0, uq = qa, mt = mt0, smt = -1;
  uint32_t ph = 0;
  float wsc[2][2] = {{1.f, 1.f}, {1.f, 1.f}};
  for (int t = 0; t < T; ++t) {
    if (producer && pt < T) issue();   // stage t + kWrStages - 1 (waits for stage t - 1's release)
    mbar_wait(&full[s], ph);
    const uint32_t sb = smem_u32(stages + s * kRgStage);
    uint32_t af[2][4], sw[2][2][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
      ldsm_x4(sb + a_off + 512 * mi, af[mi][0], af[mi][1], af[mi][2], af[mi][3]);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t x0, x1;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(sb + s_off + (16 * mi + 8 * hh) * 16));
        sw[mi][hh][0] = x0 >> ssh;   // clear bit = negative sign
        sw[mi][hh][1] = x1 >> ssh;
      }
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {   // 16 channels: two n8 tiles
      uint32_t bf[4];
      ldsm_x4(sb + b_off + 512 * nb, bf[0], bf[1], bf[2], bf[3]);
      if (nb == 3) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);   // the stage is in registers
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int ni = 2 * nb + sub;
          float d[4];
          mma16816<BF16>(d, af[mi], bf[2 * sub], bf[2 * sub + 1]);
          const int q = ni >> 2, bb = 2 * (ni & 3);
          const uint32_t s0 = sw[mi][0][q], s1 = sw[mi][1][q];
          const float2 lo = make_float2(__uint_as_float(__float_as_uint(d[0]) ^ (~(s0 << (31 - bb)) & 0x80000000u)),
                                        __uint_as_float(__float_as_uint(d[1]) ^ (~(s0 << (23 - bb)) & 0x80000000u)));
          const float2 hi = make_float2(__uint_as_float(__float_as_uint(d[2]) ^ (~(s1 << (31 - bb)) & 0x80000000u)),
                                        __uint_as_float(__float_as_uint(d[3]) ^ (~(s1 << (23 - bb)) & 0x80000000u)));
          const float2 a0 = __fadd2_rn(make_float2(acc[mi][ni][0], acc[mi][ni][1]), lo);
          const float2 a1 = __fadd2_rn(make_float2(acc[mi][ni][2], acc[mi][ni][3]), hi);
          acc[mi][ni][0] = a0.x;
          acc[mi][ni][1] = a0.y;
          acc[mi][ni][2] = a1.x;
          acc[mi][ni][3] = a1.y;
        }
    }
    if (++s == kWrStages) { s = 0; ph ^= 1u; }
    if (++i < n) continue;
    // ---- W'[rows, unit] complete
    i = 0;
    if (mt != smt) {   // a new row tile: row scale 2^-re with sum_i |U'_i| max|V'_i| < 2^15 (as rgemv WOUT)
      smt = mt;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const long long row = (long long)mt * 128 + 32 * wr + 16 * mi + 8 * hh + g;
          float bound = 0.f;
          for (int bi = 0; bi < n; ++bi) {   // this lane: ranks 4 t4 .. 4 t4 + 3
            const uint2 raw = __ldg(reinterpret_cast<const uint2*>(p.u + ((long long)bi * p.rows_pad + row) * 16 + 4 * t4));
            const uint32_t wv[2] = {raw.x, raw.y};
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
              const float2 f = BF16 ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e2]))
                                    : __half22float2(*reinterpret_cast<const __half2*>(&wv[e2]));
              const int r = 4 * t4 + 2 * e2;
              bound += fabsf(f.x) * __ldg(p.vmaxr + bi * 16 + r) + fabsf(f.y) * __ldg(p.vmaxr + bi * 16 + r + 1);
            }
          }
          bound += __shfl_xor_sync(0xffffffffu, bound, 1);
          bound += __shfl_xor_sync(0xffffffffu, bound, 2);
          int re = 0;
          if (bound > 0.f && bound < __int_as_float(0x7f800000)) re = xs_exp(__float_as_uint(bound), 15);
          if (wc == 0 && t4 == 0) p.rowexp[row] = re;
          wsc[mi][hh] = exp2i(-re);
        }
    }
    uint8_t* dst = p.wimg + ((long long)mt * p.kc + 2 * uq + wc) * kImgTileA;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = 32 * wr + 16 * mi + 8 * hh + g;
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) {
          *reinterpret_cast<uint32_t*>(dst + img_off(r, 8 * ni + 2 * t4)) =
              pack_half2(acc[mi][ni][2 * hh] * wsc[mi][hh], acc[mi][ni][2 * hh + 1] * wsc[mi][hh]);
          acc[mi][ni][2 * hh] = 0.f;
          acc[mi][ni][2 * hh + 1] = 0.f;
        }
      }
    if (++uq == p.nq) { uq = 0; ++mt; }
  }
}

}  // namespace bs
