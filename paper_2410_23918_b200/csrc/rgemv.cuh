// Restore-and-multiply path for small batches (2 < B <= 32): y = W_hat_n x with the restored
// weight never leaving the SM (VERDICT r1 "prefill without the W' round trip").
//
//     W'[j, c] = sum_{i<n} S_i[j, c] (U'_i V'_i^T)[j, c]      (Eq.5, Eq.8)
//     y[b, j]  = sum_c W'[j, c] X'[b, c],  X' = x diag(1/s)   (Eq.4)
//
// The e4m3 decode pays 48 Zq columns of tensor work per token and sign element, so from a few
// tokens on its tensor time exceeds the cost of restoring W' (2.5 ALU ops per element and block
// plus a K = 16 MMA); the prefill path restores W' once but writes and re-reads it through HBM
// as an fp16 operand and pads the GEMM to 128 tokens.  Here each CTA owns one 128-row tile and a
// balanced contiguous range of (row tile, 128-channel unit) pairs (row-tile-major; a range can span
// row-tile segments, each with its own TMEM y buffer and partial slot) and, per (unit, block):
//   producer warp   TMA tensor copies of the U'_i tile and the V'_i chunk (32-byte swizzle = the
//                   UMMA K-major layout), one bulk copy of the 128 x 128 sign tile; stage ring
//   MMA warp        P_i = U'_i V'_i^T (tcgen05 kind::f16, M128 N128 K16: exact products, fp32
//                   TMEM, triple-buffered); per unit, after its restore: y_acc += W' X'^T
//                   (kind::tf32, 16 x K8 MMAs, A = W' from SMEM, B = the unit's X' image)
//   16 restore warps  (lane quadrant, 32-column quarter): tcgen05.ld P_i, apply the signs (SHF +
//                   LOP3 per element) and sum the blocks in fp32 (FADD2); at the unit's last
//                   block round W' to tf32 (RNA) into the SMEM A image
// then y_acc (TMEM, fp32) -> per-CTA partial slots -> the row tile's last CTA sums the slots in
// order (deterministic) and writes y.  Numerics: W' and X' rounded once to tf32 (10 explicit
// mantissa bits, fp32 range: no operand scaling), fp32 accumulation.
#pragma once
#include <cuda.h>   // CUtensorMap (the encoder is fetched at run time: no libcuda link)

#include "decode_tc.cuh"
#include "prefill.cuh"

namespace bs {

struct RgParams {
  CUtensorMap tmu;        // U' as [n x kh x rows_pad][16] 16-bit, box 128 x 16, 32-byte swizzle
  CUtensorMap tmv;        // V' as [n x kh x d_in_pad][16] 16-bit, box 128 x 16, 32-byte swizzle
  const uint4* signs;     // [n_cap][nq][rows_pad] F8 layout
  const uint16_t* u;      // [n x kh][rows_pad][16] U' (bf16 / f16 storage)
  const uint16_t* v;      // [n x kh][d_in_pad][16] V'
  const uint8_t* ximg;    // [nq] X' images of BP x 128 tf32 (rg_xprep_kernel)
  float* part;            // [grid][kmax][BP][128] fp32 partial y of each (CTA, row-tile segment)
  int* counters;          // [row_tiles], zero on entry and on exit
  void* y;
  long long y_stride;
  int y_dtype;            // 0 f32, 1 bf16
  int n;                  // active 16-rank blocks (halves)
  int ksh;                // sign tile of block i is i >> ksh
  int nq, rows_pad, rows_local, row_tiles, batch, f16;
  int kmax;               // max row-tile segments per CTA (partial slots per CTA)
  int splits;             // > 0: CTA b = (row tile b / splits, unit range b % splits of it); 0: balanced
  long long* trace;       // timing build (-DBS_RG_TRACE, scripts/rg_trace.py): per-stage stamps of CTA 0
  // W'-output mode (the prefill's restore, WOUT = true): each unit's W' goes to the GEMM's fp16
  // operand image instead of the GEMV, row j scaled by 2^-rowexp[j]
  uint8_t* wimg;          // [row_tiles_img][kc] tiles of kImgTileA bytes (prefill.cuh img_off layout)
  int* rowexp;            // [rows_pad]
  const float* vmaxr;     // [n x kh][16] max_c |V'[c, r]|
  int kc;                 // 64-column K chunks (d_in_pad / 64)
};

constexpr int kRgStages = 10;
constexpr int kRgPBuf = 3;                      // TMEM P buffers per half
#ifndef BS_RG_HALVES
#define BS_RG_HALVES 2
#endif
// The 128 channels of a unit form kRgHV independent product pipelines (P MMA N = 128 / kRgHV,
// their own buffers and barriers, their own restore warps), so the two groups of restore warps do
// not wait for each other and one group's TMEM loads overlap the other's arithmetic.
constexpr int kRgHV = BS_RG_HALVES;
constexpr int kRgPCols = 128 / kRgHV;
#ifndef BS_RG_COLS
#define BS_RG_COLS 32
#endif
constexpr int kRgCols = BS_RG_COLS;             // columns of a unit per restore warp (32 or 64)
constexpr int kRgNR = 4 * (128 / kRgCols);      // restore warps (4 lane quadrants x column groups)
#ifndef BS_RG_MMA2
#define BS_RG_MMA2 1
#endif
#if BS_RG_MMA2
// one MMA warp per channel half (warp kRgWarpMma + hv; the first also issues the GEMV), so a late
// half never holds up the other half's products
constexpr int kRgMmaWarps = 2;
#else
constexpr int kRgMmaWarps = 1;
#endif
static_assert(kRgMmaWarps <= kRgHV, "each MMA warp owns at least one channel part");
constexpr int kRgWarpMma = kRgNR, kRgWarpProd = kRgNR + kRgMmaWarps;
constexpr int kRgWarps = kRgNR + kRgMmaWarps + 1;   // restore warps + MMA warp(s) + producer
constexpr int kRgMaxBatch = 32;
constexpr int kRgStage = 4096 + 4096 + 2048;    // U' tile, V' chunk, sign tile
constexpr int kRgAImg = 128 * 128 * 4;          // W' unit, tf32
template <int BP> struct RgCfg {
  static constexpr int kXImg = BP * 128 * 4;    // X' unit, tf32
  static constexpr int kBarOff = kRgStages * kRgStage + kRgAImg + 2 * kXImg;
  static constexpr int kSmem = kBarOff + 512 + 1024;   // barriers + alignment slack
};

// X' = x / s per (unit q, token t < BP, channel k < 128), tf32 (RNA) in the UMMA K-major image:
// (t, k) at ((t / 8) 32 + k / 4) 128 + (t % 8) 16 + (k % 4) 4.  Tokens >= batch and channels >=
// d_in are zero.  One thread per 16-byte core row (4 channels of one token).
__global__ void __launch_bounds__(256) rg_xprep_kernel(const void* __restrict__ x, int x_dtype, long long x_stride,
                                                      const float* __restrict__ inv_s, int batch, int d_in, int nq,
                                                      int bp, uint4* __restrict__ img) {
  // the rgemv launch that follows (programmatic dependent launch) may start its restore pipeline now:
  // only its X' loads wait for this grid (griddepcontrol.wait in its producer)
  asm volatile("griddepcontrol.launch_dependents;");
  const long long pieces = (long long)nq * bp * 32;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < pieces;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / (bp * 32));
    const int rem = (int)(e % (bp * 32));
    const int t = rem / 32, k4 = rem % 32;
    uint32_t o[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int c = q * 128 + k4 * 4 + m;
      float v = 0.f;
      if (t < batch && c < d_in) v = load_act(x, (long long)t * x_stride + c, x_dtype) * __ldg(inv_s + c);
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
      o[m] = r;
    }
    const long long off = (long long)q * bp * 128 * 4 + ((t / 8) * 32 + k4) * 128 + (t % 8) * 16;
    img[off / 16] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// TMA 2D tile copy (box 16 x 128 of 16-bit elements, 32-byte swizzle) -> shared, tx on `bar`.
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor, K-major, 32-byte swizzle: rows of 32 B (16 x 16-bit, the whole
// K = 16), 8-row groups 256 B apart (SBO); LBO unused for a K extent within one swizzle span.
__device__ __forceinline__ uint64_t smem_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;   // SWIZZLE_32B
  return d;
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

template <bool BF16>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if (BF16)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%10,%10,%10,%10};"
                 : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%10,%10,%10,%10};"
                 : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
}

// byte offset of 16-byte chunk `ch` of row r in a [128][16] 16-bit tile written by TMA with the
// 32-byte swizzle (address bit 4 ^= bit 7; the tile is 256-byte aligned)
__device__ __forceinline__ uint32_t sw32_off(int r, int ch) { return (uint32_t)(r * 32 + ((ch ^ (r >> 2)) & 1) * 16); }

// W' row bound sum_i sum_r |U'_i[row, r]| max_c |V'_i[c, r]| of the W'-output mode.  Not inlined, so
// every caller (TMEM restore warps, register-product warps) rounds it identically: the two halves
// of a row must pick the same power-of-two scale.
__device__ __noinline__ float rg_row_bound(const uint16_t* __restrict__ u, const float* __restrict__ vmaxr, long long rows_pad,
                                           long long row, int n, int f16) {
  float bound = 0.f;
  for (int bi = 0; bi < n; ++bi) {
    const uint4* up = reinterpret_cast<const uint4*>(u + ((long long)bi * rows_pad + row) * 16);
    for (int kk = 0; kk < 2; ++kk) {
      const uint4 raw = __ldg(up + kk);
      const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 f = f16 ? __half22float2(*reinterpret_cast<const __half2*>(&wv[e2]))
                             : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e2]));
        const int r = kk * 8 + 2 * e2;
        bound = __fadd_rn(bound, __fadd_rn(__fmul_rn(fabsf(f.x), __ldg(vmaxr + bi * 16 + r)),
                                           __fmul_rn(fabsf(f.y), __ldg(vmaxr + bi * 16 + r + 1))));
      }
    }
  }
  return bound;
}

#ifdef BS_RG_TRACE
#define RG_TR(t_, c_) do { if (p.trace && blockIdx.x == 0 && (t_) < 2048) p.trace[(t_) * 8 + (c_)] = clock64(); } while (0)
#else
#define RG_TR(t_, c_) do { } while (0)
#endif
// Every role waits with a suspend-time hint by default (a spinning MMA / producer warp measured no
// faster: BS_RG_SPIN_FAST).
#ifdef BS_RG_SPIN_FAST
#define RG_WAIT_FAST mbar_wait
#else
#define RG_WAIT_FAST mbar_wait_sleep
#endif
template <int BP, bool WOUT, bool HYB>
__global__ void __launch_bounds__(kRgWarps * 32, 1) rgemv_kernel(const __grid_constant__ RgParams p) {
  using C = RgCfg<BP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* stages = smem;                                   // [kRgStages][U' 4K | V' 4K | signs 2K]
  uint8_t* aimg = smem + kRgStages * kRgStage;              // W' unit (tf32 A image)
  uint8_t* ximg = aimg + kRgAImg;                           // [2] X' units
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;                      // [S] producer arrive + tx (U', V' tensor copies, sign tile)
  uint64_t* sempty = full + kRgStages;        // [S] MMA commit + the restore warps (signs read)
  uint64_t* pfull = sempty + kRgStages;       // [HV][3] commit of P_i (one channel half)
  uint64_t* pempty = pfull + kRgHV * kRgPBuf; // [HV][3] the half's restore warps
  uint64_t* afull = pempty + kRgHV * kRgPBuf; // the restore warps wrote the W' unit
  uint64_t* aempty = afull + 1;               // commit of the unit's GEMV MMAs
  uint64_t* xfull = aempty + 1;               // [2] bulk copy of an X' unit
  uint64_t* xempty = xfull + 2;               // [2] commit of the GEMV that read it
  uint64_t* yfull = xempty + 2;               // [2] commit of a segment's last GEMV (y buffer seg & 1)
  uint64_t* yempty = yfull + 2;               // [2] the 4 draining warps read y buffer seg & 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(yempty + 2);
  int* fin = reinterpret_cast<int*>(tmem_slot + 1);   // [kmax + 1] row tiles this CTA finalises

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  // balanced work: the (row tile, unit) pairs in row-tile-major order, a contiguous range per
  // CTA; a range spans row-tile segments (each with its own partial slot and y buffer)
  const long long W = (long long)p.row_tiles * p.nq;
  const int G = gridDim.x;
  auto range_of = [&](int b, long long& a, long long& e) {   // CTA b's (row tile, unit) range
    if (p.splits > 0) {
      const int m = b / p.splits, k = b % p.splits;
      a = (long long)m * p.nq + (long long)p.nq * k / p.splits;
      e = (long long)m * p.nq + (long long)p.nq * (k + 1) / p.splits;
    } else {
      a = W * b / G;
      e = W * (b + 1) / G;
    }
  };
  long long w0, w1;
  range_of(cta, w0, w1);
  const int U = (int)(w1 - w0);               // units of this CTA
  const int mt0 = (int)(w0 / p.nq), qa = (int)(w0 % p.nq);
  const int n = p.n;
  const int T = U * n;                        // stages of this CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRgStages; ++s) {
      mbar_init(&full[s], 1);   // the producer's arrive + tx bytes
#ifdef BS_RG_BARSYNC
      mbar_init(&sempty[s], 2);   // the P MMA's commit + the restore warps' representative
#else
      mbar_init(&sempty[s], kRgMmaWarps + kRgNR);   // the P MMA commit(s) + every restore warp
#endif
    }
    for (int b = 0; b < kRgHV * kRgPBuf; ++b) {
      mbar_init(&pfull[b], 1);
#ifdef BS_RG_BARSYNC
      mbar_init(&pempty[b], 1);
#else
      mbar_init(&pempty[b], kRgNR / kRgHV);
#endif
    }
    mbar_init(afull, kRgNR);
    mbar_init(aempty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], 1);
      mbar_init(&xempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&yfull[b], 1);
      mbar_init(&yempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == kRgWarpProd) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  constexpr uint32_t kColY = kRgHV * kRgPBuf * kRgPCols;   // two y buffers of BP columns

  if (warp == kRgWarpProd) {
    // ================= producer (one lane): stage t = (the CTA's unit t / n, block t % n): the U'_i
    // tile and the V'_i chunk by TMA tensor copies (32-byte swizzle: the UMMA K-major layout),
    // the sign tile by a bulk copy, all completing as tx bytes on full[s]
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int dpad = p.nq * 128;
      int qx = qa;   // unit (channel chunk) of the next X' load; issue_x is called for u = 0, 1, 2, ...
      auto issue_x = [&](int u) {   // X' of the CTA's unit u into buffer u & 1
        if (u >= 2) mbar_wait_sleep(&xempty[u & 1], (uint32_t)(((u >> 1) - 1) & 1));
        mbar_arrive_expect_tx(&xfull[u & 1], C::kXImg);
        bulk_g2s(ximg + (u & 1) * C::kXImg, p.ximg + (long long)qx * C::kXImg, C::kXImg, &xfull[u & 1], pol);
        if (++qx == p.nq) qx = 0;
      };
      if (!WOUT) asm volatile("griddepcontrol.wait;" ::: "memory");   // this call's X' image is complete
      if (!WOUT && U > 0) issue_x(0);
      if (!WOUT && U > 1) issue_x(1);
      int s = 0, u = 0, i = 0, qq = qa, mt = mt0;
      uint32_t sph = 0;
      for (int t = 0; t < T; ++t) {
        if (!WOUT && i == 0 && u >= 2) issue_x(u);
        if (t >= kRgStages) RG_WAIT_FAST(&sempty[s], sph ^ 1u);
        RG_TR(t, 0);
        uint8_t* st = stages + s * kRgStage;
        mbar_arrive_expect_tx(&full[s], 4096 + 4096 + 2048);
        tma_2d(st, &p.tmu, 0, i * p.rows_pad + mt * 128, &full[s]);
        tma_2d(st + 4096, &p.tmv, 0, i * dpad + qq * 128, &full[s]);
        bulk_g2s(st + 8192, p.signs + ((long long)(i >> p.ksh) * p.nq + qq) * p.rows_pad + mt * 128, 2048, &full[s], pol);
        if (++i == n) {
          i = 0;
          ++u;
          if (++qq == p.nq) { qq = 0; ++mt; }
        }
        if (++s == kRgStages) { s = 0; sph ^= 1u; }
      }
    }
  } else if (warp >= kRgWarpMma && warp < kRgWarpMma + kRgMmaWarps) {
    // ================= MMA warp(s)
    const int mw = warp - kRgWarpMma;   // with two MMA warps: the channel half this one issues
    const uint32_t idp = idesc_f16_f32(128, kRgPCols, p.f16 ? 0u : 1u);
    const uint32_t idg = idesc_f16_f32(128, BP, 2u);   // kind::tf32
    int gpend = -1;   // unit (CTA-local) whose GEMV is pending
    int gq = qa, gseg = 0;   // channel chunk and segment of the next GEMV (called for j = 0, 1, 2, ...)
    auto gemv = [&](int j) {   // the CTA's unit j: y buffer of its segment
      const int seg = gseg;
      const bool first = j == 0 || gq == 0;
      const bool last = j == U - 1 || gq == p.nq - 1;
      if (++gq == p.nq) { gq = 0; ++gseg; }
      if (first && seg >= 2) RG_WAIT_FAST(&yempty[seg & 1], (uint32_t)(((seg >> 1) - 1) & 1));
      RG_WAIT_FAST(afull, (uint32_t)(j & 1));
      RG_WAIT_FAST(&xfull[j & 1], (uint32_t)((j >> 1) & 1));
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a0 = smem_u32(aimg), x0 = smem_u32(ximg + (j & 1) * C::kXImg);
        const uint32_t yc = tbase + kColY + (uint32_t)((seg & 1) * BP);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          mma_tf32_ss(yc, smem_desc_kmajor(a0 + kk * 256, 128, 4096), smem_desc_kmajor(x0 + kk * 256, 128, 4096), idg,
                      (!first || kk > 0) ? 1u : 0u);
        mma_commit(aempty);
        mma_commit(&xempty[j & 1]);
        if (last) mma_commit(&yfull[seg & 1]);
      }
      __syncwarp();
    };
    int s = 0, pb = 0, u = 0, i = 0;
    uint32_t sph = 0, pph = 0;
    for (int t = 0; t < T; ++t) {
      RG_WAIT_FAST(&full[s], sph);
      if (lane == 0) RG_TR(t, 2);
#pragma unroll
      for (int hv = 0; hv < kRgHV; ++hv) {
        if (kRgMmaWarps > 1 && hv % kRgMmaWarps != mw) continue;
        if (HYB && hv == 1) {   // this half's products are formed by its restore warps (mma.sync)
          if (lane == 0) mbar_arrive(&sempty[s]);
          __syncwarp();
          continue;
        }
        if (t >= kRgPBuf) RG_WAIT_FAST(&pempty[hv * kRgPBuf + pb], pph ^ 1u);
        if (lane == 0 && hv == 0) RG_TR(t, 3);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(stages + s * kRgStage);
          mma_f16_ss(tbase + (uint32_t)((hv * kRgPBuf + pb) * kRgPCols), smem_desc_sw32(sa),
                     smem_desc_sw32(sa + 4096 + hv * kRgPCols * 32), idp, 0u);
          mma_commit(&pfull[hv * kRgPBuf + pb]);
          if (hv + kRgMmaWarps >= kRgHV) mma_commit(&sempty[s]);   // this warp's last product of the stage
        }
        __syncwarp();
      }
      if (!WOUT && mw == 0 && gpend >= 0) {   // the previous unit's GEMV, once the next unit's first product is queued
        gemv(gpend);
        gpend = -1;
      }
      if (++i == n) { gpend = u; i = 0; ++u; }
      if (++s == kRgStages) { s = 0; sph ^= 1u; }
      if (++pb == kRgPBuf) { pb = 0; pph ^= 1u; }
    }
    if (!WOUT && mw == 0 && gpend >= 0) gemv(gpend);
    __syncwarp();
  } else if (warp < kRgNR) {
    // ================= restore warps: lane quadrant qd, column group h (kRgCols columns)
    constexpr int NC = kRgCols, NW = NC / 32;
    const int qd = warp & 3, h = warp >> 2;
    const int hv = (h * NC) / kRgPCols;                // channel half of this warp's columns
    const int pcol = (h * NC) % kRgPCols;              // its columns inside the half's P buffer
    const int j = qd * 32 + lane;
    const uint32_t lq = (uint32_t)(qd * 32) << 16;
    if (HYB && hv == 1) {
      // ---- channel half 1 with the products in registers: this warp's 32 x 32 share (rows 32 qd..,
      // channels 64 + 32 (h & 1)..) of P_i = U'_i V'_i^T by mma.sync m16n8k16 from the stage's
      // U' / V' tiles, so only half 0's products are read back from TMEM
      const int g = lane >> 2, t4 = lane & 3, hq = h & 1;
      const int ssh = 16 * (t4 & 1) + (t4 >> 1);   // channel 8 ni + 2 t4 + e of the sign word -> bit 8 e + 2 ni
      const uint32_t a_off = sw32_off(32 * qd + (lane & 15), lane >> 4);
      const uint32_t b_off = 4096 + sw32_off(64 + 32 * hq + (lane & 7) + 8 * (lane >> 4), (lane >> 3) & 1);
      const uint32_t s_off = 8192 + (32 * qd + g) * 16 + h * 4;
      float ha[2][4][4];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 4; ++e) ha[a][b][e] = 0.f;
      int s = 0, u = 0, i = 0, uq = qa, useg = 0, wseg = -1;
      uint32_t sph = 0;
      float wsc[2][2] = {{1.f, 1.f}, {1.f, 1.f}};
      for (int t = 0; t < T; ++t) {
        mbar_wait_sleep(&full[s], sph);
        const uint32_t sb = smem_u32(stages + s * kRgStage);
        uint32_t af[2][4], bfr[2][4], sw[2][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) ldsm_x4(sb + a_off + 512 * mi, af[mi][0], af[mi][1], af[mi][2], af[mi][3]);
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) ldsm_x4(sb + b_off + 512 * nb, bfr[nb][0], bfr[nb][1], bfr[nb][2], bfr[nb][3]);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t x;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(sb + s_off + (16 * mi + 8 * hh) * 16));
            sw[mi][hh] = x >> ssh;   // clear bit = negative sign
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s]);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            float d[4];
            if (p.f16) mma16816<false>(d, af[mi], bfr[ni >> 1][(ni & 1) * 2], bfr[ni >> 1][(ni & 1) * 2 + 1]);
            else mma16816<true>(d, af[mi], bfr[ni >> 1][(ni & 1) * 2], bfr[ni >> 1][(ni & 1) * 2 + 1]);
            const int bb = 2 * ni;
            const uint32_t s0 = sw[mi][0], s1 = sw[mi][1];
            const float2 lo = make_float2(__uint_as_float(__float_as_uint(d[0]) ^ (~(s0 << (31 - bb)) & 0x80000000u)),
                                          __uint_as_float(__float_as_uint(d[1]) ^ (~(s0 << (23 - bb)) & 0x80000000u)));
            const float2 hi = make_float2(__uint_as_float(__float_as_uint(d[2]) ^ (~(s1 << (31 - bb)) & 0x80000000u)),
                                          __uint_as_float(__float_as_uint(d[3]) ^ (~(s1 << (23 - bb)) & 0x80000000u)));
            const float2 a0 = __fadd2_rn(make_float2(ha[mi][ni][0], ha[mi][ni][1]), lo);
            const float2 a1 = __fadd2_rn(make_float2(ha[mi][ni][2], ha[mi][ni][3]), hi);
            ha[mi][ni][0] = a0.x;
            ha[mi][ni][1] = a0.y;
            ha[mi][ni][2] = a1.x;
            ha[mi][ni][3] = a1.y;
          }
        if (++s == kRgStages) { s = 0; sph ^= 1u; }
        if (++i < n) continue;
        i = 0;
        if (WOUT) {   // W'[rows, unit] complete: scaled fp16 into the GEMM's operand image (chunk 2 uq + 1)
          if (useg != wseg) {
            wseg = useg;
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const long long row = (long long)(mt0 + useg) * 128 + 32 * qd + 16 * mi + 8 * hh + g;
                const float bound = rg_row_bound(p.u, p.vmaxr, p.rows_pad, row, n, p.f16);
                int re = 0;
                if (bound > 0.f && bound < __int_as_float(0x7f800000)) re = xs_exp(__float_as_uint(bound), 15);
                wsc[mi][hh] = exp2i(-re);
              }
          }
          uint8_t* dst = p.wimg + ((long long)(mt0 + useg) * p.kc + 2 * uq + 1) * kImgTileA;
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni)
                *reinterpret_cast<uint32_t*>(dst + img_off(32 * qd + 16 * mi + 8 * hh + g, 32 * hq + 8 * ni + 2 * t4)) =
                    pack_half2(ha[mi][ni][2 * hh] * wsc[mi][hh], ha[mi][ni][2 * hh + 1] * wsc[mi][hh]);
        } else {      // tf32 A image (after the previous GEMV read it)
          if (u > 0) mbar_wait_sleep(aempty, (uint32_t)((u - 1) & 1));
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni) {
                const int r = 32 * qd + 16 * mi + 8 * hh + g, c = 64 + 32 * hq + 8 * ni + 2 * t4;
                uint32_t o0, o1;
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(o0) : "f"(ha[mi][ni][2 * hh]));
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(o1) : "f"(ha[mi][ni][2 * hh + 1]));
                *reinterpret_cast<uint2*>(aimg + ((r >> 3) * 32 + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4) =
                    make_uint2(o0, o1);
              }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(afull);
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 4; ++e) ha[a][b][e] = 0.f;
        ++u;
        if (++uq == p.nq) { uq = 0; ++useg; }
      }
    } else {
    float acc[NC];
#pragma unroll
    for (int l = 0; l < NC; ++l) acc[l] = 0.f;
    int s = 0, pb = 0, u = 0, i = 0, uq = qa, useg = 0;
    int wseg = -1;       // WOUT: row-tile segment whose row scale wsc holds
    float wsc = 1.f;
    uint32_t sph = 0, pph = 0;
    static_assert(!WOUT || NC == 32, "W'-output mode: 32 columns per restore warp");
    for (int t = 0; t < T; ++t) {
#ifdef BS_RG_SPIN
      mbar_wait(&pfull[hv * kRgPBuf + pb], pph);
#else
      mbar_wait_sleep(&pfull[hv * kRgPBuf + pb], pph);
#endif
      if (lane == 0 && (warp == 0 || warp == kRgNR - 1)) RG_TR(t, warp == 0 ? 4 : 6);
      tc_fence_after();
      uint32_t m[NC];
#pragma unroll
      for (int g = 0; g < NW; ++g)
        tmem_ld32(tbase + lq + (uint32_t)((hv * kRgPBuf + pb) * kRgPCols + pcol + g * 32),
                  *reinterpret_cast<uint32_t(*)[32]>(m + 32 * g));
      mbar_wait(&full[s], sph);   // completed (the MMA warp waited on it): its sign tile is here
      uint32_t nw[NW];
#pragma unroll
      for (int g = 0; g < NW; ++g)
      {   // explicit shared-space load (a generic load of this word measured as the loop's top stall)
        uint32_t w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w)
                     : "r"(smem_u32(stages + s * kRgStage + 8192 + j * 16 + (h * NW + g) * 4)));
        nw[g] = ~w;
      }
      tmem_ld_wait();
      if (lane == 0 && warp == 0) RG_TR(t, 1);
      tc_fence_before();
#ifdef BS_RG_BARSYNC
      // the restore warps meet once per stage; one thread then frees the P buffer and the
      // stage's sign tile (2 mbarrier arrivals per stage instead of one per warp)
      asm volatile("bar.sync 1, %0;" ::"n"(kRgNR * 32) : "memory");
      if (threadIdx.x == 0) {
        for (int v = 0; v < kRgHV; ++v) mbar_arrive(&pempty[v * kRgPBuf + pb]);
        mbar_arrive(&sempty[s]);
      }
#else
      // each warp frees its share of the P buffer and the stage's sign tile as soon as it holds
      // them in registers, so fast warps run ahead instead of meeting the slowest every stage
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pempty[hv * kRgPBuf + pb]);
        mbar_arrive(&sempty[s]);
      }
#endif
#ifdef BS_RG_EXP_NOAPPLY   // timing experiment: no sign application (wrong values)
#pragma unroll
      for (int l = 0; l < NC; ++l) acc[l] += __uint_as_float(m[l]);
#else
#pragma unroll
      for (int l = 0; l < NC; l += 2) {   // F8 layout: column c of a word is bit (c & 3) 8 + (c >> 2)
        const int c0 = l & 31, c1 = (l + 1) & 31;
        const uint32_t w = nw[l >> 5];
        const int b0 = (c0 & 3) * 8 + (c0 >> 2), b1 = (c1 & 3) * 8 + (c1 >> 2);
        const float2 tv = make_float2(__uint_as_float(m[l] ^ ((w << (31 - b0)) & 0x80000000u)),
                                      __uint_as_float(m[l + 1] ^ ((w << (31 - b1)) & 0x80000000u)));
        const float2 a = __fadd2_rn(make_float2(acc[l], acc[l + 1]), tv);
        acc[l] = a.x;
        acc[l + 1] = a.y;
      }
#endif
      if (lane == 0 && (warp == 0 || warp == kRgNR - 1)) RG_TR(t, warp == 0 ? 5 : 7);
      if (WOUT && i + 1 == n) {   // W'[j, unit] complete: scaled fp16 into the GEMM's operand image
        if (useg != wseg) {   // a new row tile: its row scale 2^-re with sum |U'| max |V'| < 2^15
          wseg = useg;
          const long long row = (long long)(mt0 + useg) * 128 + j;
          const float bound = rg_row_bound(p.u, p.vmaxr, p.rows_pad, row, n, p.f16);
          int re = 0;
          if (bound > 0.f && bound < __int_as_float(0x7f800000)) re = xs_exp(__float_as_uint(bound), 15);
          if (h == 0) p.rowexp[row] = re;
          wsc = exp2i(-re);
        }
        const int c = 2 * uq + (h >> 1), k0 = (h & 1) * 32;
        uint8_t* dst = p.wimg + ((long long)(mt0 + useg) * p.kc + c) * kImgTileA;
#pragma unroll
        for (int mq = 0; mq < 4; ++mq)
          *reinterpret_cast<uint4*>(dst + img_off(j, k0 + 8 * mq)) =
              make_uint4(pack_half2(acc[8 * mq + 0] * wsc, acc[8 * mq + 1] * wsc),
                         pack_half2(acc[8 * mq + 2] * wsc, acc[8 * mq + 3] * wsc),
                         pack_half2(acc[8 * mq + 4] * wsc, acc[8 * mq + 5] * wsc),
                         pack_half2(acc[8 * mq + 6] * wsc, acc[8 * mq + 7] * wsc));
#pragma unroll
        for (int l = 0; l < NC; ++l) acc[l] = 0.f;
        i = 0;
        ++u;
        if (++uq == p.nq) { uq = 0; ++useg; }
      } else if (++i == n) {   // W'[j, unit] complete: tf32 A image (after the previous GEMV read it)
        if (u > 0) mbar_wait_sleep(aempty, (uint32_t)((u - 1) & 1));
#pragma unroll
        for (int mq = 0; mq < NC / 4; ++mq) {
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(o[e]) : "f"(acc[4 * mq + e]));
          *reinterpret_cast<uint4*>(aimg + ((j >> 3) * 32 + h * (NC / 4) + mq) * 128 + (j & 7) * 16) =
              make_uint4(o[0], o[1], o[2], o[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(afull);
#pragma unroll
        for (int l = 0; l < NC; ++l) acc[l] = 0.f;
        if (h == 0 && u != U - 1 && uq == p.nq - 1) {   // a segment ends mid-range: drain it now
          const int seg = useg;
          mbar_wait_sleep(&yfull[seg & 1], (uint32_t)((seg >> 1) & 1));
          tc_fence_after();
          float* slot = p.part + ((long long)cta * p.kmax + seg) * BP * 128;
#pragma unroll
          for (int b0 = 0; b0 < BP; b0 += 16) {
            uint32_t yv[16];
            tmem_ld16(tbase + lq + kColY + (uint32_t)((seg & 1) * BP + b0), yv);
            tmem_ld_wait();
#pragma unroll
            for (int b = 0; b < 16; ++b) slot[(b0 + b) * 128 + j] = __uint_as_float(yv[b]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&yempty[seg & 1]);
        }
        i = 0;
        ++u;
        if (++uq == p.nq) { uq = 0; ++useg; }
      }
      if (++s == kRgStages) { s = 0; sph ^= 1u; }
      if (++pb == kRgPBuf) { pb = 0; pph ^= 1u; }
    }
    if (!WOUT && h == 0 && U > 0) {   // the range's last segment: y buffer -> partial slot
      const int seg = (int)((w1 - 1) / p.nq) - mt0;
      mbar_wait_sleep(&yfull[seg & 1], (uint32_t)((seg >> 1) & 1));
      tc_fence_after();
      float* slot = p.part + ((long long)cta * p.kmax + seg) * BP * 128;
#pragma unroll
      for (int b0 = 0; b0 < BP; b0 += 16) {
        uint32_t yv[16];
        tmem_ld16(tbase + lq + kColY + (uint32_t)((seg & 1) * BP + b0), yv);
        tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < 16; ++b) slot[(b0 + b) * 128 + j] = __uint_as_float(yv[b]);
      }
    }
    }   // !(HYB && hv == 1)
  }

  // ---- teardown; the last CTA to finish a row tile sums its partial slots in CTA order and writes y
  __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kRgWarpProd) tmem_dealloc<512>(tbase);
  auto cover = [&](int mt, int& b_lo, int& b_hi) {   // CTAs whose range meets row tile mt
    if (p.splits > 0) {
      b_lo = mt * p.splits;
      b_hi = b_lo + p.splits - 1;
      return;
    }
    const long long a = (long long)mt * p.nq, e = a + p.nq;
    int b = (int)(a * G / W);
    while (b > 0 && W * b / G > a) --b;
    while (W * (b + 1) / G <= a) ++b;
    b_lo = b;
    while (b + 1 < G && W * (b + 1) / G < e) ++b;
    b_hi = b;
  };
  if (WOUT) return;   // the image tiles are disjoint: no split-K
  if (threadIdx.x == 0) {
    __threadfence();
    int nf = 0;
    const int nseg = U > 0 ? (int)((w1 - 1) / p.nq) - mt0 + 1 : 0;
    for (int k = 0; k < nseg; ++k) {
      int b_lo, b_hi;
      cover(mt0 + k, b_lo, b_hi);
      const int prev = atomicAdd(p.counters + mt0 + k, 1);
      if (prev == b_hi - b_lo) fin[1 + nf++] = mt0 + k;
    }
    fin[0] = nf;
  }
  __syncthreads();
  long long* slot_base = reinterpret_cast<long long*>(stages);   // the stage ring is idle now
  for (int f = 0; f < fin[0]; ++f) {
    __threadfence();
    const int mt = fin[1 + f];
    int b_lo, b_hi;
    cover(mt, b_lo, b_hi);
    for (int c = b_lo + (int)threadIdx.x; c <= b_hi; c += blockDim.x) {   // each covering CTA's slot, once
      long long ca, ce;
      range_of(c, ca, ce);
      slot_base[c - b_lo] = ((long long)c * p.kmax + (mt - (int)(ca / p.nq))) * BP * 128;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 128 * p.batch; e += blockDim.x) {
      const int b = e / 128, r = e % 128;
      const long long row = (long long)mt * 128 + r;
      float a = 0.f;
      for (int c = 0; c <= b_hi - b_lo; ++c) a += __ldcg(p.part + slot_base[c] + b * 128 + r);
      if (row < p.rows_local) {
        const long long o = (long long)b * p.y_stride + row;
        if (p.y_dtype == 0) reinterpret_cast<float*>(p.y)[o] = a;
        else reinterpret_cast<__nv_bfloat16*>(p.y)[o] = __float2bfloat16_rn(a);
      }
    }
    if (threadIdx.x == 0) p.counters[mt] = 0;
    __syncthreads();   // slot_base is rewritten for the next row tile
  }
}

#undef RG_TR
#undef RG_WAIT_FAST
}  // namespace bs
