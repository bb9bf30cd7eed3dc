// Block-scaled (MX) e4m3 decode: the production decode path for bf16 / fp16 factors.
//
// Computes y[b, j] = sum_i sum_r U'_i[j, r] (S_i (V'_i[:, r] (.) x_b / s))[j]   (Eq.4 P:111,
// Eq.7-8; the factored form of W_hat_n x) with
// tcgen05.mma.kind::mxf8f6f4.block_scale, A read from TMEM:
//   * A = S_i as e4m3 +-1.0 (a pure function of the sign bits: LOP3 + IMAD per 4 signs,
//     expand_e4m3 with the exponent fixed at 0), so the sign stream never waits for Z;
//   * B = Z = V' (.) x/s as THREE e4m3 digits per (rank, token) column, each digit with its own
//     UE8M0 scale per 32-channel K-block (the MX block scale).  Z ~= sum_d q_d 2^sigma_d, the
//     scales are chosen per (K-block, column, digit) from that K-block's own maximum, so there is
//     no shared exponent across units, tokens or channels: any finite x (tokens 2^12 apart,
//     single outlier channels, ...) keeps ~12 significant bits per element
//     (round 1's per-unit exponent / A = +-2^a scheme had a silent clamp).
//   * scale_A = 1.0 for every row (constant UE8M0 127), scale_B from the Zq unit via tcgen05.cp.
// The MX semantics on sm_100a (TS form, CUTLASS SF chunk layout through tcgen05.cp
// 32x128b.warpx4) were pinned on a B200 before use: scripts/mx_probe.cu, max error 2.4e-7 of
// sum |products| against an fp64 host reference over 4 K-blocks with random scales.
//
// Two kernels per call:
//   zq_mx_kernel<NB>   one CTA per (block i, 128-channel subchunk q) unit: Z in fp32, then per
//                      warp (= one 32-channel K-block) and column: redux.max -> sigma ->
//                      e4m3 RNE digit -> exact residual -> next digit.  Writes the unit as a
//                      ready-to-copy UMMA B image + its SFB chunks (MxCfg::kUnit bytes).
//   decode_mx_kernel   warp-specialised, one CTA per SM: a producer thread streams sign tiles
//                      (R row tiles x 128 rows x 16 B) and Zq units into a stage ring with the
//                      bulk-copy (TMA) engine; 4R expander warps turn signs into e4m3 +-1 in a
//                      TMEM A slot (one slot = the unit's R tiles, 32 columns each); one MMA
//                      thread issues tcgen05.cp (SFB) + 4 R x (MMAs per 48 NB columns) per unit
//                      (16 MMAs per hand-off at batch 1) into R fp32 TMEM accumulators; 4
//                      epilogue warps drain the accumulators at each block end
//                      (y += sum_r U'[j, r] sum_d T[j, (b, d, r)]) while the expanders keep
//                      filling the other slot; split-K partials reduced deterministically by
//                      the last CTA of each row group (decode_tc.cuh finalize_group).
// Launch: zq_mx (PDL trigger at entry) then decode_mx with programmatic stream
// serialization; only the producer's Zq copies wait (griddepcontrol.wait).
#pragma once
#include <cuda_fp8.h>

#include "decode_tc.cuh"

namespace bs {

// ------------------------------------------------------------------ operand geometry
// Column n of a Zq unit = b * 48 + d * 16 + r (token b, digit d, rank r).
// B image: (n, k) at ((k / 16) (N / 8) + n / 8) 128 + (n % 8) 16 + k % 16 (K-major, no swizzle).
// SFB chunk h (columns [128 h, 128 h + 128)): (n, kb) at 512 h + 16 (n % 32) + 4 ((n % 128) / 32) + kb.
template <int NB>
struct MxCfg {
  static constexpr int N = 48 * NB;
  static constexpr int NCH = (N + 127) / 128;
  static constexpr int kB = kSubK * N;
  static constexpr int kUnit = kB + 512 * NCH;
  static constexpr uint32_t LBO = (N / 8) * 128;   // K-adjacent core matrices
  static constexpr uint32_t SBO = 128;             // N-adjacent core matrices
  // MMA split of the N columns: first 256, then the rest (each start a multiple of 128 so that
  // its SFB chunks line up with the MMA's local columns)
  static constexpr int NM = N > 256 ? 2 : 1;
  static constexpr int N0 = N > 256 ? 256 : N;
  static constexpr int N1 = N - N0;
  static_assert(N0 % 16 == 0 && N1 % 16 == 0 && N1 <= 256, "MMA N");
};

// kind::mxf8f6f4 instruction descriptor: e4m3 x e4m3 -> f32, K-major, UE8M0 scales, M = 128,
// scale-factor byte ids (the K-block inside the 4-byte TMEM scale cell).
__host__ __device__ constexpr uint32_t idesc_mx(uint32_t N, uint32_t sf_id) {
  return (sf_id << 4) | ((N >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24) | (sf_id << 29);
}
__device__ __forceinline__ void mma_mx_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// 32 lanes x 16 B from shared memory, broadcast to the 4 lane quadrants of TMEM columns [c, c + 4).
__device__ __forceinline__ void utccp_sf(uint32_t taddr, uint32_t saddr) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr),
               "l"(smem_desc_kmajor(saddr, 128, 128))
               : "memory");
}

// 16 consecutive factor entries (bf16 / f16 / f32 storage) as fp32.
__device__ __forceinline__ void load_f16x(const void* base, int fdt, long long row, float (&f)[16]) {
  if (fdt == 0) {
    const float4* p = reinterpret_cast<const float4*>(base) + row * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 v = __ldg(p + e);
      f[4 * e] = v.x; f[4 * e + 1] = v.y; f[4 * e + 2] = v.z; f[4 * e + 3] = v.w;
    }
    return;
  }
  const uint4* p = reinterpret_cast<const uint4*>(base) + row * 2;
  const uint4 a = __ldg(p), b = __ldg(p + 1);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float2 v;
    if (fdt == 1) v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
    else v = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
    f[2 * e] = v.x;
    f[2 * e + 1] = v.y;
  }
}

// 32 device-layout sign bits (F8 layout, aux_kernels.cuh: bit p of word w = column 32 w + 4 (p & 7)
// + (p >> 3)) -> 8 TMEM columns of e4m3 +-1.0 (byte = 0x38 | !bit << 7): per column one LOP3
// (alu pipe) isolates bits t, t+8, t+16, t+24 (inverted) and one IMAD (fma pipe) moves them to
// the byte sign bits and adds the exponent of 1.0.
// `one` = 1 arrives at run time (DecodeParams::one) so that ptxas keeps IMAD (fma pipe) instead
// of turning a constant power-of-two multiply-add into LEA (alu pipe, shared with the LOP3s).
__device__ __forceinline__ void expand_pm1(uint32_t w, uint32_t one, uint32_t* o /*8*/) {
  const uint32_t e8 = 0x38383838u;
#pragma unroll
  for (int t = 0; t < 7; ++t) o[t] = mad_lo(lop3_andnot(w, 0x01010101u << t), one << (7 - t), e8);
  o[7] = lop3_andnot_or(w, 0x80808080u, e8);
}

__device__ __forceinline__ float pow2f(int e) { return __uint_as_float((uint32_t)(e + 127) << 23); }  // |e| <= 126

// ------------------------------------------------------------------ Zq (prologue, H3)
struct ZqMxParams {
  const void* v;        // [n_cap x kh][d_in_pad][16] V'
  const float* inv_s;   // [d_in_pad]
  const void* x;        // [batch][x_stride]
  uint8_t* zq;          // [n x kh][nq] units of MxCfg<NB>::kUnit bytes
  long long x_stride;
  int nq, d_in, batch, x_dtype, f_dtype;
  int kfuse;            // k > 16 at batch 1: token slot b = rank half b of block i (x row 0)
};

// Persistent CTAs, one unit (block half i, 128-channel chunk q) at a time, 128 threads per token
// group (ZqTG<NB> groups; group g computes tokens g, g + TG, ...).  Thread t of a group holds 4
// consecutive channels 4 (t >> 2) .. +3 and the 4 ranks 4 (t & 3) .. +3, so warp w of a group is
// one 32-channel K-block: the block maximum of a rank is a 4-way local max plus 3 xor-shuffles
// over the 8 lanes of the same rank group, and each (rank, digit) is one 32-bit shared store (4
// channels are contiguous in the UMMA B image).  Units alternate between two shared tiles, one
// __syncthreads per unit; V' of the next unit is loaded before the current one is computed, and
// the copy of the finished tile to global overlaps the next unit.
template <int NB> struct ZqTG { static constexpr int value = NB >= 4 ? 4 : NB; };
template <int NB> __host__ __device__ constexpr int zq_threads() { return 128 * ZqTG<NB>::value; }
template <int NB> __host__ __device__ constexpr int zq_min_ctas() { return 1024 / zq_threads<NB>(); }   // <= 64 regs

// V' of one unit for thread (rank group rg, channel quad): 4 channels x 4 ranks, raw 16-bit pairs.
__device__ __forceinline__ void zq_load_v(const ZqMxParams& p, long long blk, int q, uint2 (&raw)[4]) {
  const int t = threadIdx.x & 127;
  const long long dpad = (long long)p.nq * kSubK;
  const int col0 = q * kSubK + 4 * (t >> 2);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    raw[j] = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(p.v) +
                                                  ((blk * dpad + col0 + j) * 16 + 4 * (t & 3))));
}

template <int NB>
__device__ __forceinline__ void zq_mx_unit(const ZqMxParams& p, const int i, const int q, uint8_t* tile,
                                           const uint2 (&raw0)[4]) {
  using C = MxCfg<NB>;
  constexpr int N = C::N, TG = ZqTG<NB>::value;
  const int t = threadIdx.x & 127, tg = threadIdx.x >> 7;
  const int lane = t & 31, rg = t & 3, cq = t >> 2, kb = cq >> 3;
  const int c0 = 4 * cq, col0 = q * kSubK + c0;
  float vv[4][4];   // [channel j][rank 4 rg + r]
  auto unpack = [&](const uint2 (&raw)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f0, f1;
      if (p.f_dtype == 1) {
        f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[j].x));
        f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[j].y));
      } else {
        f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw[j].x));
        f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw[j].y));
      }
      vv[j][0] = f0.x; vv[j][1] = f0.y; vv[j][2] = f1.x; vv[j][3] = f1.y;
    }
  };
  if (!p.kfuse) unpack(raw0);
  float is[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) is[j] = col0 + j < p.d_in ? __ldg(p.inv_s + col0 + j) : 0.f;
  const int kc = (c0 >> 4) * (N / 8) * 128 + (c0 & 15);   // byte offset of channel c0 in the B image
#pragma unroll 1
  for (int b = tg; b < NB; b += TG) {
    if (p.kfuse) {
      uint2 raw[4];
      zq_load_v(p, 2 * i + b, q, raw);
      unpack(raw);
    }
    const bool on = p.kfuse || b < p.batch;
    const long long xrow = (long long)(p.kfuse ? 0 : b) * p.x_stride;
    float xs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      xs[j] = (on && col0 + j < p.d_in) ? __fmul_rn(load_act(p.x, xrow + col0 + j, p.x_dtype), is[j]) : 0.f;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // digit 0 scale: sigma puts the K-block maximum of V'[:, r] x' into [128, 256) (clamped: a
      // K-block below 2^-106 keeps sigma = -113 and its tiny digits round to 0); digit d scales
      // by 2^(sigma - 4d): the previous digit's residual is at most half an e4m3 ulp (<= 8, then
      // <= 4, in its own units), so x16 keeps it inside e4m3 range.  A non-finite value becomes
      // NaN (e4m3 0x7f in every digit), so y is NaN as in the oracle.
      float val[4];
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        val[j] = __fmul_rn(vv[j][r], xs[j]);
        m = max(m, __float_as_uint(val[j]) & 0x7fffffffu);
      }
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 4));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 8));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 16));
      const int sig = min(max((int)(m >> 23) - 134, -113), 120);
      const float sc = pow2f(-sig);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        val[j] = fabsf(val[j]) <= 3.4028235e38f ? __fmul_rn(val[j], sc) : __uint_as_float(0x7fffffffu);
      const int n0 = b * 48 + 4 * rg + r;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const __nv_fp8x2_storage_t q01 =
            __nv_cvt_float2_to_fp8x2(make_float2(val[0], val[1]), __NV_SATFINITE, __NV_E4M3);
        const __nv_fp8x2_storage_t q23 =
            __nv_cvt_float2_to_fp8x2(make_float2(val[2], val[3]), __NV_SATFINITE, __NV_E4M3);
        const int n = n0 + 16 * d;
        *reinterpret_cast<uint32_t*>(tile + kc + (n / 8) * 128 + (n % 8) * 16) =
            (uint32_t)q01 | ((uint32_t)q23 << 16);
        if (d < 2) {   // exact: the residual of a 4-significant-bit rounding, times 16
          const float2 b01 = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(q01, __NV_E4M3)));
          const float2 b23 = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(q23, __NV_E4M3)));
          val[0] = __fmul_rn(__fsub_rn(val[0], b01.x), 16.f);
          val[1] = __fmul_rn(__fsub_rn(val[1], b01.y), 16.f);
          val[2] = __fmul_rn(__fsub_rn(val[2], b23.x), 16.f);
          val[3] = __fmul_rn(__fsub_rn(val[3], b23.y), 16.f);
        }
        if (lane < 4)   // lanes 0..3 (rank groups 0..3 of channel quad 0): this K-block's scale bytes
          tile[C::kB + 512 * (n / 128) + 16 * (n & 31) + 4 * ((n & 127) >> 5) + kb] = (uint8_t)(sig + 127 - 4 * d);
      }
    }
  }
}

// Units [0, units) of one layer (or of a group: `locate` maps a global unit to its parameters).
template <int NB, typename Locate>
__device__ __forceinline__ void zq_mx_loop(const int units, Locate locate) {
  using C = MxCfg<NB>;
  constexpr int N = C::N, NT = zq_threads<NB>();
  extern __shared__ __align__(128) uint8_t zq_tiles[];   // 2 x C::kUnit bytes
  asm volatile("griddepcontrol.launch_dependents;");
  // SFB bytes of columns >= N in the last chunk: defined (never used by an MMA), written once
  for (int t = 0; t < 2; ++t)
    for (int e = N + (int)threadIdx.x; e < 128 * C::NCH; e += NT)
      for (int k4 = 0; k4 < 4; ++k4)
        zq_tiles[t * C::kUnit + C::kB + 512 * (e / 128) + 16 * (e & 31) + 4 * ((e & 127) >> 5) + k4] = 0;
  int u = blockIdx.x;
  if (u >= units) return;
  const ZqMxParams* p;
  int lu;
  locate(u, p, lu);
  int bi = lu / p->nq, bq = lu - bi * p->nq;   // (block half, chunk) of the unit, once per unit
  uint2 raw[4];
  if (!p->kfuse) zq_load_v(*p, bi, bq, raw);
#pragma unroll 1
  for (int it = 0;; ++it) {
    const int un = u + gridDim.x;
    const ZqMxParams* pn = p;
    int lun = 0, bin = 0, bqn = 0;
    uint2 rawn[4];
    if (un < units) {   // next unit's V' in flight while this one is computed
      locate(un, pn, lun);
      bin = lun / pn->nq;
      bqn = lun - bin * pn->nq;
      if (!pn->kfuse) zq_load_v(*pn, bin, bqn, rawn);
    }
    uint8_t* tile = zq_tiles + (it & 1) * C::kUnit;
    zq_mx_unit<NB>(*p, bi, bq, tile, raw);
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(p->zq + (long long)lu * C::kUnit);
    for (int e = threadIdx.x; e < C::kUnit / 16; e += NT) dst[e] = reinterpret_cast<const uint4*>(tile)[e];
    if (un >= units) break;
    u = un;
    p = pn;
    lu = lun;
    bi = bin;
    bq = bqn;
#pragma unroll
    for (int j = 0; j < 4; ++j) raw[j] = rawn[j];
  }
}

template <int NB>
__global__ void __launch_bounds__(zq_threads<NB>(), zq_min_ctas<NB>()) zq_mx_kernel(const __grid_constant__ ZqMxParams p, const int units) {
  zq_mx_loop<NB>(units, [&](int u, const ZqMxParams*& pp, int& lu) { pp = &p; lu = u; });
}

constexpr int kMaxMxGroup = 8;
struct ZqMxGroup {
  int count;
  int unit_start[kMaxMxGroup + 1];
  ZqMxParams prm[kMaxMxGroup];
};
template <int NB>
__global__ void __launch_bounds__(zq_threads<NB>(), zq_min_ctas<NB>()) zq_mx_grouped_kernel(const __grid_constant__ ZqMxGroup grp) {
  zq_mx_loop<NB>(grp.unit_start[grp.count], [&](int u, const ZqMxParams*& pp, int& lu) {
    int i = 0;
    while (i + 1 < grp.count && u >= grp.unit_start[i + 1]) ++i;
    pp = &grp.prm[i];
    lu = u - grp.unit_start[i];
  });
}

// ------------------------------------------------------------------ decode kernel (H4-H7)
template <int NB> struct MxGeom;                        // row tiles per CTA by batch class
#ifndef BS_MX_R1
#define BS_MX_R1 4
#endif
#ifndef BS_MX_OCC1
#define BS_MX_OCC1 1
#endif
template <> struct MxGeom<1> { static constexpr int R = BS_MX_R1, OCC = BS_MX_OCC1; };
template <> struct MxGeom<2> { static constexpr int OCC = 1, R = 2; };
template <> struct MxGeom<3> { static constexpr int OCC = 1, R = 2; };
template <> struct MxGeom<4> { static constexpr int OCC = 1, R = 1; };
template <> struct MxGeom<5> { static constexpr int OCC = 1, R = 1; };
template <> struct MxGeom<6> { static constexpr int OCC = 1, R = 1; };
template <> struct MxGeom<7> { static constexpr int OCC = 1, R = 1; };
template <> struct MxGeom<8> { static constexpr int OCC = 1, R = 1; };

#ifndef BS_MX_SMEM_KB
#define BS_MX_SMEM_KB 200
#endif
#ifndef BS_MX_STAGES
#define BS_MX_STAGES 8
#endif

// Warp roles (R row tiles per CTA).  Synchronisation operations per unit are the cost that
// bounds this kernel (scripts/sync_probe.cu, mbar_tput.cu: a completed-phase wait ~90 cycles of
// latency, an arrive ~7 cycles of the SM's synchronisation unit), so few, fat warps hand off
// large pieces of work:
//   warps 0 .. 4NI-1   expanders: warp w owns TMEM lane quadrant w % 4 of the TPI tiles of
//                      issuer group w / 4; per unit it expands its 32 rows of those tiles and
//                      arrives once (two warps per SMSP keep the LOP3 -> IMAD chains busy)
//   next NI warps      issuers: issuer i owns TPI consecutive tiles (their accumulators, A slots
//                      and SFB copies); per unit one wait, one tcgen05.cp, 4 TPI MMAs, 2 commits
//   next 4 warps       epilogue (lane quadrant warp % 4, all tiles)
//   last warp          producer (bulk copies; allocates TMEM)
template <int NB>
struct DecodeMxCfg {
  using Z = MxCfg<NB>;
  static constexpr int N = Z::N, R = MxGeom<NB>::R;
#ifndef BS_MX_TPI
#define BS_MX_TPI 1
#endif
  static constexpr int TPI = R >= BS_MX_TPI ? BS_MX_TPI : 1;   // tiles per issuer
  static constexpr int NI = R / TPI;                   // issuers
  static_assert(R % TPI == 0, "tiles per issuer");
  static constexpr int kWarpIss = 4 * NI;
  static constexpr int kWarpEpi = 5 * NI;
  static constexpr int kWarpProd = 5 * NI + 4;
  static constexpr int kThreads = 32 * (5 * NI + 5);
  static constexpr int kSignBytes = R * kTileRows * 16;
  static constexpr int kStageBytes = (kSignBytes + Z::kUnit + 1023) / 1024 * 1024;
  static constexpr int OCC = MxGeom<NB>::OCC;         // resident CTAs per SM (TMEM / smem split)
  static constexpr int kTmemCols = 512 / OCC;
  static constexpr int S0 = BS_MX_SMEM_KB * 1024 / OCC / kStageBytes;
  static constexpr int STAGES = S0 > BS_MX_STAGES ? BS_MX_STAGES : (S0 < 2 ? 2 : S0);
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarBytes + 1024;   // + alignment slack
  // TMEM columns: A slots [slot][tile] (32 each) | accumulators [t] (N each) | SFA (4) | SFB [i][slot]
  static constexpr int kSfCols = 4 * Z::NCH;
  static constexpr int NS0 = (kTmemCols - R * N - 4) / (R * 32 + NI * kSfCols);
#ifndef BS_MX_NSLOT
#define BS_MX_NSLOT 4
#endif
  static constexpr int NSLOT = NS0 > BS_MX_NSLOT ? BS_MX_NSLOT : NS0;
  static constexpr uint32_t kColAcc = NSLOT * R * 32;
  static constexpr uint32_t kColSfa = kColAcc + R * N;
  static constexpr uint32_t kColSfb = kColSfa + 4;
  static_assert(NSLOT >= 2, "need a double-buffered A slot");
  static_assert(kColSfb + NI * NSLOT * kSfCols <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes <= 227 * 1024, "smem overflow");
  static_assert(R * kTileRows * NB <= kPartStride, "split-K slot");
};

template <int NB>
__device__ __forceinline__ void decode_mx_body(const DecodeParams& p, const int cta) {
  using C = DecodeMxCfg<NB>;
  using Z = MxCfg<NB>;
  constexpr int N = C::N, R = C::R, STAGES = C::STAGES, NSLOT = C::NSLOT, TPI = C::TPI, NI = C::NI;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* full = bars;                     // [STAGES] sign tiles + Zq unit landed (tx)
  uint64_t* sempty = full + STAGES;          // [STAGES] one commit per active issuer
  uint64_t* aempty = sempty + STAGES;        // [NI][NSLOT] commit after the group's MMAs on the slot
  uint64_t* afull = aempty + NI * NSLOT;     // [NI][NSLOT] the 4 expander warps stored the group's tiles
  uint64_t* accfull = afull + NI * NSLOT;    // [R] commit at a block's last unit
  uint64_t* accempty = accfull + R;          // [R] 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + R);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = cta / p.ctas_per_group;
  const int jc = cta % p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const long long u0 = L * jc / p.ctas_per_group;
  const int nunits = (int)(L * (jc + 1) / p.ctas_per_group - u0);
  const int i_start = (int)(u0 / p.nq), q_start = (int)(u0 % p.nq);
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int NIg = (Rg + TPI - 1) / TPI;              // active issuers
  const int row0 = g * R * kTileRows;
#ifdef BS_MX_TRACE   // timing build (scripts/mx_trace.py): per-unit clock64 stamps of CTA 0
  long long* trace = (p.dbg_acc && cta == 0) ? reinterpret_cast<long long*>(p.dbg_acc) : nullptr;
  __shared__ long long tstart_sh;
  if (threadIdx.x == 0) tstart_sh = clock64();
  __syncthreads();
  const long long tstart = tstart_sh;
#define BS_TR(k_, c_) do { if (trace && (k_) < 4000) trace[(k_) * 16 + (c_)] = clock64() - tstart; } while (0)
  if (p.dbg_acc && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta] = (long long)gt;
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta + 2] = nunits;
  }
#else
#define BS_TR(k_, c_) do { } while (0)
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sempty[s], NIg);
    }
    for (int a = 0; a < NI * NSLOT; ++a) {
      mbar_init(&aempty[a], 1);
      mbar_init(&afull[a], 4);
    }
    for (int t = 0; t < R; ++t) {
      mbar_init(&accfull[t], 1);
      mbar_init(&accempty[t], 4);
    }
    fence_mbar_init();
  }
  if (warp == C::kWarpProd) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (warp >= C::kWarpEpi && warp < C::kWarpEpi + 4) {
    // scale_A = 1.0 (UE8M0 127) in every byte of the 4 SFA columns, lane quadrant warp % 4
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(
                     tbase + ((uint32_t)((warp & 3) * 32) << 16) + C::kColSfa),
                 "r"(0x7f7f7f7fu)
                 : "memory");
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == C::kWarpProd) {
    // ================= producer: sign tiles now, Zq units after the Zq grid completed
    if (lane == 0) {
      const uint64_t pol_sign = policy_evict_first();
      const uint64_t pol_zq = policy_evict_last();
      const uint32_t sign_bytes = (uint32_t)Rg * kTileRows * 16;
      int q = q_start, iv = i_start;
      const int pre = nunits < STAGES ? nunits : STAGES;
#define SIGN_ADDR (p.signs + ((long long)(iv >> p.ksh) * p.nq + q) * p.rows_pad + row0)
      for (int k = 0; k < pre; ++k) {   // sign tiles of the first units before the dependency wait
        mbar_arrive_expect_tx(&full[k], sign_bytes + Z::kUnit);
        bulk_g2s(smem + k * C::kStageBytes, SIGN_ADDR, sign_bytes, &full[k], pol_sign);
        if (++q == p.nq) { q = 0; ++iv; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");   // this call's Zq units are complete
      for (int k = 0; k < pre; ++k)
        bulk_g2s(smem + k * C::kStageBytes + C::kSignBytes, p.zq + (u0 + k) * Z::kUnit, Z::kUnit, &full[k], pol_zq);
      int s = pre % STAGES;
      uint32_t ph = pre == STAGES ? 1u : 0u;
      for (int k = pre; k < nunits; ++k) {
        mbar_wait(&sempty[s], ph ^ 1);
        BS_TR(k, 0);
        uint8_t* st = smem + s * C::kStageBytes;
#if defined(BS_MX_EXP_NODATA)   // timing experiment: no copies after the first ring fill (wrong values)
        mbar_arrive(&full[s]);
#else
        mbar_arrive_expect_tx(&full[s], sign_bytes + Z::kUnit);
        bulk_g2s(st + C::kSignBytes, p.zq + (u0 + k) * Z::kUnit, Z::kUnit, &full[s], pol_zq);
        bulk_g2s(st, SIGN_ADDR, sign_bytes, &full[s], pol_sign);
#endif
        if (++q == p.nq) { q = 0; ++iv; }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
#undef SIGN_ADDR
    }
  } else if (warp < C::kWarpIss) {
    // ================= expander warp: TMEM lane quadrant qd of the tiles of issuer group gi
    const int qd = warp & 3, gi = warp >> 2;
    if (gi < NIg) {
      const uint32_t sw0 = smem_u32(smem) + (uint32_t)((qd * 32 + lane) * 16);
      const uint32_t one = p.one;
      const uint32_t a0 = tbase + ((uint32_t)(qd * 32) << 16);
      int s = 0, a = 0;
      uint32_t ph = 0, aph = 0;
      for (int k = 0; k < nunits; ++k) {
        // the try_waits go out first so that their latency overlaps the loads and the expansion
        const bool landed = mbar_try_wait(&full[s], ph);
        const bool sfree = k < NSLOT || mbar_try_wait(&aempty[gi * NSLOT + a], aph ^ 1);
        if (!landed) mbar_wait(&full[s], ph);
        if (warp == 0 && lane == 0) BS_TR(k, 1);
        const uint32_t sw = sw0 + (uint32_t)(s * C::kStageBytes);
        uint4 w[TPI];
#pragma unroll
        for (int tt = 0; tt < TPI; ++tt)
          if (gi * TPI + tt < Rg)
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(w[tt].x), "=r"(w[tt].y), "=r"(w[tt].z), "=r"(w[tt].w)
                         : "r"(sw + (uint32_t)((gi * TPI + tt) * kTileRows * 16)));
#pragma unroll
        for (int tt = 0; tt < TPI; ++tt) {
          const int t = gi * TPI + tt;
          if (t < Rg) {
            uint32_t o[32];
#ifndef BS_MX_EXP_NOEXP
            expand_pm1(w[tt].x, one, o);
            expand_pm1(w[tt].y, one, o + 8);
            expand_pm1(w[tt].z, one, o + 16);
            expand_pm1(w[tt].w, one, o + 24);
#else
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = w[tt].x;
#endif
            if (tt == 0) {
              if (!sfree) mbar_wait(&aempty[gi * NSLOT + a], aph ^ 1);
              tc_fence_after();
            }
#ifndef BS_MX_EXP_NOST
            tmem_st32(a0 + (uint32_t)((a * R + t) * 32), o);
#else
            if ((o[0] ^ o[31]) == 0x12345u) p.y_part[0] = 1.f;
#endif
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[gi * NSLOT + a]);
        if (warp == 0 && lane == 0) BS_TR(k, 3);
        if (++s == STAGES) { s = 0; ph ^= 1; }
        if (++a == NSLOT) { a = 0; aph ^= 1; }
      }
    }
  } else if (warp < C::kWarpEpi) {
    // ================= issuer i: tiles [i TPI, (i+1) TPI); per unit one wait for the group's
    // A slot, then tcgen05.cp (SFB) + 4 TPI MMAs from one elected lane and the commits that
    // release the slot, the stage and (at a block end) the accumulators
    const int i = warp - C::kWarpIss;
    if (i < NIg) {
      const uint32_t sfa = tbase + C::kColSfa;
      int s = 0, a = 0, q = q_start, seg = 0;
      uint32_t aph = 0;
      for (int k = 0; k < nunits; ++k) {
        const bool first = (k == 0) || (q == 0);
        const bool last = (k + 1 == nunits) || (q + 1 == p.nq);
        if (i == 0 && lane == 0) BS_TR(k, 8);
        const bool ready = mbar_try_wait(&afull[i * NSLOT + a], aph);
        if (first && seg > 0) {
#pragma unroll
          for (int tt = 0; tt < TPI; ++tt)
            if (i * TPI + tt < Rg) mbar_wait(&accempty[i * TPI + tt], (seg - 1) & 1);
        }
        if (!ready) mbar_wait(&afull[i * NSLOT + a], aph);
        if (i == 0 && lane == 0) BS_TR(k, 5);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t zs = smem_u32(smem + s * C::kStageBytes + C::kSignBytes);
          const uint32_t sfb = tbase + C::kColSfb + (uint32_t)((i * NSLOT + a) * C::kSfCols);
#ifndef BS_MX_EXP_NOCP
#pragma unroll
          for (int h = 0; h < Z::NCH; ++h) utccp_sf(sfb + 4 * h, zs + Z::kB + 512 * h);
#endif
          const uint64_t bdesc = smem_desc_kmajor(zs, Z::LBO, Z::SBO);
#pragma unroll
          for (int tt = 0; tt < TPI; ++tt) {
            const int t = i * TPI + tt;
            if (t < Rg) {
              const uint32_t dacc = tbase + C::kColAcc + (uint32_t)(t * N);
              const uint32_t acol = tbase + (uint32_t)((a * R + t) * 32);
#pragma unroll
              for (int kb = 0; kb < 4; ++kb) {
                const uint32_t acc = (first && kb == 0) ? 0u : 1u;
                const uint64_t bk = bdesc + (uint64_t)((kb * 2 * Z::LBO) >> 4);
#ifndef BS_MX_EXP_NOMMA
                mma_mx_ts(dacc, acol + (uint32_t)(kb * 8), bk, idesc_mx(Z::N0, kb), sfa | ((uint32_t)kb << 30),
                          sfb | ((uint32_t)kb << 30), acc);
                if constexpr (Z::NM == 2)
                  mma_mx_ts(dacc + Z::N0, acol + (uint32_t)(kb * 8), bk + (uint64_t)(((Z::N0 / 8) * 128) >> 4),
                            idesc_mx(Z::N1, kb), sfa | ((uint32_t)kb << 30), (sfb + 8) | ((uint32_t)kb << 30), acc);
#else
                (void)acc; (void)bk; (void)dacc; (void)acol;
#endif
              }
            }
          }
          mma_commit(&aempty[i * NSLOT + a]);
          mma_commit(&sempty[s]);
          if (last) {
#pragma unroll
            for (int tt = 0; tt < TPI; ++tt)
              if (i * TPI + tt < Rg) mma_commit(&accfull[i * TPI + tt]);
          }
          if (i == 0) BS_TR(k, 7);
        }
        __syncwarp();
        if (last) ++seg;
        if (++q == p.nq) q = 0;
        if (++s == STAGES) s = 0;
        if (++a == NSLOT) { a = 0; aph ^= 1; }
      }
    }
  } else if (warp < C::kWarpProd) {
    // ================= epilogue warps: lane quadrant e, all R tiles
    const int e = warp & 3;
    const uint32_t lq = (uint32_t)(e * 32) << 16;
    float yacc[R][NB];
#pragma unroll
    for (int t = 0; t < R; ++t)
#pragma unroll
      for (int b = 0; b < NB; ++b) yacc[t][b] = 0.f;
    int k = 0, q = q_start, i = i_start, seg = 0;
    while (k < nunits) {
      const int cnt = (nunits - k) < (p.nq - q) ? (nunits - k) : (p.nq - q);   // units of block i here
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (t < Rg) {
          const long long row = row0 + t * kTileRows + e * 32 + lane;
          float uu[16];
          if (!p.kfuse) load_f16x(p.u, p.f_dtype, (long long)i * p.rows_pad + row, uu);
          mbar_wait(&accfull[t], seg & 1);
          tc_fence_after();
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (p.kfuse) load_f16x(p.u, p.f_dtype, (long long)(2 * i + b) * p.rows_pad + row, uu);
            uint32_t v0[16], v1[16], v2[16];
            const uint32_t base = tbase + lq + C::kColAcc + (uint32_t)(t * N + b * 48);
            tmem_ld16(base, v0);
            tmem_ld16(base + 16, v1);
            tmem_ld16(base + 32, v2);
            tmem_ld_wait();
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r)
              acc = fmaf(uu[r], __uint_as_float(v0[r]) + __uint_as_float(v1[r]) + __uint_as_float(v2[r]), acc);
            if (p.kfuse) yacc[t][0] += acc;
            else yacc[t][b] += acc;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&accempty[t]);
        }
      }
      ++seg;
      k += cnt;
      q += cnt;
      if (q == p.nq) { q = 0; ++i; }
    }
#pragma unroll
    for (int t = 0; t < R; ++t)
      if (t < Rg)
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < p.batch) store_partial(p, cta, R * kTileRows, t * kTileRows + e * 32 + lane, b, yacc[t][b]);
  }

  // ---- teardown + last-CTA-of-group finalisation (deterministic split-K, H7)
#ifdef BS_MX_TRACE
  if (p.dbg_acc && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta + 1] = (long long)gt;
  }
#endif
#undef BS_TR
  __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kWarpProd) tmem_dealloc<C::kTmemCols>(tbase);
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(p.counters + g, 1);
    *last_flag = (prev == p.ctas_per_group - 1);
  }
  __syncthreads();
  if (*last_flag) {
    __threadfence();
    finalize_group(p, g, R * kTileRows, Rg, row0);
    if (threadIdx.x == 0) p.counters[g] = 0;
  }
}

template <int NB>
__global__ void __launch_bounds__(DecodeMxCfg<NB>::kThreads, DecodeMxCfg<NB>::OCC) decode_mx_kernel(const DecodeParams p) {
  decode_mx_body<NB>(p, (int)blockIdx.x);
}

struct DecodeMxGroup {
  int count;
  int cta_start[kMaxMxGroup + 1];
  DecodeParams prm[kMaxMxGroup];
};
template <int NB>
__global__ void __launch_bounds__(DecodeMxCfg<NB>::kThreads, DecodeMxCfg<NB>::OCC) decode_mx_grouped_kernel(
    const __grid_constant__ DecodeMxGroup grp) {
  int i = 0;
  while (i + 1 < grp.count && (int)blockIdx.x >= grp.cta_start[i + 1]) ++i;
  decode_mx_body<NB>(grp.prm[i], (int)blockIdx.x - grp.cta_start[i]);
}

}  // namespace bs
