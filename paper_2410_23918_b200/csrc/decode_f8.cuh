// tcgen05 decode kernel, e4m3 variant: the production decode path for bf16/f16 factors.
//
// Same computation as decode_tc.cuh (Eq.4, Eq.7, Eq.8; y = sum_i sum_r U'_i[:,r] *
// (S_i (V'_i[:,r] * x/s))), mapped differently onto the tensor core because a
// tcgen05.mma costs ~19 cycles minimum per instruction (scripts/mma_issue_bench.cu):
// with kind::f16 and N = 16 (rank k at batch 1) that caps the kernel at 128x16 sign
// elements per 19 cycles.  kind::f8f6f4 has K = 32 per instruction:
//   * A = S as e4m3 +-2^delta (1 byte per sign, half the tcgen05.st traffic and half the
//     expansion ALU work of fp16: 8 LOP3 + 7 IMAD per 32 signs),
//   * B = Z as THREE e4m3 digits (N = 48 per batch column): Z 2^E ~= d0 + d1 + d2 with
//     d_t = e4m3(residual_t), ~12 significant bits (precision study: 6.4e-5 rel-L2 vs
//     2.6e-4 for one fp16 digit),
//   * 24.9 cycles per MMA (N = 48) -> 164 sign elements / clk / SM at the tensor floor.
// Two kernels:
//   zq_kernel<NB>      once per call: for every (block i, 128-column subchunk q) unit,
//                      Z = V'_i (.) x/s, its max, a per-unit exponent e_u putting max|Z 2^e_u|
//                      in (224, 448], and the three round-to-nearest e4m3 digits, written
//                      as a ready-to-copy UMMA B tile (+16 B of metadata) -- built ONCE per
//                      unit instead of once per row group;
//   decode kernel      bulk-copies sign tiles + Zq tiles (TMA engine), expands signs to
//                      e4m3 +-2^a_u in TMEM, a_u = E - e_u (E = the CTA's first unit's e_u),
//                      so A*B = +-Z 2^E for every unit; the epilogue multiplies by 2^-E.
//                      The production schedule is decode_f8i_kernel (decode_f8i.cuh: one MMA
//                      issuer warp per warpgroup); decode_f8_kernel below (self-issuing
//                      warpgroups) stays selectable with BS_DECODE_WG=1 for A/B runs.
// The decode kernel is launched with programmatic dependent launch: its setup and first
// sign loads overlap the Zq kernel; only the Zq copies wait (griddepcontrol.wait).
#pragma once
#include <cuda_fp8.h>

#include "decode_tc.cuh"

namespace bs {

// Device sign layout for this kernel ("F8 layout"): bit p of word w of a row's 128-column
// subchunk holds column 32 w + 4 (p & 7) + (p >> 3), so that one LOP3 + one IMAD turn
// bits (t, t+8, t+16, t+24) into the 4 bytes of TMEM column 8 w + t (K elements 4t..4t+3).
__device__ __forceinline__ void expand_e4m3(uint32_t w, uint32_t e8, uint32_t* o /*8*/) {
#pragma unroll
  for (int t = 0; t < 7; ++t) o[t] = mad_lo(lop3_andnot(w, 0x01010101u << t), 1u << (7 - t), e8);
  o[7] = lop3_andnot_or(w, 0x80808080u, e8);
}

// Round-to-nearest to 4 significant bits (the e4m3 significand) by Veltkamp splitting,
// in plain fp32 arithmetic (no FMA contraction): exact for |z| < 2^100.
__device__ __forceinline__ float rn4(float z) {
  const float t = __fmul_rn(z, 1048577.0f);  // 2^20 + 1
  return __fsub_rn(t, __fsub_rn(t, z));
}



constexpr int kZqSentinel = 127;         // e_u of an all-zero unit

// Zq unit geometry (depends on the batch width only).
template <int NB>
struct ZqCfg {
  static constexpr int N = 48 * NB;                          // 3 digits x 16 ranks x batch
  static constexpr int kZBytes = kSubK * N;                  // e4m3 B tile of one unit
  static constexpr int kZUnit = kZBytes + 16;                // + metadata (int32 e_u)
};

// Self-issuing warpgroups.  Warpgroup w (warps 4w..4w+3, TMEM lane
// quadrant = warp % 4) owns row tile w of the CTA's R tiles: for every unit it expands
// its 128x128 sign tile into an e4m3 A slot in TMEM, syncs its own 4 warps on a named
// barrier, and one elected thread of the warpgroup issues the tile's 4 MMAs itself --
// there is no cross-warp handshake with a separate MMA warp (whose round trip, ~300-500
// cycles, dwarfed the 100 cycles of MMA work per tile).  Each warpgroup keeps a 2-slot A
// ring released by its own tcgen05.commit, and its own accumulator (no cross-issuer
// hazards).  TMEM: R x N accumulator columns + R x NSLOT x 32 A columns <= 512.
template <int NB, int R_, int P_ = 1>
struct DecodeF8Cfg {
  static constexpr int N = ZqCfg<NB>::N;
  static constexpr int P = P_;                               // units per warpgroup iteration
  static constexpr int R = R_;                               // row tiles = warpgroups
  static constexpr int kThreads = 32 * (4 * R + 1);          // + producer warp
  static constexpr int kWarpProducer = 4 * R;
  static constexpr int kZBytes = ZqCfg<NB>::kZBytes;
  static constexpr int kZUnit = ZqCfg<NB>::kZUnit;
  static constexpr int kSignBytes = R * kTileRows * 16;
  static constexpr int kOffZ = kSignBytes;
  static constexpr int kOffMeta = kOffZ + kZBytes;
  static constexpr int kStageBytes = (kOffZ + kZUnit + 127) / 128 * 128;
  static constexpr int S0 = (200 * 1024) / kStageBytes;
  static constexpr int STAGES = S0 > 12 ? 12 : (S0 < 2 ? 2 : S0);
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarBytes;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kACols = 32;                          // 128 rows x 128 e4m3 per tile
  static constexpr int NS0 = (512 - R * N) / (R * P * kACols);
  static constexpr int NSLOT = NS0 > 4 ? 4 : NS0;            // A slots (of P tiles) per warpgroup
  static constexpr uint32_t kAccCol = R * NSLOT * P * kACols;
  static constexpr uint32_t LBO = (N / 8) * 128;
  static constexpr uint32_t SBO = 128;
  static_assert(N <= 256 && N % 16 == 0, "invalid MMA N");
  static_assert(NSLOT >= (P == 1 ? 2 : 1), "need at least double-buffered A");
  static_assert(kAccCol + R * N <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes <= 227 * 1024, "smem overflow");
  static_assert(R >= 1 && R <= 7, "named barriers 1..R");
};

struct ZqParams {
  const void* v;        // [n_cap][d_in_pad][16] V' (bf16 or f32)
  const float* inv_s;   // [d_in_pad]
  const void* x;        // [batch][x_stride]
  uint8_t* zq;          // [n][nq] units of kZUnit bytes
  long long x_stride;
  int nq, d_in, d_in_pad, batch, x_dtype, f_dtype;
  int kfuse;            // 1: k > 16 at batch 1 -- column b of the NB = 2 layout is rank half b of
                        //    block i (internal block 2 i + b), all on x row 0
};

// One CTA per unit (block i, subchunk q); thread c = column q*128 + c.
template <int NB>
__device__ __forceinline__ void zq_body(const ZqParams& p, const int unit) {
  using C = ZqCfg<NB>;
  constexpr int N = C::N;
  __shared__ __align__(16) uint8_t tile[C::kZBytes];
  __shared__ float red[4];
  asm volatile("griddepcontrol.launch_dependents;");
  const int i = unit / p.nq, q = unit % p.nq;
  const int c = threadIdx.x;
  const int col = q * kSubK + c;
  float vv[16];
  auto load_v = [&](int blk) {
    const long long base = ((long long)blk * p.d_in_pad + col) * 16;
    if (p.f_dtype == 1) {
      const uint4* vp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.v) + base);
      const uint4 a = __ldg(vp), b = __ldg(vp + 1);
      const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f0 = __bfloat1622float2(h0[e]), f1 = __bfloat1622float2(h1[e]);
        vv[2 * e] = f0.x; vv[2 * e + 1] = f0.y; vv[8 + 2 * e] = f1.x; vv[8 + 2 * e + 1] = f1.y;
      }
    } else {
      const float4* vp = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.v) + base);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 f = __ldg(vp + e);
        vv[4 * e] = f.x; vv[4 * e + 1] = f.y; vv[4 * e + 2] = f.z; vv[4 * e + 3] = f.w;
      }
    }
  };
  if (!p.kfuse) load_v(i);
  const float is = col < p.d_in ? __ldg(p.inv_s + col) : 0.f;
  float z[NB][16];
  float m = 0.f;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (p.kfuse) load_v(2 * i + b);
    const int xb = p.kfuse ? 0 : b;
    const bool on = p.kfuse ? true : b < p.batch;
    const float xs = (on && col < p.d_in) ? load_act(p.x, (long long)xb * p.x_stride + col, p.x_dtype) * is : 0.f;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      z[b][r] = vv[r] * xs;
      m = fmaxf(m, fabsf(z[b][r]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((c & 31) == 0) red[c >> 5] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  int e_u = kZqSentinel;
  if (m > 0.f && isfinite(m)) {
    e_u = (int)floorf(log2f(448.0f / m));
    if (__fmul_rn(m, exp2f((float)e_u)) > 448.0f) e_u -= 1;   // guard log2 rounding
    e_u = e_u > 100 ? 100 : (e_u < -100 ? -100 : e_u);
  }
  const float sc = e_u == kZqSentinel ? 0.f : exp2f((float)e_u);
  const int kg = c >> 4, kk = c & 15;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const float zz = __fmul_rn(z[b][r], sc);
      const float d0 = rn4(zz);
      const float r1 = __fsub_rn(zz, d0);
      const float d1 = rn4(r1);
      const float d2 = __fsub_rn(r1, d1);
      const float dg[3] = {d0, d1, d2};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int n = (b * 3 + d) * 16 + r;
        const __nv_fp8_storage_t byte = __nv_cvt_float_to_fp8(dg[d], __NV_SATFINITE, __NV_E4M3);
        tile[(kg * (N / 8) + n / 8) * 128 + (n % 8) * 16 + kk] = byte;
      }
    }
  }
  __syncthreads();
  uint8_t* dst = p.zq + (long long)unit * C::kZUnit;
  for (int e = c; e < C::kZBytes / 16; e += 128)
    reinterpret_cast<uint4*>(dst)[e] = reinterpret_cast<const uint4*>(tile)[e];
  if (c == 0) reinterpret_cast<int4*>(dst + C::kZBytes)[0] = make_int4(e_u, 0, 0, 0);
}

template <int NB>
__global__ void __launch_bounds__(128) zq_kernel(const ZqParams p) {
  zq_body<NB>(p, (int)blockIdx.x);
}

// Grouped Zq (bitstack_matmul_grouped): units [unit_start[i], unit_start[i+1]) belong to layer i.
constexpr int kMaxZqGroup = 8;
struct ZqGroup {
  int count;
  int unit_start[kMaxZqGroup + 1];
  ZqParams prm[kMaxZqGroup];
};

template <int NB>
__global__ void __launch_bounds__(128) zq_grouped_kernel(const __grid_constant__ ZqGroup grp) {
  int i = 0;
  while (i + 1 < grp.count && (int)blockIdx.x >= grp.unit_start[i + 1]) ++i;
  zq_body<NB>(grp.prm[i], (int)blockIdx.x - grp.unit_start[i]);
}

template <int NB, int R_>
__global__ void __launch_bounds__(DecodeF8Cfg<NB, R_>::kThreads, 1) decode_f8_kernel(const DecodeParams p) {
  using C = DecodeF8Cfg<NB, R_>;
  constexpr int N = C::N, R = C::R, STAGES = C::STAGES, NSLOT = C::NSLOT, P = C::P;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_empty = empty + STAGES;     // [R warpgroups][NSLOT]
  uint64_t* acc_full = a_empty + R * NSLOT; // [R]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + R);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int g = blockIdx.x / p.ctas_per_group;
  const int jc = blockIdx.x % p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const long long u0 = L * jc / p.ctas_per_group;
  const long long u1 = L * (jc + 1) / p.ctas_per_group;
  const int nunits = (int)(u1 - u0);
  const int i_start = (int)(u0 / p.nq), q_start = (int)(u0 % p.nq);
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int row0 = g * R * kTileRows;
#ifdef BS_DECODE_TRACE
  // debug build only (scripts/trace_f8.py): CTA 0 timeline of warpgroup 3, clock64 relative
  // to kernel entry, 16 slots per unit, written to the bitstack_debug_set buffer; every
  // CTA's entry / exit %globaltimer (ns) at slots 65536 + 4 * blockIdx.x
  long long* trace = (p.dbg_acc && blockIdx.x == 0) ? reinterpret_cast<long long*>(p.dbg_acc) : nullptr;
  const long long tstart = clock64();
  if (p.dbg_acc && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * blockIdx.x] = (long long)gt;
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * blockIdx.x + 2] = nunits;
  }
#define BS_TRACE(k_unit, k) do { if (warp == 12 && trace && lane == 0) trace[(k_unit) * 16 + (k)] = clock64() - tstart; } while (0)
#else
#define BS_TRACE(k_unit, k) do { } while (0)
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Rg);           // one tcgen05.commit per active warpgroup
    }
    for (int b = 0; b < R * NSLOT; ++b) mbar_init(&a_empty[b], 1);
    for (int w = 0; w < R; ++w) mbar_init(&acc_full[w], 1);
    fence_mbar_init();
  }
  if (warp == C::kWarpProducer) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == C::kWarpProducer) {
    // ================= producer: sign tiles now, Zq tiles once the Zq kernel is done =================
    if (lane == 0) {
      const uint64_t pol_sign = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      const uint32_t sign_bytes = (uint32_t)Rg * kTileRows * 16;
      const int pre = nunits < STAGES ? nunits : STAGES;
      int i = i_start, q = q_start;
      for (int k = 0; k < pre; ++k) {  // first `pre` stages: sign tiles before the dependency wait
        mbar_arrive_expect_tx(&full[k], sign_bytes + C::kZUnit);
        bulk_g2s(smem + k * C::kStageBytes, p.signs + ((long long)(i >> p.ksh) * p.nq + q) * p.rows_pad + row0, sign_bytes,
                 &full[k], pol_sign);
        if (++q == p.nq) { q = 0; ++i; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");  // Zq of this call is complete and visible
      for (int k = 0; k < pre; ++k) {
        bulk_g2s(smem + k * C::kStageBytes + C::kOffZ, p.zq + (u0 + k) * C::kZUnit, C::kZUnit, &full[k], pol_keep);
      }
      int s = pre % STAGES;
      uint32_t ph = pre == STAGES ? 1u : 0u;
      for (int k = pre; k < nunits; ++k) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * C::kStageBytes;
        mbar_arrive_expect_tx(&full[s], sign_bytes + C::kZUnit);
        bulk_g2s(st, p.signs + ((long long)(i >> p.ksh) * p.nq + q) * p.rows_pad + row0, sign_bytes, &full[s], pol_sign);
        bulk_g2s(st + C::kOffZ, p.zq + (u0 + k) * C::kZUnit, C::kZUnit, &full[s], pol_keep);
        if (++q == p.nq) { q = 0; ++i; }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ================= warpgroup w: expand tile w, issue its MMAs, drain it =================
    const int wg = warp >> 2;
    const int qd = warp & 3;
    const int t = wg;                      // this warpgroup's row tile
    const bool active = t < Rg;
    const bool issuer = qd == 0;           // warp 4w issues the warpgroup's MMAs
    const int row_in_tile = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
    const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
    float yacc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) yacc[b] = 0.f;
    int s = 0, slot = 0, i = i_start, q = q_start;
    uint32_t ph = 0, sph = 0, acc_ph = 0;
    int E = 0;
    bool have_e = false;
    int cnt = 1;
    // Each iteration takes P units (P tiles into one P x 32-column A slot) -- fewer than P
    // when a block ends, so an iteration never straddles two accumulations.
    for (int k = 0; active && k < nunits; k += cnt) {
      const bool first = (k == 0) || (q == 0);
      cnt = 1;
      while (cnt < P && k + cnt < nunits && q + cnt < p.nq) ++cnt;    // same block, in range
      const bool last = (k + cnt == nunits) || (q + cnt == p.nq);
      // Warp 1 of the warpgroup polls the stage / slot mbarriers of an iteration (the named
      // barrier below releases the other three); for iterations after the first it does so
      // at the end of the PREVIOUS iteration, while warp 0 issues the MMAs, so the ~150-cycle
      // mbarrier waits leave the warpgroup's critical path.
      auto waits = [&](int s_, uint32_t ph_, int cnt_, int slot_, uint32_t sph_) {
        for (int u = 0; u < cnt_; ++u) {
          mbar_wait(&full[s_], ph_);
          if (++s_ == STAGES) { s_ = 0; ph_ ^= 1; }
        }
        mbar_wait(&a_empty[wg * NSLOT + slot_], sph_ ^ 1);
      };
      if (qd == 1 && k == 0) waits(s, ph, cnt, slot, sph);
      BS_TRACE(k, 0);
      asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
      BS_TRACE(k, 1);
      tc_fence_after();
      const uint32_t a_col = tbase + (uint32_t)(C::kACols * P * (wg * NSLOT + slot));
      int su = s;
      for (int u = 0; u < cnt; ++u) {
        const uint8_t* st = smem + su * C::kStageBytes;
        // A = +-2^a with a = E - e_u, so that A * (Z 2^e_u) = +-Z 2^E for every unit
        const int e_u = *reinterpret_cast<const int*>(st + C::kOffMeta);
        int a_exp = 0;
        if (e_u != kZqSentinel) {
          if (!have_e) { E = e_u; have_e = true; }
          a_exp = E - e_u;
          if (a_exp < -6 || a_exp > 8) {  // |x/s| range across this CTA's units beyond e4m3 A range
            if (lane == 0 && p.status) atomicOr(p.status, 1);
            a_exp = a_exp < -6 ? -6 : 8;
          }
        }
        const uint32_t e8 = (uint32_t)((7 + a_exp) << 3) * 0x01010101u;
        const uint4 sw = reinterpret_cast<const uint4*>(st)[t * kTileRows + row_in_tile];
        uint32_t o[32];
#ifdef BS_EXP_NO_EXPAND   // timing experiments only (scripts/exp_decode.sh): results are wrong
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = e8 ^ sw.x;
#else
        expand_e4m3(sw.x, e8, o);
        expand_e4m3(sw.y, e8, o + 8);
        expand_e4m3(sw.z, e8, o + 16);
        expand_e4m3(sw.w, e8, o + 24);
#endif
#ifndef BS_EXP_NO_STTM
        tmem_st32(a_col + (uint32_t)(C::kACols * u) + lane_base, o);
#else
        if (o[0] == 0x12345u && o[31] == 0x777u) p.status[1] = 1;   // keep the expansion alive
#endif
        if (++su == STAGES) su = 0;
      }
      BS_TRACE(k, 3);
      tmem_st_wait();
      BS_TRACE(k, 4);
      tc_fence_before();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");   // the warpgroup's 4 lane quadrants are in TMEM
      BS_TRACE(k, 5);
      if (issuer) {
        tc_fence_after();
        if (elect_one()) {
          int sm_ = s;
          for (int u = 0; u < cnt; ++u) {
            const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(smem + sm_ * C::kStageBytes + C::kOffZ), C::LBO, C::SBO);
#ifndef BS_EXP_NO_MMA
#pragma unroll
            for (int m = 0; m < kSubK / 32; ++m) {
              mma_f8_ts(d_acc, a_col + (uint32_t)(C::kACols * u) + 8 * m, bdesc0 + (uint64_t)((m * 2 * C::LBO) >> 4),
                        idesc, (m > 0 || u > 0 || !first) ? 1u : 0u);
              BS_TRACE(k, 12 + m);
            }
#else
            (void)bdesc0;
#endif
            if (++sm_ == STAGES) sm_ = 0;
          }
          mma_commit(&a_empty[wg * NSLOT + slot]);
          sm_ = s;
          for (int u = 0; u < cnt; ++u) {
            mma_commit(&empty[sm_]);
            if (++sm_ == STAGES) sm_ = 0;
          }
          if (last) mma_commit(&acc_full[wg]);
        }
        __syncwarp();
      }
      BS_TRACE(k, 6);
      if (++slot == NSLOT) { slot = 0; sph ^= 1; }
      s += cnt;
      if (s >= STAGES) { s -= STAGES; ph ^= 1; }
      const int ci = i;
      q += cnt;
      if (q == p.nq) { q = 0; ++i; }
      if (qd == 1 && k + cnt < nunits) {   // the next iteration's waits (see above)
        int ncnt = 1;
        while (ncnt < P && k + cnt + ncnt < nunits && q + ncnt < p.nq) ++ncnt;
        waits(s, ph, ncnt, slot, sph);
      }

      if (last) {
        // ---- epilogue for block ci: y += 2^-E sum_r U'_ci[row, r] (T_d0 + T_d1 + T_d2)[row, r]
        float uu[16];
        {
          const long long row = row0 + t * kTileRows + row_in_tile;
          const long long base = ((long long)ci * p.rows_pad + row) * 16;
          if (p.f_dtype == 1) {
            const uint4* up = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.u) + base);
            const uint4 r0v = __ldg(up), r1v = __ldg(up + 1);
            const __nv_bfloat162* b0 = reinterpret_cast<const __nv_bfloat162*>(&r0v);
            const __nv_bfloat162* b1 = reinterpret_cast<const __nv_bfloat162*>(&r1v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f0 = __bfloat1622float2(b0[e]);
              const float2 f1 = __bfloat1622float2(b1[e]);
              uu[2 * e] = f0.x; uu[2 * e + 1] = f0.y;
              uu[8 + 2 * e] = f1.x; uu[8 + 2 * e + 1] = f1.y;
            }
          } else {
            const float4* up = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.u) + base);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float4 f = __ldg(up + e);
              uu[4 * e] = f.x; uu[4 * e + 1] = f.y; uu[4 * e + 2] = f.z; uu[4 * e + 3] = f.w;
            }
          }
        }
        mbar_wait(&acc_full[wg], acc_ph);
        acc_ph ^= 1;
        tc_fence_after();
        const float esc = exp2f((float)-E);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          float tsum[16];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            uint32_t v[16];
            tmem_ld16(d_acc + lane_base + (uint32_t)((b * 3 + d) * 16), v);
            tmem_ld_wait();
#pragma unroll
            for (int r = 0; r < 16; ++r) tsum[r] = (d == 0) ? __uint_as_float(v[r]) : tsum[r] + __uint_as_float(v[r]);
          }
          float acc = 0.f;
#pragma unroll
          for (int r = 0; r < 16; ++r) acc = fmaf(uu[r], tsum[r], acc);
          yacc[b] = fmaf(acc, esc, yacc[b]);
        }
        // the next piece's first MMA (issued after this warpgroup's next bar.sync)
        // overwrites the accumulator: order these tcgen05.ld before that barrier
        tc_fence_before();
      }
    }
#undef BS_TRACE
    if (active) {   // this CTA's partial y -> its split-K slot (zeros if it had no units)
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < p.batch) store_partial(p, (int)blockIdx.x, R * kTileRows, t * kTileRows + row_in_tile, b, yacc[b]);
    }
  }

#ifdef BS_DECODE_TRACE
  if (p.dbg_acc && threadIdx.x == 32 * 12) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * blockIdx.x + 1] = (long long)gt;
  }
#endif
  // ---- teardown + last-CTA-of-group finalisation
  __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kWarpProducer) tmem_dealloc<C::kTmemCols>(tbase);
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

}  // namespace bs
