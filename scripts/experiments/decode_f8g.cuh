// EXPERIMENT (not built into the library): group-pipelined decode kernel, measured 33 us vs
// (Written against the round-1 atomicAdd y workspace `p.y_acc`; the library now uses per-CTA
// split-K slots -- replace its fold/finalise with store_partial / finalize_group to rebuild.)
// 29.8 us for decode_f8_kernel on C2 n=16 B=1. Kept for the record; to try it,
// include it from bitstack.cu and launch decode_f8g_kernel<NB, 2> with R = 2 row tiles per CTA.
// Group-pipelined variant of the e4m3 decode kernel.
//
// Same computation and operands as decode_f8_kernel (decode_f8.cuh): y = sum_i sum_r
// U'_i[:,r] * (S_i (V'_i[:,r] * x/s)) with S_i expanded to e4m3 +-2^a in TMEM and Z as three
// e4m3 digits (zq_kernel).  What differs is how the work is handed between warps, shaped by
// the B200 costs measured in scripts/ring_bench.cu and scripts/pingpong.cu:
//   * 16 warps expand + tcgen05.st a 128x128 tile every ~76 cycles per SM;
//   * one warp issues back-to-back MMAs (M128 N48 K32) every ~25 cycles alone, ~36 with the
//     expanders' tcgen05.st traffic -- but only inside ONE elected block: every elect /
//     reconvergence costs ~120 cycles;
//   * every mbarrier operation costs the issuing warp ~100-150 cycles.
// So hand-offs are per GROUP of 4 tiles (P units x R row tiles, R * P = 4): each of the 16
// expander warps (team tau = w / 4 -> row tile tau % R, unit tau / R of the group; lane
// quadrant w % 4) writes one 32-row quarter per group and arrives once; the MMA warp waits
// once per group and issues all 16 MMAs and the group's commits in one elected block.
// NG slot groups ring through TMEM; with ACCB = 2 the accumulators are double-buffered by
// block parity, so a block's drain overlaps the next block's MMAs.
#pragma once
#include "../../paper_2410_23918_b200/csrc/decode_f8.cuh"

namespace bs {

template <int NB, int R_>
struct DecodeF8GCfg {
  static constexpr int N = ZqCfg<NB>::N;
  static constexpr int R = R_;                               // row tiles per CTA
  static constexpr int P = 4 / R;                            // units per group
  static constexpr int kThreads = 32 * 18;
  static constexpr int kWarpProducer = 16, kWarpMma = 17;
  static constexpr int kZBytes = ZqCfg<NB>::kZBytes;
  static constexpr int kZUnit = ZqCfg<NB>::kZUnit;
  static constexpr int kSignBytes = R * kTileRows * 16;
  static constexpr int kOffZ = kSignBytes;
  static constexpr int kOffMeta = kOffZ + kZBytes;
  static constexpr int kStageBytes = (kOffZ + kZUnit + 127) / 128 * 128;
  static constexpr int S0 = (200 * 1024) / kStageBytes;
  static constexpr int STAGES = S0 > 16 ? 16 : (S0 < 2 * P ? 2 * P : S0);
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarBytes;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kACols = 32;                          // 128 rows x 128 e4m3 per tile
  static constexpr int kGroupCols = 4 * kACols;              // R * P = 4 tiles per group
  static constexpr int ACCB = (2 * R * N + 2 * kGroupCols <= 512) ? 2 : 1;
  static constexpr int NG0 = (512 - ACCB * R * N) / kGroupCols;
  static constexpr int NG = NG0 > 3 ? 3 : NG0;               // A slot groups in TMEM
  static constexpr uint32_t kAccCol = NG * kGroupCols;
  static constexpr uint32_t LBO = (N / 8) * 128;
  static constexpr uint32_t SBO = 128;
  static_assert(R == 1 || R == 2 || R == 4, "R * P = 4 teams");
  static_assert(N <= 256 && N % 16 == 0, "invalid MMA N");
  static_assert(NG >= 1, "TMEM");
  static_assert(kAccCol + ACCB * R * N <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes <= 227 * 1024, "smem overflow");
};

template <int NB, int R_>
__global__ void __launch_bounds__(DecodeF8GCfg<NB, R_>::kThreads, 1) decode_f8g_kernel(const DecodeParams p) {
  using C = DecodeF8GCfg<NB, R_>;
  constexpr int N = C::N, R = C::R, P = C::P, STAGES = C::STAGES, NG = C::NG, ACCB = C::ACCB;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_full = empty + STAGES;          // [NG] 16 expander-warp arrivals per group
  uint64_t* a_empty = a_full + NG;            // [NG] tcgen05.commit after the group's MMAs
  uint64_t* acc_full = a_empty + NG;          // [R][ACCB]
  uint64_t* acc_empty = acc_full + R * ACCB;  // [R][ACCB] 4 draining warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + R * ACCB);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x / p.ctas_per_group;
  const int jc = blockIdx.x % p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const long long u0 = L * jc / p.ctas_per_group;
  const long long u1 = L * (jc + 1) / p.ctas_per_group;
  const int nunits = (int)(u1 - u0);
  const int ngroups = (nunits + P - 1) / P;
  const int i_start = (int)(u0 / p.nq), q_start = (int)(u0 % p.nq);
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int row0 = g * R * kTileRows;
#ifdef BS_DECODE_TRACE
  long long* trace = (p.dbg_acc && blockIdx.x == 0) ? reinterpret_cast<long long*>(p.dbg_acc) : nullptr;
  const long long tstart = clock64();
#define BS_GTRACE(j_, k_) do { if (trace && lane == 0) trace[(j_) * 16 + (k_)] = clock64() - tstart; } while (0)
#else
#define BS_GTRACE(j_, k_) do { } while (0)
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NG; ++b) {
      mbar_init(&a_full[b], 16);
      mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < R * ACCB; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == C::kWarpMma) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == C::kWarpProducer) {
    if (lane == 0) {
      const uint64_t pol_sign = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      const uint32_t sign_bytes = (uint32_t)Rg * kTileRows * 16;
      const int pre = nunits < STAGES ? nunits : STAGES;
      int i = i_start, q = q_start;
      for (int k = 0; k < pre; ++k) {   // sign tiles before the dependency wait (PDL overlap)
        mbar_arrive_expect_tx(&full[k], sign_bytes + C::kZUnit);
        bulk_g2s(smem + k * C::kStageBytes, p.signs + ((long long)i * p.nq + q) * p.rows_pad + row0, sign_bytes,
                 &full[k], pol_sign);
        if (++q == p.nq) { q = 0; ++i; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int k = 0; k < pre; ++k)
        bulk_g2s(smem + k * C::kStageBytes + C::kOffZ, p.zq + (u0 + k) * C::kZUnit, C::kZUnit, &full[k], pol_keep);
      int s = pre % STAGES;
      uint32_t ph = pre == STAGES ? 1u : 0u;
      for (int k = pre; k < nunits; ++k) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * C::kStageBytes;
        mbar_arrive_expect_tx(&full[s], sign_bytes + C::kZUnit);
        bulk_g2s(st, p.signs + ((long long)i * p.nq + q) * p.rows_pad + row0, sign_bytes, &full[s], pol_sign);
        bulk_g2s(st + C::kOffZ, p.zq + (u0 + k) * C::kZUnit, C::kZUnit, &full[s], pol_keep);
        if (++q == p.nq) { q = 0; ++i; }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == C::kWarpMma) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
    // descriptor of stage 0's Zq tile; stage s adds s * kStageBytes to the start address (>> 4)
    const uint64_t bdesc_s0 = smem_desc_kmajor(smem_u32(smem + C::kOffZ), C::LBO, C::SBO);
    int gslot = 0, s = 0, q = q_start, i = i_start;
    uint32_t gph = 0;
    for (int j = 0; j < ngroups; ++j) {
      BS_GTRACE(j, 0);
      mbar_wait(&a_full[gslot], gph);   // the expanders waited full[] for these units first
      BS_GTRACE(j, 1);
      const int kn = (j + 1) * P <= nunits ? P : nunits - j * P;
      // a block starting inside this group needs its accumulator buffer drained
      {
        int qq = q, ii = i;
        for (int u = 0; u < kn; ++u) {
          const int rel = ii - i_start;
          if ((j * P + u == 0 || qq == 0) && rel >= ACCB) {
            const int ab = ACCB == 2 ? (rel & 1) : 0;
            for (int t = 0; t < Rg; ++t)
              mbar_wait(&acc_empty[t * ACCB + ab], (uint32_t)(((rel - ACCB) / ACCB) & 1));
          }
          if (++qq == p.nq) { qq = 0; ++ii; }
        }
      }
      tc_fence_after();
      if (elect_one()) {   // ONE elected block per group: its MMAs and commits
        int ss = s, qq = q, ii = i;
        const uint32_t a_grp = tbase + (uint32_t)(gslot * C::kGroupCols);
#pragma unroll
        for (int u = 0; u < P; ++u) {
          if (u < kn) {
            const bool first = (j * P + u == 0) || (qq == 0);
            const bool last = (j * P + u == nunits - 1) || (qq == p.nq - 1);
            const int ab = ACCB == 2 ? ((ii - i_start) & 1) : 0;
            const uint64_t bdesc0 = bdesc_s0 + (uint64_t)((ss * C::kStageBytes) >> 4);
            const uint32_t d_base = tbase + C::kAccCol + (uint32_t)(ab * R * N);
#pragma unroll
            for (int t = 0; t < R; ++t) {
              if (t < Rg) {
                const uint32_t a_col = a_grp + (uint32_t)((u * R + t) * C::kACols);
#pragma unroll
                for (int m = 0; m < kSubK / 32; ++m)
                  mma_f8_ts(d_base + (uint32_t)(t * N), a_col + 8 * m, bdesc0 + (uint64_t)((m * 2 * C::LBO) >> 4),
                            idesc, (m > 0 || !first) ? 1u : 0u);
                if (last) mma_commit(&acc_full[t * ACCB + ab]);
              }
            }
            mma_commit(&empty[ss]);
            if (++ss == STAGES) ss = 0;
            if (++qq == p.nq) { qq = 0; ++ii; }
          }
        }
        mma_commit(&a_empty[gslot]);
      }
      __syncwarp();
      BS_GTRACE(j, 2);
      s += kn;
      if (s >= STAGES) s -= STAGES;
      q += kn;
      while (q >= p.nq) { q -= p.nq; ++i; }
      if (++gslot == NG) { gslot = 0; gph ^= 1; }
    }
  } else {
    // ================= expander warp: team tau -> (row tile t, unit uo of each group) =================
    const int tau = warp >> 2, qd = warp & 3;
    const int t = tau % R;
    const int uo = tau / R;
    const int row_in_tile = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    float yacc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) yacc[b] = 0.f;
    bool drained = false;
    int E = 0, e_block = -1;
    // Zq metadata (e_u) is also read from global memory (E_i below): the Zq kernel's
    // writes are visible after griddepcontrol.wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int gslot = 0;
    uint32_t gph = 0;
    long long u = u0 + uo;
    int i = (int)(u / p.nq), q = (int)(u % p.nq);
    for (int j = 0; j < ngroups; ++j) {
      const int k = j * P + uo;
      const bool mine = k < nunits && t < Rg;
      if (warp == 0) BS_GTRACE(j, 4);
      mbar_wait(&a_empty[gslot], gph ^ 1);       // the group's A slots are free
      if (warp == 0) BS_GTRACE(j, 5);
      bool last = false;
      if (mine) {
        last = (k == nunits - 1) || (q == p.nq - 1);
        if (i != e_block) {
          // E_i: e_u of the first non-empty unit of block i in this CTA's range -- the same
          // value in every team, so every unit accumulated for block i shares the scale 2^E_i
          e_block = i;
          E = 0;
          const long long ub = (long long)i * p.nq > u0 ? (long long)i * p.nq : u0;
          const long long ue = (long long)(i + 1) * p.nq < u1 ? (long long)(i + 1) * p.nq : u1;
          for (long long uu = ub; uu < ue; ++uu) {
            const int e = __ldcg(reinterpret_cast<const int*>(p.zq + uu * C::kZUnit + C::kZBytes));
            if (e != kZqSentinel) { E = e; break; }
          }
        }
        const int s = k % STAGES;
        mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
        if (warp == 0) BS_GTRACE(j, 6);
        const uint8_t* st = smem + s * C::kStageBytes;
        const int e_u = *reinterpret_cast<const int*>(st + C::kOffMeta);
        int a_exp = 0;
        if (e_u != kZqSentinel) {
          a_exp = E - e_u;
          if (a_exp < -6 || a_exp > 8) {  // |x/s| range across the block's units beyond e4m3 A range
            if (lane == 0 && p.status) atomicOr(p.status, 1);
            a_exp = a_exp < -6 ? -6 : 8;
          }
        }
        const uint32_t e8 = (uint32_t)((7 + a_exp) << 3) * 0x01010101u;
        const uint4 sw = reinterpret_cast<const uint4*>(st)[t * kTileRows + row_in_tile];
        tc_fence_after();
        uint32_t o[32];
        expand_e4m3(sw.x, e8, o);
        expand_e4m3(sw.y, e8, o + 8);
        expand_e4m3(sw.z, e8, o + 16);
        expand_e4m3(sw.w, e8, o + 24);
        tmem_st32(tbase + (uint32_t)(gslot * C::kGroupCols + (uo * R + t) * C::kACols) + lane_base, o);
        tmem_st_wait();
        tc_fence_before();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[gslot]);
      if (warp == 0) BS_GTRACE(j, 7);
      if (++gslot == NG) { gslot = 0; gph ^= 1; }

      if (mine && last) {
        // ---- drain block i: y += 2^-E_i sum_r U'_i[row, r] (T_d0 + T_d1 + T_d2)[row, r]
        const int rel = i - i_start;
        const int ab = ACCB == 2 ? (rel & 1) : 0;
        const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)((ab * R + t) * N);
        float uu[16];
        {
          const long long row = row0 + t * kTileRows + row_in_tile;
          const long long base = ((long long)i * p.rows_pad + row) * 16;
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
        mbar_wait(&acc_full[t * ACCB + ab], (uint32_t)((rel / ACCB) & 1));
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
        drained = true;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[t * ACCB + ab]);
      }
      // next unit of this team: P units later
      q += P;
      while (q >= p.nq) { q -= p.nq; ++i; }
    }
    if (drained) {
      const int row = row0 + t * kTileRows + row_in_tile;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < p.batch) atomicAdd(p.y_acc + (long long)b * p.rows_pad + row, yacc[b]);
    }
  }
#undef BS_GTRACE

  // ---- teardown + last-CTA-of-group finalisation
  __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == C::kWarpMma) tmem_dealloc<C::kTmemCols>(tbase);
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(p.counters + g, 1);
    *last_flag = (prev == p.ctas_per_group - 1);
  }
  __syncthreads();
  if (*last_flag) {
    __threadfence();
    const int rows_in_group = Rg * kTileRows;
    const int total = rows_in_group * p.batch;
    for (int e = threadIdx.x; e < total; e += C::kThreads) {
      const int b = e / rows_in_group;
      const int row = row0 + e % rows_in_group;
      float* src = p.y_acc + (long long)b * p.rows_pad + row;
      const float val = __ldcg(src);
      *src = 0.f;
      if (row < p.rows_local) {
        const long long o = (long long)b * p.y_stride + row;
        if (p.y_dtype == 0) reinterpret_cast<float*>(p.y)[o] = val;
        else reinterpret_cast<__nv_bfloat16*>(p.y)[o] = __float2bfloat16_rn(val);
      }
    }
    if (threadIdx.x == 0) p.counters[g] = 0;
  }
}

}  // namespace bs
