// EXPERIMENT (not built into the library): MMA warp fed by named barriers; measured 28.7 us vs
// (Written against the round-1 atomicAdd y workspace `p.y_acc`; the library now uses per-CTA
// split-K slots -- replace its fold/finalise with store_partial / finalize_group to rebuild.)
// 28.3 us for decode_f8_kernel on C2 n=16 B=1.
// e4m3 decode kernel with a dedicated MMA warp fed through NAMED barriers.
//
// Same computation and operands as decode_f8_kernel (decode_f8.cuh).  Measured on B200: an
// mbarrier hand-off costs the waiting warp ~150 cycles, a named-barrier hand-off ~40, an
// elected MMA block ~120 plus ~25-40 cycles per MMA.  Here each unit's 4 row tiles are
// expanded by 4 warpgroups (warp 1 of each polls the stage / slot mbarriers one iteration
// ahead and releases its warpgroup with a named barrier) and handed to the MMA warp with a
// double-buffered named barrier per tile (bar.arrive by the 128 expander threads, bar.sync
// by the MMA warp): the MMA warp issues all 16 MMAs of a unit in ONE elected block, so the
// warpgroups never wait for MMA issue and MMA issue never waits on an mbarrier.
// Double-buffering the tile barriers by unit parity is race-free because a warpgroup can
// only reach unit k+2 after its A slot (NSLOT = 2) was released by the MMAs of unit k,
// which the MMA warp issued after its bar.sync of unit k.
#pragma once
#include "../../paper_2410_23918_b200/csrc/decode_f8.cuh"

namespace bs {

template <int NB, int R_>
struct DecodeF8NCfg {
  static constexpr int N = ZqCfg<NB>::N;
  static constexpr int R = R_;                               // row tiles = warpgroups
  static constexpr int kThreads = 32 * (4 * R + 2);          // + producer + MMA warp
  static constexpr int kWarpProducer = 4 * R, kWarpMma = 4 * R + 1;
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
  static constexpr int NSLOT = 2;                            // A slots per row tile
  static constexpr uint32_t kAccCol = R * NSLOT * kACols;
  static constexpr uint32_t LBO = (N / 8) * 128;
  static constexpr uint32_t SBO = 128;
  static_assert(N <= 256 && N % 16 == 0, "invalid MMA N");
  static_assert(kAccCol + R * N <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes <= 227 * 1024, "smem overflow");
  static_assert(3 * R <= 15, "named barriers 1..3R");
};

template <int NB, int R_>
__global__ void __launch_bounds__(DecodeF8NCfg<NB, R_>::kThreads, 1) decode_f8n_kernel(const DecodeParams p) {
  using C = DecodeF8NCfg<NB, R_>;
  constexpr int N = C::N, R = C::R, STAGES = C::STAGES, NSLOT = C::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_empty = empty + STAGES;     // [NSLOT] one commit per unit (all R tiles)
  uint64_t* acc_full = a_empty + NSLOT;   // [R]
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
  // named barriers: tile-ready (t, parity) = 1 + 2t + parity, warpgroup "go" = 1 + 2R + t

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);            // the MMA warp's commit after the unit's MMAs
    }
    for (int b = 0; b < NSLOT; ++b) mbar_init(&a_empty[b], 1);
    for (int w = 0; w < R; ++w) mbar_init(&acc_full[w], 1);
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
      for (int k = 0; k < pre; ++k) {  // first `pre` stages: sign tiles before the dependency wait
        mbar_arrive_expect_tx(&full[k], sign_bytes + C::kZUnit);
        bulk_g2s(smem + k * C::kStageBytes, p.signs + ((long long)i * p.nq + q) * p.rows_pad + row0, sign_bytes,
                 &full[k], pol_sign);
        if (++q == p.nq) { q = 0; ++i; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");  // Zq of this call is complete and visible
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
    // ================= MMA warp: one elected block of 4 x Rg MMAs per unit =================
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
    const uint64_t bdesc_s0 = smem_desc_kmajor(smem_u32(smem + C::kOffZ), C::LBO, C::SBO);
    int s = 0, slot = 0, q = q_start;
    for (int k = 0; k < nunits; ++k) {
      const bool first = (k == 0) || (q == 0);
      const bool last = (k == nunits - 1) || (q == p.nq - 1);
      for (int t = 0; t < Rg; ++t)       // every warpgroup's quarter tiles are in TMEM
        asm volatile("bar.sync %0, 160;" ::"r"(1 + 2 * t + (k & 1)) : "memory");
      tc_fence_after();
      if (elect_one()) {
        const uint64_t bdesc0 = bdesc_s0 + (uint64_t)((s * C::kStageBytes) >> 4);
#pragma unroll
        for (int t = 0; t < R; ++t) {
          if (t < Rg) {
            const uint32_t a_col = tbase + (uint32_t)(C::kACols * (t * NSLOT + slot));
            const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
#pragma unroll
            for (int m = 0; m < kSubK / 32; ++m)
              mma_f8_ts(d_acc, a_col + 8 * m, bdesc0 + (uint64_t)((m * 2 * C::LBO) >> 4), idesc,
                        (m > 0 || !first) ? 1u : 0u);
            if (last) mma_commit(&acc_full[t]);
          }
        }
        mma_commit(&a_empty[slot]);
        mma_commit(&empty[s]);
      }
      __syncwarp();
      if (++slot == NSLOT) slot = 0;
      if (++s == STAGES) s = 0;
      if (++q == p.nq) q = 0;
    }
  } else {
    // ================= warpgroup w: expand tile w, drain it =================
    const int wg = warp >> 2;
    const int qd = warp & 3;
    const int t = wg;                      // this warpgroup's row tile
    const bool active = t < Rg;
    const int row_in_tile = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
    const int bar_go = 1 + 2 * R + wg;
    float yacc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) yacc[b] = 0.f;
    int s = 0, slot = 0, i = i_start, q = q_start;
    uint32_t ph = 0, sph = 0, acc_ph = 0;
    int E = 0;
    bool have_e = false;
    // warp 1 polls the stage / slot mbarriers, one unit ahead after the first
    auto waits = [&](int s_, uint32_t ph_, int slot_, uint32_t sph_) {
      mbar_wait(&full[s_], ph_);
      mbar_wait(&a_empty[slot_], sph_ ^ 1);
    };
    for (int k = 0; active && k < nunits; ++k) {
      const bool last = (k == nunits - 1) || (q == p.nq - 1);
      if (qd == 1 && k == 0) waits(s, ph, slot, sph);
      asm volatile("bar.sync %0, 128;" ::"r"(bar_go) : "memory");
      tc_fence_after();
      const uint8_t* st = smem + s * C::kStageBytes;
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
      {
        uint32_t o[32];
        expand_e4m3(sw.x, e8, o);
        expand_e4m3(sw.y, e8, o + 8);
        expand_e4m3(sw.z, e8, o + 16);
        expand_e4m3(sw.w, e8, o + 24);
        tmem_st32(tbase + (uint32_t)(C::kACols * (t * NSLOT + slot)) + lane_base, o);
      }
      tmem_st_wait();
      tc_fence_before();
      asm volatile("bar.arrive %0, 160;" ::"r"(1 + 2 * t + (k & 1)) : "memory");   // tile quarter in TMEM
      if (++slot == NSLOT) { slot = 0; sph ^= 1; }
      if (++s == STAGES) { s = 0; ph ^= 1; }
      const int ci = i;
      if (++q == p.nq) { q = 0; ++i; }
      if (qd == 1 && k + 1 < nunits) waits(s, ph, slot, sph);

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
        // the next block's first MMA (issued after this warpgroup's next tile-ready
        // barrier) overwrites the accumulator: order these tcgen05.ld before it
        tc_fence_before();
      }
    }
    if (active && nunits > 0) {
      const int row = row0 + t * kTileRows + row_in_tile;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < p.batch) atomicAdd(p.y_acc + (long long)b * p.rows_pad + row, yacc[b]);
    }
  }

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
