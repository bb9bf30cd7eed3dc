// e4m3 decode kernel with one MMA-issuing warp PER WARPGROUP.
//
// Same computation and operands as decode_f8_kernel (decode_f8.cuh).  Each of the R
// warpgroups owns a row tile and has 4 expander warps (TMEM lane quadrants) plus its own
// issuer warp.  Work moves in GROUPS of up to P consecutive units of one block (a unit = one
// 128-column subchunk): the producer fills one ring stage per group, the expanders expand the
// group's P sign tiles into one A slot (P x 32 TMEM columns) and hand it to their issuer
// through a named barrier (bar.arrive by the 128 expander threads, bar.sync by the issuer),
// so they never wait for MMA issue; the issuer polls the stage / slot mbarriers one group
// ahead and releases the expanders for the next group on a named "go" barrier before issuing
// the group's 4P MMAs.  P > 1 amortises the per-hand-off synchronisation and control code
// over P units.  Measured motivation (scripts/exp_decode.sh): the per-unit chain of
// hand-offs, not data movement or math, bounds the kernel.
#pragma once
#include "decode_f8.cuh"

namespace bs {

#ifndef BS_F8_STAGES
#define BS_F8_STAGES 6      // ring depth cap (scripts/exp_stages.sh: 6 beats 4, 8, 10, 12, 14, 15)
#endif
#ifndef BS_F8_PRE
#define BS_F8_PRE 2         // ring stages whose sign tiles are requested before griddepcontrol.wait
#endif
#ifndef BS_F8_SMEM_KB
#define BS_F8_SMEM_KB 200   // shared memory the ring may use per SM
#endif

template <int NB, int R_, int P_ = 1, int OCC_ = 1>
struct DecodeF8ICfg {
  static constexpr int OCC = OCC_;                           // resident CTAs per SM (TMEM / smem split)
  static constexpr int N = ZqCfg<NB>::N;
  static constexpr int R = R_;                               // row tiles = warpgroups
  static constexpr int P = P_;                               // units per group (hand-off)
  static constexpr int kThreads = 32 * (5 * R + 1);          // R x (4 expanders + issuer) + producer
  static constexpr int kWarpProducer = 5 * R;
  static constexpr int kZBytes = ZqCfg<NB>::kZBytes;
  static constexpr int kZUnit = ZqCfg<NB>::kZUnit;
  static constexpr int kUnitSign = R * kTileRows * 16;       // sign bytes of one unit (R row tiles)
  static constexpr int kOffZ = P * kUnitSign;                // Zq of unit u at kOffZ + u kZUnit
  static constexpr int kStageBytes = (kOffZ + P * kZUnit + 127) / 128 * 128;
  static constexpr int S0 = (BS_F8_SMEM_KB * 1024 / OCC_) / kStageBytes;
  static constexpr int STAGES = S0 > BS_F8_STAGES ? BS_F8_STAGES : (S0 < 2 ? 2 : S0);
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarBytes;
  static constexpr uint32_t kTmemCols = 512 / OCC_;
  static constexpr int kACols = 32;                          // 128 rows x 128 e4m3 per unit
  static constexpr int NSLOT = 2;                            // A slots per row tile
  static constexpr uint32_t kAccCol = R * NSLOT * P * kACols;
  static constexpr uint32_t LBO = (N / 8) * 128;
  static constexpr uint32_t SBO = 128;
  static_assert(N <= 256 && N % 16 == 0, "invalid MMA N");
  static_assert(kAccCol + R * N <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes * OCC_ <= 227 * 1024, "smem overflow");
  static_assert(2 * R <= 15, "named barriers 1..2R");
  static_assert(5 * R + 1 <= 32, "warps");
  static_assert(kZUnit % 16 == 0, "Zq unit alignment (smem descriptor)");
};

// Units [k, k + cnt) of a CTA's range form one group: at most P, never across a block end.
template <int P>
__device__ __forceinline__ int group_count(int k, int q, int nunits, int nq) {
  if constexpr (P == 1) return 1;
  int c = nq - q;
  c = c < P ? c : P;
  return c < nunits - k ? c : nunits - k;
}

// The kernel body, for CTA `cta` of the launch that computes the layer described by p
// (decode_f8i_kernel: one layer, cta = cta; decode_f8i_grouped_kernel: several).
template <int NB, int R_, int P_, int OCC_>
__device__ __forceinline__ void decode_f8i_body(const DecodeParams& p, const int cta) {
  using C = DecodeF8ICfg<NB, R_, P_, OCC_>;
  constexpr int N = C::N, R = C::R, P = C::P, STAGES = C::STAGES, NSLOT = C::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_empty = empty + STAGES;     // [R][NSLOT] per warpgroup
  uint64_t* acc_full = a_empty + R * NSLOT; // [R]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + R);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = cta / p.ctas_per_group;
  const int jc = cta % p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const long long u0 = L * jc / p.ctas_per_group;
  const long long u1 = L * (jc + 1) / p.ctas_per_group;
  const int nunits = (int)(u1 - u0);
  const int i_start = (int)(u0 / p.nq), q_start = (int)(u0 % p.nq);
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int row0 = g * R * kTileRows;
  // named barriers of warpgroup w: go = 1 + 2w (issuer arrives, expanders sync), tile-ready =
  // 2 + 2w (expanders arrive, issuer syncs).  Single-buffered is race-free: the issuer
  // releases group k+1 only after syncing on group k's tile, and the expanders arrive on
  // group k+1's tile only after that release.
#ifdef BS_DECODE_TRACE
  long long* trace = (p.dbg_acc && cta == 0) ? reinterpret_cast<long long*>(p.dbg_acc) : nullptr;
  const long long tstart = clock64();
#define BS_ITRACE(k_, c_) do { if (trace && lane == 0) trace[(k_) * 16 + (c_)] = clock64() - tstart; } while (0)
  if (p.dbg_acc && threadIdx.x == 0) {   // every CTA's entry %globaltimer (ns), unit count
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta] = (long long)gt;
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta + 2] = nunits;
  }
#else
#define BS_ITRACE(k_, c_) do { } while (0)
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Rg);           // one commit per active warpgroup's issuer
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
    if (lane == 0) {
      const uint64_t pol_sign = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      const uint32_t sign_bytes = (uint32_t)Rg * kTileRows * 16;
      // first STAGES groups: sign tiles before the dependency wait, then their Zq
      int k = 0, q = q_start, gi = 0, iv = i_start;
      long long ui = (long long)(iv >> p.ksh) * p.nq;   // (sign block of block iv) * nq
      for (; gi < (BS_F8_PRE < STAGES ? BS_F8_PRE : STAGES) && k < nunits; ++gi) {
        const int cnt = group_count<P>(k, q, nunits, p.nq);
#ifndef BS_EXP_NOSIGN   // timing experiment: no sign-tile copies (wrong results)
        mbar_arrive_expect_tx(&full[gi], (uint32_t)cnt * (sign_bytes + C::kZUnit));
        for (int u = 0; u < cnt; ++u)
          bulk_g2s(smem + gi * C::kStageBytes + u * C::kUnitSign, p.signs + (ui + q + u) * p.rows_pad + row0,
                   sign_bytes, &full[gi], pol_sign);
#else
        mbar_arrive_expect_tx(&full[gi], (uint32_t)cnt * C::kZUnit);
#endif
        k += cnt;
        q += cnt;
        if (q == p.nq) { q = 0; ++iv; ui = (long long)(iv >> p.ksh) * p.nq; }
      }
      const int pre = gi;
      asm volatile("griddepcontrol.wait;" ::: "memory");  // Zq of this call is complete and visible
      {
        int kk = 0, qq = q_start;
        for (int g2 = 0; g2 < pre; ++g2) {
          const int cnt = group_count<P>(kk, qq, nunits, p.nq);
          bulk_g2s(smem + g2 * C::kStageBytes + C::kOffZ, p.zq + (u0 + kk) * C::kZUnit,
                   (uint32_t)cnt * C::kZUnit, &full[g2], pol_keep);
          kk += cnt;
          qq += cnt;
          if (qq == p.nq) qq = 0;
        }
      }
      int s = pre % STAGES;
      uint32_t ph = pre == STAGES ? 1u : 0u;
      while (k < nunits) {
        const int cnt = group_count<P>(k, q, nunits, p.nq);
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * C::kStageBytes;
#ifndef BS_EXP_NOSIGN
        mbar_arrive_expect_tx(&full[s], (uint32_t)cnt * (sign_bytes + C::kZUnit));
        for (int u = 0; u < cnt; ++u)
          bulk_g2s(st + u * C::kUnitSign, p.signs + (ui + q + u) * p.rows_pad + row0, sign_bytes, &full[s], pol_sign);
#else
        mbar_arrive_expect_tx(&full[s], (uint32_t)cnt * C::kZUnit);
#endif
        bulk_g2s(st + C::kOffZ, p.zq + (u0 + k) * C::kZUnit, (uint32_t)cnt * C::kZUnit, &full[s], pol_keep);
        k += cnt;
        q += cnt;
        if (q == p.nq) { q = 0; ++iv; ui = (long long)(iv >> p.ksh) * p.nq; }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp % 5 == 4) {
    // ================= issuer of warpgroup t =================
    // Polls the stage / slot mbarriers of group k+1 while the expanders work on group k, and
    // releases them for group k+1 (bar.arrive "go") as soon as group k's tile is in TMEM --
    // before issuing group k's MMAs, so expansion of k+1 overlaps MMA issue of k.
    const int t = warp / 5;
    if (t < Rg) {
      constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
      const uint64_t bdesc_s0 = smem_desc_kmajor(smem_u32(smem + C::kOffZ), C::LBO, C::SBO);
      const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
      const int bar_go = 1 + 2 * t, bar_tile = 2 + 2 * t;
      int s = 0, slot = 0, q = q_start, k = 0, gk = 0;
      int sn = 0, slotn = 0;                 // stage / slot of group gk+1
      uint32_t phn = 0, sphn = 0;
      mbar_wait(&full[0], 0);
      mbar_wait(&a_empty[t * NSLOT], 1);
      asm volatile("bar.arrive %0, 160;" ::"r"(bar_go) : "memory");
      while (k < nunits) {
        const int cnt = group_count<P>(k, q, nunits, p.nq);
        const bool first = (k == 0) || (q == 0);
        const bool last = (k + cnt == nunits) || (q + cnt == p.nq);
        if (++sn == STAGES) { sn = 0; phn ^= 1; }
        if (++slotn == NSLOT) { slotn = 0; sphn ^= 1; }
        if (k + cnt < nunits) {
          mbar_wait(&full[sn], phn);
          mbar_wait(&a_empty[t * NSLOT + slotn], sphn ^ 1);
        }
        if (t == 1) BS_ITRACE(gk, 8);
        asm volatile("bar.sync %0, 160;" ::"r"(bar_tile) : "memory");   // group k's tile in TMEM
        if (k + cnt < nunits) asm volatile("bar.arrive %0, 160;" ::"r"(bar_go) : "memory");
        if (t == 1) BS_ITRACE(gk, 9);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bdesc0 = bdesc_s0 + (uint64_t)((s * C::kStageBytes) >> 4);
          const uint32_t a_col = tbase + (uint32_t)(C::kACols * P * (t * NSLOT + slot));
#pragma unroll
          for (int u = 0; u < P; ++u) {
            if (u < cnt) {
#pragma unroll
              for (int m = 0; m < kSubK / 32; ++m) {
#ifndef BS_EXP_SKEL   // timing experiment (scripts/exp_skeleton.sh): no MMAs
                mma_f8_ts(d_acc, a_col + (uint32_t)(C::kACols * u + 8 * m),
                          bdesc0 + (uint64_t)((u * C::kZUnit + m * 2 * C::LBO) >> 4), idesc,
                          (m > 0 || u > 0 || !first) ? 1u : 0u);
#endif
              }
            }
          }
          mma_commit(&a_empty[t * NSLOT + slot]);
          mma_commit(&empty[s]);
          if (last) mma_commit(&acc_full[t]);
        }
        __syncwarp();
        if (t == 1) BS_ITRACE(gk, 10);
        s = sn;
        slot = slotn;
        k += cnt;
        q += cnt;
        if (q == p.nq) q = 0;
        ++gk;
      }
    }
  } else {
    // ================= expander warps of warpgroup wg (TMEM lane quadrant = warp % 4) =================
    const int wg = warp / 5;
    const int qd = warp & 3;
    const int t = wg;                      // this warpgroup's row tile
    const bool active = t < Rg;
    const int row_in_tile = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
    const int bar_go = 1 + 2 * wg, bar_tile = 2 + 2 * wg;
    float yacc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) yacc[b] = 0.f;
    int s = 0, i = i_start, q = q_start, k = 0, gk = 0;
    uint32_t acc_ph = 0;
    int E = kZqSentinel;                   // set by the CTA's first non-empty unit
    // per-thread constant addresses: this row's 16-byte sign vector in stage 0, the two A slots
    const uint32_t sw_addr0 = smem_u32(smem) + (uint32_t)((t * kTileRows + row_in_tile) * 16);
    const uint32_t meta_addr0 = smem_u32(smem) + (uint32_t)(C::kOffZ + C::kZBytes);
    const uint32_t a_slot0 = tbase + (uint32_t)(C::kACols * P * t * NSLOT) + lane_base;
    uint32_t a_addr = a_slot0;
    const uint32_t a_flip = a_slot0 ^ (a_slot0 + (uint32_t)(C::kACols * P));   // slot 0 <-> slot 1
    static_assert(NSLOT == 2, "slot toggle");
    const long long row_abs = row0 + t * kTileRows + row_in_tile;
    while (active && k < nunits) {
      const int cnt = group_count<P>(k, q, nunits, p.nq);
      const bool last = (k + cnt == nunits) || (q + cnt == p.nq);
      if (warp == 5) BS_ITRACE(gk, 0);
      asm volatile("bar.sync %0, 160;" ::"r"(bar_go) : "memory");   // stage full, slot free
      if (warp == 5) BS_ITRACE(gk, 1);
      tc_fence_after();
      const uint32_t so = (uint32_t)(s * C::kStageBytes);
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (u < cnt) {
          uint4 sw;
          int e_u;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(sw.x), "=r"(sw.y), "=r"(sw.z), "=r"(sw.w)
                       : "r"(sw_addr0 + so + (uint32_t)(u * C::kUnitSign)));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(e_u) : "r"(meta_addr0 + so + (uint32_t)(u * C::kZUnit)));
          // A = +-2^a with a = E - e_u, so that A * (Z 2^e_u) = +-Z 2^E for every unit; E = e_u
          // of the CTA's first non-empty unit (the same in every warpgroup)
          if (E == kZqSentinel) E = e_u;
          const int a_raw = (e_u == kZqSentinel) ? 0 : E - e_u;
          const int a_exp = min(max(a_raw, -6), 8);
          if (a_exp != a_raw && lane == 0 && p.status) atomicOr(p.status, 1);   // beyond the e4m3 A range
          const uint32_t e8 = (uint32_t)((7 + a_exp) << 3) * 0x01010101u;
          uint32_t o[32];
#ifndef BS_EXP_SKEL   // timing experiment: no expansion / TMEM stores (wrong results)
          expand_e4m3(sw.x, e8, o);
          expand_e4m3(sw.y, e8, o + 8);
          expand_e4m3(sw.z, e8, o + 16);
          expand_e4m3(sw.w, e8, o + 24);
          tmem_st32(a_addr + (uint32_t)(C::kACols * u), o);
#else
          (void)o;
          if ((sw.x ^ sw.y ^ sw.z ^ sw.w ^ e8) == 0x12345u && p.status) p.status[1] = 1;
#endif
        }
      }
      if (warp == 5) BS_ITRACE(gk, 2);
      tmem_st_wait();
      if (warp == 5) BS_ITRACE(gk, 3);
      tc_fence_before();
      asm volatile("bar.arrive %0, 160;" ::"r"(bar_tile) : "memory");   // quarter in TMEM
      a_addr ^= a_flip;
      if (++s == STAGES) s = 0;
      const int ci = i;
      k += cnt;
      q += cnt;
      if (q == p.nq) { q = 0; ++i; }
      if (warp == 5) BS_ITRACE(gk, 4);
      ++gk;

      if (last) {
        // ---- epilogue for block ci: y += 2^-E sum_r U'_ci[row, r] (T_d0 + T_d1 + T_d2)[row, r]
        float uu[16];
        auto load_u = [&](long long blk) {
          const long long base = (blk * p.rows_pad + row_abs) * 16;
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
        };
        if (!p.kfuse) load_u(ci);
        mbar_wait(&acc_full[wg], acc_ph);
        acc_ph ^= 1;
        tc_fence_after();
        const float esc = exp2f((float)-E);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (p.kfuse) load_u(2LL * ci + b);     // rank half b of block ci
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
          if (p.kfuse) yacc[0] = fmaf(acc, esc, yacc[0]);
          else yacc[b] = fmaf(acc, esc, yacc[b]);
        }
        // the next block's first MMA (issued after this warpgroup's next tile-ready
        // barrier) overwrites the accumulator: order these tcgen05.ld before it
        tc_fence_before();
      }
    }
    if (active) {   // this CTA's partial y -> its split-K slot (zeros if it had no units)
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b < p.batch) store_partial(p, cta, R * kTileRows, t * kTileRows + row_in_tile, b, yacc[b]);
    }
  }

#undef BS_ITRACE
#ifdef BS_DECODE_TRACE
  if (p.dbg_acc && threadIdx.x == 0) {   // exit of the main phase (before the teardown barrier)
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    reinterpret_cast<long long*>(p.dbg_acc)[65536 + 4 * cta + 1] = (long long)gt;
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

template <int NB, int R_, int P_, int OCC_>
__global__ void __launch_bounds__(DecodeF8ICfg<NB, R_, P_, OCC_>::kThreads, OCC_) decode_f8i_kernel(const DecodeParams p) {
  decode_f8i_body<NB, R_, P_, OCC_>(p, (int)blockIdx.x);
}

// Grouped launch (bitstack_matmul_grouped): layers [0, count) of one launch, CTAs
// [cta_start[i], cta_start[i+1]) compute layer i -- several matrices that share a batch
// (e.g. the q/k/v projections of a token) pay the launch, the Zq dependency and the tail once.
constexpr int kMaxGroup = 8;
struct DecodeGroup {
  int count;
  int cta_start[kMaxGroup + 1];
  DecodeParams prm[kMaxGroup];
};

template <int NB, int R_, int P_, int OCC_>
__global__ void __launch_bounds__(DecodeF8ICfg<NB, R_, P_, OCC_>::kThreads, OCC_) decode_f8i_grouped_kernel(const __grid_constant__ DecodeGroup grp) {
  int i = 0;
  while (i + 1 < grp.count && (int)blockIdx.x >= grp.cta_start[i + 1]) ++i;
  decode_f8i_body<NB, R_, P_, OCC_>(grp.prm[i], (int)blockIdx.x - grp.cta_start[i]);
}

}  // namespace bs
