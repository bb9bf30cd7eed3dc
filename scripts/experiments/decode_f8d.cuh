// EXPERIMENT (not built into the library; needs an int* wq [n_groups] field in DecodeParams):
// (Written against the round-1 atomicAdd y workspace `p.y_acc`; the library now uses per-CTA
// split-K slots -- replace its fold/finalise with store_partial / finalize_group to rebuild.)
// dynamic unit assignment; correct but 27.9 us vs 24.4 us static (shorter accumulation runs ->
// more drains, atomics on the producer path).  DESIGN.md §6.2.
// e4m3 decode kernel: per-warpgroup issuer warps + DYNAMIC unit assignment.
//
// Same computation and operands as decode_f8_kernel (decode_f8.cuh); same warp roles and
// hand-offs as decode_f8i_kernel (decode_f8i.cuh): R warpgroups (one row tile each) of 4
// expander warps + 1 issuer warp, and a producer warp.  What differs: the CTAs of a row group
// do not split the group's (block, subchunk) units into fixed contiguous ranges -- the
// producer grabs chunks of kChunk consecutive units from a per-group atomic work counter as
// its ring has room, so SMs that run faster take more units (measured on the static split:
// CTAs with equal unit counts finished up to 2.2 us apart, ~12% of the kernel).
//   * The producer writes each stage's unit index (or -1 = end) to SMEM before arming the
//     stage's mbarrier; consumers read it after the mbarrier wait.
//   * A warpgroup's accumulator runs over consecutive units of one block ("first" when the
//     unit does not continue the previous one, "last" when the next one does not continue
//     it); the issuer, which sees unit k+1 before releasing the expanders, publishes the
//     "last" flag of unit k, and the expanders drain after the release (the drain still
//     precedes unit k+1's tile hand-off, hence its accumulate-0 MMA).
//   * The last CTA of the group (finalisation) resets the group's work counter.
#pragma once
#include "../../paper_2410_23918_b200/csrc/decode_f8i.cuh"

namespace bs {

template <int NB, int R_>
struct DecodeF8DCfg : DecodeF8ICfg<NB, R_> {
#ifndef BS_DYN_CHUNK
#define BS_DYN_CHUNK 8
#endif
  static constexpr int kChunk = BS_DYN_CHUNK;                // units per grab
  static_assert((2 * DecodeF8ICfg<NB, R_>::STAGES + DecodeF8ICfg<NB, R_>::R * DecodeF8ICfg<NB, R_>::NSLOT +
                 DecodeF8ICfg<NB, R_>::R) * 8 + 8 + 4 * DecodeF8ICfg<NB, R_>::STAGES * (1 + DecodeF8ICfg<NB, R_>::R) <=
                    DecodeF8ICfg<NB, R_>::kBarBytes,
                "barrier area");
};

template <int NB, int R_>
__global__ void __launch_bounds__(DecodeF8DCfg<NB, R_>::kThreads, 1) decode_f8d_kernel(const DecodeParams p) {
  using C = DecodeF8DCfg<NB, R_>;
  constexpr int N = C::N, R = C::R, STAGES = C::STAGES, NSLOT = C::NSLOT;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_empty = empty + STAGES;       // [R][NSLOT] per warpgroup
  uint64_t* acc_full = a_empty + R * NSLOT; // [R]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + R);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  int* stage_unit = last_flag + 1;          // [STAGES] unit index in the group's unit space, -1 = end
  int* stage_last = stage_unit + STAGES;    // [STAGES][R] "last unit of an accumulation run" (issuer t -> its expanders)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x / p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int row0 = g * R * kTileRows;
  // named barriers of warpgroup w: go = 1 + 2w (issuer arrives, expanders sync), tile-ready =
  // 2 + 2w (expanders arrive, issuer syncs); single-buffered is race-free (decode_f8i.cuh).

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
      int pos = 0, end = 0;
      auto next_unit = [&]() -> int {
        if (pos >= end) {
          const int c = atomicAdd(p.wq + g, C::kChunk);
          if (c >= L) return -1;
          pos = c;
          end = c + C::kChunk < L ? c + C::kChunk : (int)L;
        }
        return pos++;
      };
      auto sign_copy = [&](int s, int u) {
        bulk_g2s(smem + s * C::kStageBytes, p.signs + (long long)u * p.rows_pad + row0, sign_bytes, &full[s], pol_sign);
      };
      // first ring fill: sign tiles before the dependency wait (PDL overlap), Zq after it
      int pre = 0;
      bool done = false;
      for (; pre < STAGES; ++pre) {
        const int u = next_unit();
        stage_unit[pre] = u;
        if (u < 0) {
          mbar_arrive(&full[pre]);
          done = true;
          break;
        }
        mbar_arrive_expect_tx(&full[pre], sign_bytes + C::kZUnit);
        sign_copy(pre, u);
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");  // Zq of this call is complete and visible
      for (int k = 0; k < pre; ++k)
        bulk_g2s(smem + k * C::kStageBytes + C::kOffZ, p.zq + (long long)stage_unit[k] * C::kZUnit, C::kZUnit,
                 &full[k], pol_keep);
      int s = 0;
      uint32_t ph = 1;          // stages 0..STAGES-1 used once: their next use waits phase 0 of empty
      while (!done) {
        mbar_wait(&empty[s], ph ^ 1);
        const int u = next_unit();
        stage_unit[s] = u;
        if (u < 0) {
          mbar_arrive(&full[s]);
          break;
        }
        mbar_arrive_expect_tx(&full[s], sign_bytes + C::kZUnit);
        sign_copy(s, u);
        bulk_g2s(smem + s * C::kStageBytes + C::kOffZ, p.zq + (long long)u * C::kZUnit, C::kZUnit, &full[s], pol_keep);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp % 5 == 4) {
    // ================= issuer of warpgroup t =================
    const int t = warp / 5;
    if (t < Rg) {
      constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
      const uint64_t bdesc_s0 = smem_desc_kmajor(smem_u32(smem + C::kOffZ), C::LBO, C::SBO);
      const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
      const int bar_go = 1 + 2 * t, bar_tile = 2 + 2 * t;
      int s = 0, slot = 0;
      int sn = 0, slotn = 0;
      uint32_t phn = 0, sphn = 0;
      mbar_wait(&full[0], 0);
      int u = stage_unit[0];
      if (u >= 0) mbar_wait(&a_empty[t * NSLOT], 1);
      asm volatile("bar.arrive %0, 160;" ::"r"(bar_go) : "memory");
      int prev = -2;
      int q = u >= 0 ? u % p.nq : 0;         // subchunk of u, tracked incrementally below
      while (u >= 0) {
        const bool first = (u != prev + 1) || (q == 0);
        if (++sn == STAGES) { sn = 0; phn ^= 1; }
        if (++slotn == NSLOT) { slotn = 0; sphn ^= 1; }
        mbar_wait(&full[sn], phn);
        const int un = stage_unit[sn];
        const bool last = (un != u + 1) || (q == p.nq - 1);   // includes un == -1
        if (un >= 0) mbar_wait(&a_empty[t * NSLOT + slotn], sphn ^ 1);
        if (lane == 0) stage_last[s * R + t] = last ? 1 : 0;
        __syncwarp();
        asm volatile("bar.sync %0, 160;" ::"r"(bar_tile) : "memory");   // unit's tile in TMEM
        asm volatile("bar.arrive %0, 160;" ::"r"(bar_go) : "memory");   // next unit (or the end)
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bdesc0 = bdesc_s0 + (uint64_t)((s * C::kStageBytes) >> 4);
          const uint32_t a_col = tbase + (uint32_t)(C::kACols * (t * NSLOT + slot));
#pragma unroll
          for (int m = 0; m < kSubK / 32; ++m)
            mma_f8_ts(d_acc, a_col + 8 * m, bdesc0 + (uint64_t)((m * 2 * C::LBO) >> 4), idesc,
                      (m > 0 || !first) ? 1u : 0u);
          mma_commit(&a_empty[t * NSLOT + slot]);
          mma_commit(&empty[s]);
          if (last) mma_commit(&acc_full[t]);
        }
        __syncwarp();
        prev = u;
        if (un == u + 1) q = (q + 1 == p.nq) ? 0 : q + 1;
        else if (un >= 0) q = un % p.nq;
        u = un;
        s = sn;
        slot = slotn;
      }
    }
  } else {
    // ================= expander warps of warpgroup wg (TMEM lane quadrant = warp % 4) =================
    const int wg = warp / 5;
    const int qd = warp & 3;
    const int t = wg;
    const bool active = t < Rg;
    const int row_in_tile = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t d_acc = tbase + C::kAccCol + (uint32_t)(t * N);
    const int bar_go = 1 + 2 * wg, bar_tile = 2 + 2 * wg;
    float yacc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) yacc[b] = 0.f;
    bool any = false;
    int s = 0, slot = 0, s_prev = -1;
    int u_prev = -1;
    uint32_t acc_ph = 0;
    int E = 0;
    bool have_e = false;
    while (active) {
      asm volatile("bar.sync %0, 160;" ::"r"(bar_go) : "memory");   // stage full, slot free (or end)
      if (s_prev >= 0 && stage_last[s_prev * R + t]) {
        // ---- drain the run that ended with unit u_prev: y += 2^-E sum_r U'_i[row, r] T[row, r]
        const int ci = u_prev / p.nq;
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
        any = true;
        // the next run's first MMA (issued after this warpgroup's next tile hand-off) overwrites
        // the accumulator: order these tcgen05.ld before it
        tc_fence_before();
      }
      const int u = stage_unit[s];
      if (u < 0) break;
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
      asm volatile("bar.arrive %0, 160;" ::"r"(bar_tile) : "memory");   // quarter in TMEM
      u_prev = u;
      s_prev = s;
      if (++slot == NSLOT) slot = 0;
      if (++s == STAGES) s = 0;
    }
    if (any) {
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
  if (warp == C::kWarpProducer) tmem_dealloc<C::kTmemCols>(tbase);
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
    if (threadIdx.x == 0) {
      p.counters[g] = 0;
      p.wq[g] = 0;
    }
  }
}

}  // namespace bs
