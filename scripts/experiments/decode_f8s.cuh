// EXPERIMENT (not built into the library): staggered warpgroups (4 chains on different units,
// (Written against the round-1 atomicAdd y workspace `p.y_acc`; the library now uses per-CTA
// split-K slots -- replace its fold/finalise with store_partial / finalize_group to rebuild.)
// shared double-buffered accumulators); correct, measured 31.8 us vs 28.3 us.
// e4m3 decode kernel with STAGGERED warpgroups -- the production decode
// kernel for bf16 / fp16 factors.
//
// Same computation and operands as decode_f8_kernel (decode_f8.cuh): y = sum_i sum_r
// U'_i[:,r] * (S_i (V'_i[:,r] * x/s)), S_i expanded to e4m3 +-2^a in TMEM, Z as three e4m3
// digits built by zq_kernel.  What differs is the schedule.  Measured on B200 (scripts/
// exp_decode.sh): with the tensor-core work and the TMEM stores compiled OUT, the
// warpgroup-per-row-tile kernel still needed 22 of its 28 us -- every warpgroup walked every
// unit, so the ~1300-cycle chain of hand-offs per unit (mbarrier waits ~150 cycles each,
// named barriers, elected issue blocks ~120) WAS the kernel.  Here the W = 4 warpgroups
// walk DIFFERENT units (warpgroup w takes units k = w, w + 4, ...) and each expands all R
// row tiles of its unit and issues their MMAs itself, so four chains run concurrently and
// the tensor pipe, not the chain latency, sets the pace.
//   * A slots: one per warpgroup (R tiles x 32 columns), released by its own commit.
//   * Accumulators are SHARED by the warpgroups (several issuers accumulate into the same
//     TMEM columns; all MMAs accumulate, so order does not matter) and double-buffered by
//     block parity; they are zeroed with tcgen05.st at start and after each drain.
//   * acc_full[b] completes when every warpgroup has closed block i (b = parity of i): a
//     tcgen05.commit after its last MMA of the block, or a plain arrive when it had no unit
//     in it.  The warpgroup that processed the block's last unit drains it (U'-weighted sum
//     over ranks and digits into per-thread y partials), re-zeroes the buffer and arrives on
//     acc_empty[b]; nobody touches buffer b for block i + 2 before that.
//   * E_i (the e4m3 scale reference of block i) is read from the Zq metadata in global
//     memory, so every warpgroup uses the same value for the block.
#pragma once
#include "../../paper_2410_23918_b200/csrc/decode_f8.cuh"

namespace bs {

template <int NB, int R_>
struct DecodeF8SCfg {
  static constexpr int N = ZqCfg<NB>::N;
  static constexpr int R = R_;                               // row tiles per CTA
  static constexpr int W = 4;                                // warpgroups (independent chains)
  static constexpr int kThreads = 32 * (4 * W + 1);          // + producer warp
  static constexpr int kWarpProducer = 4 * W;
  static constexpr int kZBytes = ZqCfg<NB>::kZBytes;
  static constexpr int kZUnit = ZqCfg<NB>::kZUnit;
  static constexpr int kSignBytes = R * kTileRows * 16;
  static constexpr int kOffZ = kSignBytes;
  static constexpr int kOffMeta = kOffZ + kZBytes;
  static constexpr int kStageBytes = (kOffZ + kZUnit + 127) / 128 * 128;
  static constexpr int S0 = (200 * 1024) / kStageBytes;
  static constexpr int STAGES = S0 > 16 ? 16 : (S0 < 2 * W ? 2 * W : S0);
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes = STAGES * kStageBytes + kBarBytes;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kACols = 32;                          // 128 rows x 128 e4m3 per tile
  static constexpr int kSlotCols = R * kACols;               // one warpgroup's A slot
  static constexpr uint32_t kAccCol = W * kSlotCols;
  static constexpr int ACCB = 2;                             // accumulator buffers (block parity)
  static constexpr uint32_t LBO = (N / 8) * 128;
  static constexpr uint32_t SBO = 128;
  static_assert(N <= 256 && N % 16 == 0, "invalid MMA N");
  static_assert(kAccCol + ACCB * R * N <= kTmemCols, "TMEM overflow");
  static_assert(kSmemBytes <= 227 * 1024, "smem overflow");
  static_assert(STAGES >= W, "every warpgroup needs a stage in flight");
};

// Zero this warp's lane quadrant of `cols` accumulator columns starting at taddr.
template <int COLS>
__device__ __forceinline__ void tmem_zero(uint32_t taddr) {
  static_assert(COLS % 16 == 0, "16-column granules");
  uint32_t z[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
  for (int c = 0; c < COLS; c += 16) tmem_st16(taddr + (uint32_t)c, z);
}

template <int NB, int R_>
__global__ void __launch_bounds__(DecodeF8SCfg<NB, R_>::kThreads, 1) decode_f8s_kernel(const DecodeParams p) {
  using C = DecodeF8SCfg<NB, R_>;
  constexpr int N = C::N, R = C::R, W = C::W, STAGES = C::STAGES, ACCB = C::ACCB;
  extern __shared__ __align__(1024) uint8_t smem[];

  uint8_t* bar_area = smem + STAGES * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_area);
  uint64_t* empty = full + STAGES;
  uint64_t* a_empty = empty + STAGES;     // [W]
  uint64_t* acc_full = a_empty + W;       // [ACCB] W closes per block
  uint64_t* acc_empty = acc_full + ACCB;  // [ACCB] 4 draining warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + ACCB);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x / p.ctas_per_group;
  const int jc = blockIdx.x % p.ctas_per_group;
  const long long L = (long long)p.n * p.nq;
  const long long u0 = L * jc / p.ctas_per_group;
  const long long u1 = L * (jc + 1) / p.ctas_per_group;
  const int nunits = (int)(u1 - u0);
  const int i_start = (int)(u0 / p.nq);
  const int i_end = nunits > 0 ? (int)((u1 - 1) / p.nq) : i_start - 1;   // last block in range
  const int tiles_left = p.row_tiles - g * R;
  const int Rg = tiles_left < R ? tiles_left : R;
  const int row0 = g * R * kTileRows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);             // the unit's warpgroup commits after its MMAs
    }
    for (int w = 0; w < W; ++w) mbar_init(&a_empty[w], 1);
    for (int b = 0; b < ACCB; ++b) {
      mbar_init(&acc_full[b], W);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == C::kWarpProducer) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (warp < 4) {   // zero both accumulator buffers (warpgroup 0, one lane quadrant per warp)
    tmem_zero<ACCB * R * N>(tbase + C::kAccCol + ((uint32_t)(warp * 32) << 16));
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == C::kWarpProducer) {
    if (lane == 0) {
      const uint64_t pol_sign = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      const uint32_t sign_bytes = (uint32_t)Rg * kTileRows * 16;
      const int pre = nunits < STAGES ? nunits : STAGES;
      int i = i_start, q = (int)(u0 % p.nq);
      for (int k = 0; k < pre; ++k) {  // sign tiles before the dependency wait (PDL overlap)
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
  } else {
    // ================= warpgroup wg: units k = wg, wg + W, ...; all Rg row tiles of each =================
    const int wg = warp >> 2;
    const int qd = warp & 3;
    const bool issuer = qd == 0;
    const int row_q = qd * 32 + lane;        // row within each tile
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t a_slot = tbase + (uint32_t)(wg * C::kSlotCols);
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
    float yacc[R][NB];
#pragma unroll
    for (int t = 0; t < R; ++t)
#pragma unroll
      for (int b = 0; b < NB; ++b) yacc[t][b] = 0.f;
    bool drained = false;
    int E = 0, e_block = -1;
    int closed = i_start;                    // blocks < closed: this warpgroup has closed them
    asm volatile("griddepcontrol.wait;" ::: "memory");   // Zq metadata is read from global memory

    // block-level protocol (see the header comment).  wait_buf: before this warpgroup's first
    // action for block i, buffer i & 1 must have been drained of block i - 2.
    auto wait_buf = [&](int i) {
      const int rel = i - i_start;
      if (rel >= ACCB && qd == 0) mbar_wait(&acc_empty[i & 1], (uint32_t)(((rel - ACCB) >> 1) & 1));
    };
    auto close_empty_blocks = [&](int upto) {   // plain arrive for blocks in [closed, upto)
      for (; closed < upto; ++closed) {
        wait_buf(closed);
        if (qd == 0 && lane == 0) mbar_arrive(&acc_full[closed & 1]);
      }
    };

    int j = 0;                               // this warpgroup's unit count (A-slot phase)
    for (int k = wg; k < nunits; k += W, ++j) {
      const long long u = u0 + k;
      const int i = (int)(u / p.nq), q = (int)(u % p.nq);
      // the next unit of this warpgroup (if any) is in block i_next
      const int i_next = k + W < nunits ? (int)((u + W) / p.nq) : i_end + 1;
      const bool closes = i_next != i;       // my last unit of block i
      close_empty_blocks(i);                 // blocks I skipped entirely
      if (e_block != i) wait_buf(i);         // first unit of block i for this warpgroup
      if (i != e_block) {
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
      if (qd == 0) {
        mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
        mbar_wait(&a_empty[wg], (uint32_t)((j & 1) ^ 1));
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
      tc_fence_after();
      const uint8_t* st = smem + s * C::kStageBytes;
      const int e_u = *reinterpret_cast<const int*>(st + C::kOffMeta);
      int a_exp = 0;
      if (e_u != kZqSentinel) {
        a_exp = E - e_u;
        if (a_exp < -6 || a_exp > 8) {      // |x/s| range across the block's units beyond e4m3 A range
          if (lane == 0 && p.status) atomicOr(p.status, 1);
          a_exp = a_exp < -6 ? -6 : 8;
        }
      }
      const uint32_t e8 = (uint32_t)((7 + a_exp) << 3) * 0x01010101u;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (t < Rg) {
          const uint4 sw = reinterpret_cast<const uint4*>(st)[t * kTileRows + row_q];
          uint32_t o[32];
          expand_e4m3(sw.x, e8, o);
          expand_e4m3(sw.y, e8, o + 8);
          expand_e4m3(sw.z, e8, o + 16);
          expand_e4m3(sw.w, e8, o + 24);
          tmem_st32(a_slot + (uint32_t)(t * C::kACols) + lane_base, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");   // all 4 lane quadrants in TMEM
      const int ab = i & 1;
      if (issuer) {
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(st + C::kOffZ), C::LBO, C::SBO);
          const uint32_t d_base = tbase + C::kAccCol + (uint32_t)(ab * R * N);
#pragma unroll
          for (int t = 0; t < R; ++t) {
            if (t < Rg) {
#pragma unroll
              for (int m = 0; m < kSubK / 32; ++m)
                mma_f8_ts(d_base + (uint32_t)(t * N), a_slot + (uint32_t)(t * C::kACols) + 8 * m,
                          bdesc0 + (uint64_t)((m * 2 * C::LBO) >> 4), idesc, 1u);
            }
          }
          mma_commit(&a_empty[wg]);
          mma_commit(&empty[s]);
          if (closes) mma_commit(&acc_full[ab]);
        }
        __syncwarp();
      }
      if (closes) closed = i + 1;
      const bool block_last = (k == nunits - 1) || (q == p.nq - 1);
      if (block_last) {
        // ---- drain block i (every warpgroup has closed it once acc_full completes)
        const int rel = i - i_start;
        float uu[R][16];
#pragma unroll
        for (int t = 0; t < R; ++t) {
          if (t < Rg) {
            const long long row = row0 + t * kTileRows + row_q;
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
                uu[t][2 * e] = f0.x; uu[t][2 * e + 1] = f0.y;
                uu[t][8 + 2 * e] = f1.x; uu[t][8 + 2 * e + 1] = f1.y;
              }
            } else {
              const float4* up = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.u) + base);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float4 f = __ldg(up + e);
                uu[t][4 * e] = f.x; uu[t][4 * e + 1] = f.y; uu[t][4 * e + 2] = f.z; uu[t][4 * e + 3] = f.w;
              }
            }
          }
        }
        mbar_wait(&acc_full[ab], (uint32_t)((rel >> 1) & 1));
        tc_fence_after();
        const float esc = exp2f((float)-E);
        const uint32_t d_base = tbase + C::kAccCol + (uint32_t)(ab * R * N) + lane_base;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          if (t < Rg) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              float tsum[16];
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                uint32_t v[16];
                tmem_ld16(d_base + (uint32_t)(t * N + (b * 3 + d) * 16), v);
                tmem_ld_wait();
#pragma unroll
                for (int r = 0; r < 16; ++r) tsum[r] = (d == 0) ? __uint_as_float(v[r]) : tsum[r] + __uint_as_float(v[r]);
              }
              float acc = 0.f;
#pragma unroll
              for (int r = 0; r < 16; ++r) acc = fmaf(uu[t][r], tsum[r], acc);
              yacc[t][b] = fmaf(acc, esc, yacc[t][b]);
            }
          }
        }
        drained = true;
        tmem_zero<R * N>(d_base);           // ready for block i + 2
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ab]);
      }
    }
    close_empty_blocks(i_end + 1);          // blocks after my last unit
    if (drained) {
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (t < Rg) {
          const int row = row0 + t * kTileRows + row_q;
#pragma unroll
          for (int b = 0; b < NB; ++b)
            if (b < p.batch) atomicAdd(p.y_acc + (long long)b * p.rows_pad + row, yacc[t][b]);
        }
      }
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
    if (threadIdx.x == 0) p.counters[g] = 0;
  }
}

}  // namespace bs
