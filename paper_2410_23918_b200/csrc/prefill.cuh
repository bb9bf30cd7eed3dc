// Large-batch ("prefill") path for y = W_hat_n x, B >= kPrefillMinBatch.
//
// At large B the factored contraction S_i . (V_i (.) X) costs 2 n k B flops per sign element
// (120x the dense GEMM at B = 2048, SURVEY §8 finding 5), so this path materialises the
// restored weight tile by tile and runs one dense tensor-core GEMM:
//
//     W'  = sum_{i<n} S_i (.) (U'_i V'_i^T)          (Eq.5, Eq.8 P:135-138;
//                                                     U'V'^T = U V^T exactly)
//     X'  = X diag(1/s)                              (Eq.4: the scaling acts on x)
//     Y   = X' W'^T      i.e.  y[b, j] = sum_c W'[j, c] X'[b, c]  =  (W_hat_n x_b)[j]
//
// Three kernels:
//   xprep_kernel       X' rounded to fp16, written as a ready-to-copy UMMA operand image;
//   wtile_kernel       per (128-row tile, 64-column chunk): U'_i V'_i^T on tcgen05
//                      (kind::f16, bf16 factors, M = 128, N = 64, K = 16 -- exact products,
//                      fp32 accumulate in TMEM), sign application + sum over blocks in fp32
//                      registers (SHF + LOP3 + FADD per element and block), fp16 operand image;
//   prefill_gemm_kernel persistent tcgen05 GEMM, 256 x BN output tiles (two M = 128 MMAs
//                      sharing the B tile), 1D bulk copies (TMA engine) of the operand images
//                      into a STAGES-deep mbarrier ring, fp32 accumulators in TMEM, y written
//                      straight from the tcgen05.ld registers (coalesced along rows j).
// fp16 for both GEMM operands: W' ~ W s and X' = x / s are both well inside fp16 range; the
// rounding costs ~3e-4 relative L2 (tests/test_gpu_parity.py::test_prefill_*); bf16 would
// cost 8x more.
#pragma once
#include "decode_tc.cuh"

namespace bs {

constexpr int kPK = 64;                     // K (columns of W / x) per operand tile
constexpr int kImgTileA = 128 * kPK * 2;    // 16 KB: 128 rows x 64 fp16

// Operand image of R rows x 64 K fp16: 8-row x 16-byte core matrices at
// ((r / 8) * 8 + k / 8) * 128 -> K-major, no swizzle, LBO = 128 B (K-adjacent), SBO = 1024 B.
__host__ __device__ constexpr uint32_t img_off(int r, int k) {
  return (uint32_t)(((r >> 3) * 8 + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// ------------------------------------------------------------------ X' image
// Tiles (nt, c) of BN tokens x 64 columns, [nt][kc] order; one 16-byte core row per thread,
// dense in image order.  Tokens >= batch and columns >= d_in are zero.
__global__ void __launch_bounds__(256) xprep_kernel(const void* __restrict__ x, int x_dtype, long long x_stride,
                                                   const float* __restrict__ inv_s, int batch, int d_in,
                                                   int kc, int bn, long long pieces, uint4* __restrict__ img, bool vec,
                                                   const unsigned* __restrict__ xmax) {
  // X'_t = x_t / s scaled by 2^-e_t per token (|X'| < 2^14: fp16 in range for any scale of x, s)
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < pieces;
       e += (long long)gridDim.x * blockDim.x) {
    const long long tile = e / (bn * 8);
    const int p = (int)(e % (bn * 8));
    const int core = p >> 3, r8 = p & 7;
    const int g = core >> 3, k8 = core & 7;
    const int nt = (int)(tile / kc), c = (int)(tile % kc);
    const int tok = nt * bn + g * 8 + r8;
    const int col0 = c * kPK + k8 * 8;
    float v[8];
    if (vec && tok < batch && col0 + 8 <= d_in) {   // 16-byte aligned row segment: vector loads
      const float4 s0 = __ldg(reinterpret_cast<const float4*>(inv_s + col0));
      const float4 s1 = __ldg(reinterpret_cast<const float4*>(inv_s + col0) + 1);
      const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const long long o = (long long)tok * x_stride + col0;
      if (x_dtype == 0) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + o));
        const float4 b = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + o) + 1);
        const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = xv[t] * sc[t];
      } else {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(x) + o));
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 f;
          if (x_dtype == 1) f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[t]));
          else f = __half22float2(*reinterpret_cast<const __half2*>(&w[t]));
          v[2 * t] = f.x * sc[2 * t];
          v[2 * t + 1] = f.y * sc[2 * t + 1];
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int col = col0 + t;
        v[t] = (tok < batch && col < d_in) ? load_act(x, (long long)tok * x_stride + col, x_dtype) * __ldg(inv_s + col) : 0.f;
      }
    }
    const float xsc = tok < batch ? exp2i(-xs_exp(xmax[tok], 14)) : 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] *= xsc;
    img[e] = make_uint4(pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]), pack_half2(v[6], v[7]));
  }
}

// ------------------------------------------------------------------ W' image
struct WtileParams {
  const uint4* signs;     // [n_cap][nq][rows_pad] F8 device layout
  const uint16_t* u;      // [n_cap][rows_pad][16] U' (bf16 or f16 storage)
  const uint16_t* v;      // [n_cap][d_in_pad][16] V'
  const float* vmaxr;     // [n_cap][16] max_c |V'[c, r]|
  int f16;                // 1: fp16 factor storage (MMA format 0), 0: bf16 (format 1)
  uint8_t* img;           // [row_tiles_img][kc] tiles of kImgTileA bytes
  int* rowexp;            // [rows_pad] W' row j is stored as W'[j,:] 2^-rowexp[j] (fp16 range)
  int n, nq, rows_pad, row_tiles, row_tiles_img, kc;
  int ksh;                // sign tile of block i is i >> ksh (16-rank halves of a k > 16 block)
};

template <int G>  // blocks per MMA step
struct WtileCfg {
  static constexpr int kThreads = 256;
  static constexpr int kUBytes = 128 * 32;            // U' tile: 128 rows x 16 bf16
  static constexpr int kVBytes = kPK * 32;            // V' chunk: 64 rows x 16 bf16
  static constexpr int kVBufs = 3;
  static constexpr int kTmemCols = 2 * G * kPK;       // two buffers of G blocks x 64 columns
  static constexpr int kSmem(int n) { return n * kUBytes + kVBufs * G * kVBytes + 64; }
};

// Persistent: CTA b restores the contiguous range [T b / grid, T (b+1) / grid) of the
// T = row_tiles_img x kc (row tile, chunk) pairs in row-tile-major order, as "segments" of
// one row tile each (U'_i tiles reloaded per segment).  A step is (chunk c, group of G
// blocks): V' chunks stream in 2 steps ahead (cp.async), the MMAs of step t+1 run while the
// 256 threads apply the signs of step t (TMEM double buffer), sign words are fetched one
// step ahead.  Thread (quadrant q, half h) owns row 32q + lane, columns 32h..32h+31.
// Sign of column l (0..31) of word w of the F8 layout: bit (l & 3) * 8 + (l >> 2).
template <int G>
__global__ void __launch_bounds__(256, (2 * G * kPK <= 256) ? 2 : 1) wtile_kernel(const WtileParams p) {
  using C = WtileCfg<G>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* su = smem;                                   // [n] U' tiles (core layout)
  uint8_t* sv = smem + p.n * C::kUBytes;                // [3][G] V' chunks (core layout)
  uint64_t* mma_bar = reinterpret_cast<uint64_t*>(sv + C::kVBufs * G * C::kVBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;                // TMEM lane quadrant, 32-column half
  const int j = q * 32 + lane;                          // row within the tile
  const int NG = (p.n + G - 1) / G;
  const long long T = (long long)p.row_tiles_img * p.kc;
  const long long e0 = T * blockIdx.x / gridDim.x, e1 = T * (blockIdx.x + 1) / gridDim.x;

  if (tid == 0) {
    mbar_init(&mma_bar[0], 1);
    mbar_init(&mma_bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(q * 32) << 16;
  const uint32_t idesc = idesc_f16_f32(128, kPK, p.f16 ? 0u : 1u);   // bf16 / fp16 factors -> f32

  int gstep = 0;   // steps issued by this CTA so far (TMEM buffer = gstep & 1, barrier phase)
  for (long long e = e0; e < e1;) {
    const int mt = (int)(e / p.kc);
    const int c0 = (int)(e % p.kc);
    const int c1 = (int)((long long)p.kc < c0 + (e1 - e) ? (long long)p.kc : c0 + (e1 - e));
    e += c1 - c0;
    if (mt >= p.row_tiles) {            // padding row tile of the image: zeros
      for (int c = c0; c < c1; ++c) {
        uint8_t* dst = p.img + ((long long)mt * p.kc + c) * kImgTileA;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          *reinterpret_cast<uint4*>(dst + img_off(j, h * 32 + t * 8)) = make_uint4(0, 0, 0, 0);
      }
      continue;
    }
    const long long row = (long long)mt * 128 + j;
    const int S = (c1 - c0) * NG;
    const int sbase = gstep;

    for (int x = tid; x < p.n * 256; x += C::kThreads) {   // U' tiles: 16-byte pieces (row, K half)
      const int i = x >> 8, jj = (x & 255) >> 1, kk = x & 1;
      cp_async16(su + i * C::kUBytes + ((jj >> 3) * 2 + kk) * 128 + (jj & 7) * 16,
                 p.u + ((long long)i * p.rows_pad + mt * 128 + jj) * 16 + kk * 8);
    }
    cp_async_commit();
    // Per-thread constant parts of the addresses: G x 128 16-byte V' pieces per step, VP per thread.
    constexpr int VP = G * 128 / C::kThreads;
    static_assert(VP * C::kThreads == G * 128, "whole V' pieces per thread");
    const long long v_blk = (long long)p.kc * kPK * 32;                     // bytes per V' block
    const uint8_t* v_src[VP];
    uint32_t v_dst[VP];
    int v_gl[VP];
#pragma unroll
    for (int r = 0; r < VP; ++r) {
      const int x = tid + r * C::kThreads;
      const int gl = x >> 7, cc = (x & 127) >> 1, kk = x & 1;
      v_gl[r] = gl;
      v_src[r] = reinterpret_cast<const uint8_t*>(p.v) + gl * v_blk + cc * 32 + kk * 16;
      v_dst[r] = smem_u32(sv) + gl * C::kVBytes + ((cc >> 3) * 2 + kk) * 128 + (cc & 7) * 16;
    }
    const uint8_t* s_src = reinterpret_cast<const uint8_t*>(p.signs) + row * 16 + h * 4;
    const long long s_blk = (long long)p.nq * p.rows_pad * 16;              // bytes per sign block
    auto load_v = [&](int buf, int c, int gi) {   // V' chunk rows of one step -> SMEM buffer buf
#pragma unroll
      for (int r = 0; r < VP; ++r)
        if (gi * G + v_gl[r] < p.n)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(v_dst[r] + buf * (G * C::kVBytes)),
                       "l"(v_src[r] + (gi * G) * v_blk + c * (kPK * 32))
                       : "memory");
      cp_async_commit();
    };
    auto issue = [&](int buf, int tb, int gi) {   // one thread: the step's G MMAs into TMEM buffer tb
      tc_fence_after();
#pragma unroll
      for (int gl = 0; gl < G; ++gl) {
        const int i = gi * G + gl;
        if (i < p.n) {
          const uint64_t ad = smem_desc_kmajor(smem_u32(su + i * C::kUBytes), 128, 256);
          const uint64_t bd = smem_desc_kmajor(smem_u32(sv + (buf * G + gl) * C::kVBytes), 128, 256);
          mma_f16_ss(tbase + (uint32_t)(tb * G * kPK + gl * kPK), ad, bd, idesc, 0u);
        }
      }
      mma_commit(&mma_bar[tb]);
    };
    auto load_signs = [&](int c, int gi, uint32_t (&w)[G]) {
      const uint8_t* b = s_src + (long long)(c >> 1) * p.rows_pad * 16 + (c & 1) * 8;
#pragma unroll
      for (int gl = 0; gl < G; ++gl)
        w[gl] = gi * G + gl < p.n ? __ldg(reinterpret_cast<const uint32_t*>(b + ((gi * G + gl) >> p.ksh) * s_blk)) : 0u;
    };

    // (chunk, group) of steps s, s+1, s+2 -- advanced incrementally (no divisions in the loop)
    int c_0 = c0, g_0 = 0, c_1 = c0, g_1 = 0, c_2 = c0, g_2 = 0;
    auto adv = [&](int& c, int& g) { if (++g == NG) { g = 0; ++c; } };
    adv(c_1, g_1);
    adv(c_2, g_2);
    adv(c_2, g_2);
    int vb0 = sbase % C::kVBufs;                          // V' buffer of step s (rolls mod 3)
    load_v(vb0, c_0, g_0);
    if (S > 1) load_v(vb0 == C::kVBufs - 1 ? 0 : vb0 + 1, c_1, g_1);
    uint32_t sw[G], sw_next[G];
    load_signs(c_0, g_0, sw);
    if (S > 1) cp_async_wait<1>(); else cp_async_wait<0>();
    fence_proxy_async_smem();
    __syncthreads();                 // U' and V'(0) in SMEM (the previous segment's MMAs all waited)
    if (tid == 0) issue(vb0, sbase & 1, g_0);
    // |W'[row, c]| <= sum_i sum_r |U'_i[row, r]| max_c |V'_i[c, r]|: the row's fp16 image is
    // W' 2^-re with that bound below 2^15
    int re = 0;
    {
      float bound = 0.f;
      for (int i = 0; i < p.n; ++i)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint4 raw = *reinterpret_cast<const uint4*>(su + i * C::kUBytes + ((j >> 3) * 2 + kk) * 128 + (j & 7) * 16);
          const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 f = p.f16 ? __half22float2(*reinterpret_cast<const __half2*>(&wv[e2]))
                                   : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e2]));
            const int r = kk * 8 + 2 * e2;
            bound += fabsf(f.x) * __ldg(p.vmaxr + i * 16 + r) + fabsf(f.y) * __ldg(p.vmaxr + i * 16 + r + 1);
          }
        }
      if (bound > 0.f && bound < __int_as_float(0x7f800000)) re = xs_exp(__float_as_uint(bound), 15);
      if (h == 0 && c0 == 0) p.rowexp[row] = re;
    }
    const float wsc = exp2i(-re);
    float acc[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) acc[l] = 0.f;
    for (int s = 0; s < S; ++s) {
      const int gs = sbase + s;
      const int c = c_0, gi = g_0;
      if (s + 1 < S) load_signs(c_1, g_1, sw_next);
      const int vb1 = vb0 == C::kVBufs - 1 ? 0 : vb0 + 1, vb2 = vb1 == C::kVBufs - 1 ? 0 : vb1 + 1;
      if (s + 2 < S) load_v(vb2, c_2, g_2);
      if (s + 1 < S) {
        if (s + 2 < S) cp_async_wait<1>(); else cp_async_wait<0>();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();          // V'(s+1) in SMEM; TMEM buffer (gs+1)&1 drained by every thread
        if (tid == 0) issue(vb1, (gs + 1) & 1, g_1);
      }
      adv(c_0, g_0);
      adv(c_1, g_1);
      adv(c_2, g_2);
      vb0 = vb1;
      mbar_wait(&mma_bar[gs & 1], (uint32_t)((gs >> 1) & 1));
      tc_fence_after();
#pragma unroll
      for (int gl = 0; gl < G; ++gl) {
        if (gi * G + gl < p.n) {
          uint32_t m[32];
          tmem_ld32(tbase + lane_base + (uint32_t)((gs & 1) * G * kPK + gl * kPK + h * 32), m);
          tmem_ld_wait();
          const uint32_t nw = ~sw[gl];
#pragma unroll
          for (int l = 0; l < 32; l += 2) {   // LOP3 (sign) + SHF per element, one FADD2 per pair
            const int b0 = (l & 3) * 8 + (l >> 2), b1 = ((l + 1) & 3) * 8 + ((l + 1) >> 2);
            const float2 t = make_float2(__uint_as_float(m[l] ^ ((nw << (31 - b0)) & 0x80000000u)),
                                         __uint_as_float(m[l + 1] ^ ((nw << (31 - b1)) & 0x80000000u)));
            const float2 a = __fadd2_rn(make_float2(acc[l], acc[l + 1]), t);
            acc[l] = a.x;
            acc[l + 1] = a.y;
          }
        }
      }
      if (gi == NG - 1) {   // W'[row, chunk c] complete: fp16 operand image, reset
        uint8_t* dst = p.img + ((long long)mt * p.kc + c) * kImgTileA;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          *reinterpret_cast<uint4*>(dst + img_off(j, h * 32 + t * 8)) =
              make_uint4(pack_half2(acc[8 * t + 0] * wsc, acc[8 * t + 1] * wsc),
                         pack_half2(acc[8 * t + 2] * wsc, acc[8 * t + 3] * wsc),
                         pack_half2(acc[8 * t + 4] * wsc, acc[8 * t + 5] * wsc),
                         pack_half2(acc[8 * t + 6] * wsc, acc[8 * t + 7] * wsc));
        }
#pragma unroll
        for (int l = 0; l < 32; ++l) acc[l] = 0.f;
      }
#pragma unroll
      for (int gl = 0; gl < G; ++gl) sw[gl] = sw_next[gl];
    }
    gstep += S;
    tc_fence_before();
    __syncthreads();                 // every thread done with this segment's TMEM / SMEM
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::kTmemCols>(tbase);
}

// ------------------------------------------------------------------ GEMM  Y = X' W'^T
struct GemmParams {
  const uint8_t* a_img;   // W' image [row_tiles_img][kc] x 16 KB
  const uint8_t* b_img;   // X' image [nt_count][kc] x (BN x 128 B)
  void* y;                // [batch][y_stride]
  const int* rowexp;      // [rows_pad] W' row scale exponents (wtile_kernel)
  const unsigned* xmax;   // [batch] max_c |x_bc / s_c| (absmax_xs_kernel): the X' token scales
  int y_dtype;            // 0 f32, 1 bf16
  long long y_stride;
  int batch, rows_local, row_tiles, m2_count, nt_count, kc;   // m2_count: row-tile groups of MH
};

template <int BN, int MH>
struct GemmCfg {
  static constexpr int kThreads = 192;                 // producer, MMA, 4 epilogue warps
  static constexpr int kBBytes = BN * kPK * 2;
  static constexpr int kOffB = MH * kImgTileA;         // stage: MH A tiles (128 rows each), then B
  static constexpr int kStageBytes = kOffB + kBBytes;
  static constexpr int STAGES = (220 * 1024) / kStageBytes;
  static constexpr int NACC = 512 / (MH * BN);         // accumulator sets (128 MH x BN fp32 each)
  static constexpr int kSmemBytes = STAGES * kStageBytes + 256;
  static_assert(BN % 32 == 0 && BN <= 256, "BN");
  static_assert(MH == 1 || MH == 2, "MH");
  static_assert(NACC >= 1, "TMEM");
};

// Output tile = (128 MH rows) x BN tokens; tile t -> (row tile group mt = t / nt_count,
// token tile nt = t % nt_count); the MH row tiles share each B (X') stage.
template <int BN, int MH>
__global__ void __launch_bounds__(192, 1) prefill_gemm_kernel(const GemmParams p) {
  using C = GemmCfg<BN, MH>;
  constexpr int STAGES = C::STAGES, NACC = C::NACC;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = p.m2_count * p.nt_count;
  auto halves = [&](int mt) { const int left = p.row_tiles - MH * mt; return left < MH ? left : MH; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int mt = t / p.nt_count, nt = t % p.nt_count;
        const int nh = halves(mt);
        const uint32_t bytes = nh * kImgTileA + C::kBBytes;
        for (int c = 0; c < p.kc; ++c) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * C::kStageBytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          for (int h = 0; h < nh; ++h)
            bulk_g2s(st + h * kImgTileA, p.a_img + ((long long)(MH * mt + h) * p.kc + c) * kImgTileA, kImgTileA,
                     &full[s], pol_a);
          bulk_g2s(st + C::kOffB, p.b_img + ((long long)nt * p.kc + c) * C::kBBytes, C::kBBytes, &full[s], pol_b);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_f16_f32(128, BN, 0);   // fp16 x fp16 -> f32
    int s = 0, lt = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++lt) {
      const int nh = halves(t / p.nt_count);
      const int ab = lt % NACC;
      mbar_wait(&acc_empty[ab], (uint32_t)(((lt / NACC) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d0 = tbase + (uint32_t)(ab * MH * BN);
      for (int c = 0; c < p.kc; ++c) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * C::kStageBytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kPK / 16; ++kk) {
            const uint64_t bd = smem_desc_kmajor(st + C::kOffB + kk * 256, 128, 1024);
#pragma unroll
            for (int h = 0; h < MH; ++h)
              if (h < nh)
                mma_f16_ss(d0 + (uint32_t)(h * BN), smem_desc_kmajor(st + h * kImgTileA + kk * 256, 128, 1024), bd,
                           idesc, (c | kk) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          if (c == p.kc - 1) mma_commit(&acc_full[ab]);
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    const int q = warp & 3;                       // TMEM lane quadrant of this warp
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int lt = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++lt) {
      const int mt = t / p.nt_count, nt = t % p.nt_count;
      const int nh = halves(mt);
      const int ab = lt % NACC;
      mbar_wait(&acc_full[ab], (uint32_t)((lt / NACC) & 1));
      tc_fence_after();
      for (int hh = 0; hh < nh; ++hh) {
        const int j = (MH * mt + hh) * 128 + q * 32 + lane;
        const float sc = j < p.rows_local ? exp2i(p.rowexp[j]) : 0.f;   // undo the W' row scale
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t v[32];
          tmem_ld32(tbase + lane_base + (uint32_t)(ab * MH * BN + hh * BN + cc * 32), v);
          tmem_ld_wait();
          const int b0 = nt * BN + cc * 32;
          // and the X' token scales: lane l fetches token b0 + l's, the loop broadcasts them
          const float tf = exp2i(xs_exp(b0 + lane < p.batch ? __ldg(p.xmax + b0 + lane) : 0u, 14));
#pragma unroll
          for (int l = 0; l < 32; ++l)
            v[l] = __float_as_uint(__uint_as_float(v[l]) * (sc * __shfl_sync(0xffffffffu, tf, l)));
          if (j < p.rows_local) {
            if (p.y_dtype == 0) {
              float* yp = reinterpret_cast<float*>(p.y) + (long long)b0 * p.y_stride + j;
#pragma unroll
              for (int l = 0; l < 32; ++l)
                if (b0 + l < p.batch) __stcs(yp + (long long)l * p.y_stride, __uint_as_float(v[l]));
            } else {
              __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(p.y) + (long long)b0 * p.y_stride + j;
#pragma unroll
              for (int l = 0; l < 32; ++l)
                if (b0 + l < p.batch) yp[(long long)l * p.y_stride] = __float2bfloat16_rn(__uint_as_float(v[l]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tbase);
}

}  // namespace bs
