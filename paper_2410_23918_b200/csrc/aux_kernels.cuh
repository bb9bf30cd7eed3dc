// Load-time and reference kernels of the BitStack library (sm_100a):
//   repack_signs_kernel   canonical packed bits -> device tile layout (bijective, bit-exact)
//   prep_factors_kernel   per-(block, r) power-of-two rebalancing U' = U 2^-e, V' = V 2^e
//   inv_s_kernel          1/s (Eq.4 P:111 diag(1/s)), zero in the pad
//   matmul_simt_kernel    K0: FP32 CUDA-core y = sum_i sum_r u (.) S (v (.) x/s) (any shape)
//   reconstruct_kernel    K2: W_hat_n = sum_i (S_i (.) U_i V_i^T) diag(1/s)  (Eq.8 + Eq.4)
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace bs {

// Device sign layouts: per block, per 128-column subchunk q, per
// (padded) local row j, one uint4 = 4 words.  Bit p of word w holds column
//   layout 0 ("F16", fp16 A operand):  c = 128 q + 32 w + 2 (p & 15) + (p >> 4)
//   layout 1 ("F8",  e4m3 A operand):  c = 128 q + 32 w + 4 (p & 7)  + (p >> 3)
// so that one LOP3 + one IMAD expands a pair (fp16) or a quad (e4m3) of K-adjacent
// elements.  Pad rows/columns hold bit 0 (-1); Z and U are 0 there.
__host__ __device__ __forceinline__ int dev_bit_to_col(int layout, int w, int p) {
  return layout == 0 ? 32 * w + 2 * (p & 15) + (p >> 4) : 32 * w + 4 * (p & 7) + (p >> 3);
}
__host__ __device__ __forceinline__ int col_to_dev_bit(int layout, int cl /*0..31*/) {
  return layout == 0 ? (cl >> 1) + 16 * (cl & 1) : (cl >> 2) + 8 * (cl & 3);
}

__global__ void repack_signs_kernel(const uint8_t* __restrict__ canon, uint32_t* __restrict__ dev,
                                    int count, long long canon_bytes, long long d_in, int nq,
                                    int rows_pad, long long rows_local, long long row_begin, int layout) {
  const long long words_per_block = (long long)nq * rows_pad * 4;
  const long long total = words_per_block * count;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int blk = (int)(e / words_per_block);
    long long rem = e % words_per_block;
    const int q = (int)(rem / ((long long)rows_pad * 4));
    rem %= (long long)rows_pad * 4;
    const int j = (int)(rem / 4);
    const int w = (int)(rem % 4);
    uint32_t word = 0;
    if (j < rows_local) {
      const long long rowg = row_begin + j;
      const uint8_t* src = canon + (long long)blk * canon_bytes;
#pragma unroll 4
      for (int pb = 0; pb < 32; ++pb) {
        const long long c = 128LL * q + dev_bit_to_col(layout, w, pb);
        if (c < d_in) {
          const long long bit = rowg * d_in + c;
          word |= (uint32_t)((src[bit >> 3] >> (bit & 7)) & 1u) << pb;
        }
      }
    }
    dev[e] = word;
  }
}

// Fast repack for byte-aligned rows (d_in % 8 == 0), used by the block loads: one thread per
// (block, local row, 128-column subchunk) with the subchunk index fastest, so a warp reads
// consecutive 16-byte pieces of one canonical row (coalesced), and stores the row's 16
// device-layout bytes as one uint4.  Columns >= d_in and rows >= rows_local become 0 bits,
// as in repack_signs_kernel.  `canon` points at local row 0 of block 0 (the caller copies
// just the shard's rows); consecutive blocks are `canon_stride` bytes apart.
// The bit permutation inside a 32-bit word maps the 5-bit column index (layout 1:
// cl = 4a + b -> 8b + a; layout 0: cl = 2a + b -> 16b + a) and is applied per canonical byte
// through a 256-entry table: byte k holds columns 8k..8k+7, whose device positions are the
// table entry of that byte shifted by 2k (layout 1) or 4k (layout 0).
__global__ void repack_rows_kernel(const uint8_t* __restrict__ canon, long long canon_stride, uint4* __restrict__ dev,
                                   int count, long long d_in, int nq, int rows_pad, long long rows_local, int layout) {
  __shared__ uint32_t lut[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    uint32_t o = 0;
    for (int bit = 0; bit < 8; ++bit)
      if ((v >> bit) & 1) o |= 1u << col_to_dev_bit(layout, bit);   // column bit of byte 0
    lut[v] = o;
  }
  __syncthreads();
  const int sh = layout == 1 ? 2 : 4;   // device-position shift per canonical byte
  const long long per_block = (long long)rows_pad * nq;
  const long long total = per_block * count;
  const long long row_bytes = d_in / 8;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int blk = (int)(e / per_block);
    const long long rem = e % per_block;
    const int j = (int)(rem / nq);
    const int q = (int)(rem % nq);
    uint32_t in[4] = {0u, 0u, 0u, 0u};
    if (j < rows_local) {
      const uint8_t* src = canon + blk * canon_stride + j * row_bytes + 16LL * q;
      const long long nb = row_bytes - 16LL * q;
      if (nb >= 16 && (reinterpret_cast<uintptr_t>(src) & 3) == 0) {
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
#pragma unroll
        for (int w = 0; w < 4; ++w) in[w] = __ldg(s4 + w);
      } else {
        for (int b = 0; b < 16 && b < nb; ++b) in[b >> 2] |= (uint32_t)__ldg(src + b) << (8 * (b & 3));
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t o = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) o |= lut[(in[w] >> (8 * k)) & 0xFFu] << (sh * k);
      out[w] = o;
    }
    dev[((long long)blk * nq + q) * rows_pad + j] = make_uint4(out[0], out[1], out[2], out[3]);
  }
}

__device__ __forceinline__ float ld_factor(const void* p, long long idx, int dt) {
  if (dt == 0) return reinterpret_cast<const float*>(p)[idx];
  if (dt == 1) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return __half2float(reinterpret_cast<const __half*>(p)[idx]);
}

// Parallel form of prep_factors_kernel for one block (the block loads): factor_max_kernel
// reduces max_c |V[c, r]| into vmax[16] (float bits as uint: |v| >= 0 orders like its bits;
// vmax zeroed before), factor_scale_kernel derives the same power-of-two e_r and writes
// U' = U 2^-e_r, V' = V 2^e_r (rows_pad x 16 and d_in_pad x 16, zero padded) and zscale.
// The input is the stored [rows, ld] factor; columns [col0, col0 + k) (k <= 16) form one rank
// half (k > 16 is held as two 16-rank halves sharing the sign tile).
__global__ void factor_max_kernel(const void* __restrict__ v_in, int in_dt, int ld, int col0, int k, long long d_in,
                                  unsigned int* __restrict__ vmax) {
  __shared__ float red[16];
  if (threadIdx.x < 16) red[threadIdx.x] = 0.f;
  __syncthreads();
  float m[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) m[r] = 0.f;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d_in; c += (long long)gridDim.x * blockDim.x)
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < k) m[r] = fmaxf(m[r], fabsf(ld_factor(v_in, c * ld + col0 + r, in_dt)));
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    float x = m[r];
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(&red[r]), __float_as_uint(x));
  }
  __syncthreads();
  if (threadIdx.x < 16) atomicMax(vmax + threadIdx.x, __float_as_uint(red[threadIdx.x]));
}

__device__ __forceinline__ float factor_scale(const unsigned int* vmax, int r) {
  const float m = __uint_as_float(vmax[r]);
  int e = 0;
  if (m > 0.f && isfinite(m)) {
    e = (int)floorf(log2f(256.0f / m));
    e = e > 60 ? 60 : (e < -60 ? -60 : e);
  }
  return ldexpf(1.0f, e);
}

// U' = U / 2^e_r, V' = V 2^e_r (exact power-of-two rebalancing, U'V'^T == UV^T) into the device
// dtype out_dt (0 f32, 1 bf16, 2 f16).  fp16 storage is NOT rebalanced (e_r = 0): fp16's range is
// too small for U / 2^e_r, and the stored fp16 values are kept bit for bit (Eq.9's 16-bit
// factors); the MX decode's per-K-block scales do not need max |V'| near 2^8.
// vmaxr_out[r] = max_c |V'[c, r]| (the prefill restore's per-row fp16 range bound).
__global__ void factor_scale_kernel(const void* __restrict__ u_in, const void* __restrict__ v_in, int in_dt, int ld,
                                    int col0, int k, long long rows_local, int rows_pad, long long d_in, long long d_in_pad,
                                    const unsigned int* __restrict__ vmax, void* u_out, void* v_out, int out_dt,
                                    float* zscale_out, float* vmaxr_out) {
  __shared__ float scale[16];
  if (threadIdx.x < 16) scale[threadIdx.x] = out_dt == 2 ? 1.f : factor_scale(vmax, threadIdx.x);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 16 && zscale_out) zscale_out[threadIdx.x] = scale[threadIdx.x];
  if (blockIdx.x == 0 && threadIdx.x < 16 && vmaxr_out)
    vmaxr_out[threadIdx.x] = __uint_as_float(vmax[threadIdx.x]) * scale[threadIdx.x];
  const long long nu = (long long)rows_pad * 16, nv = d_in_pad * 16;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nu + nv;
       e += (long long)gridDim.x * blockDim.x) {
    float val = 0.f;
    if (e < nu) {
      const long long j = e / 16;
      const int r = (int)(e % 16);
      if (j < rows_local && r < k) val = ld_factor(u_in, j * ld + col0 + r, in_dt) / scale[r];
      if (out_dt == 0) reinterpret_cast<float*>(u_out)[e] = val;
      else if (out_dt == 1) reinterpret_cast<__nv_bfloat16*>(u_out)[e] = __float2bfloat16_rn(val);
      else reinterpret_cast<__half*>(u_out)[e] = __float2half_rn(val);
    } else {
      const long long ev = e - nu;
      const long long c = ev / 16;
      const int r = (int)(ev % 16);
      if (c < d_in && r < k) val = ld_factor(v_in, c * ld + col0 + r, in_dt) * scale[r];
      if (out_dt == 0) reinterpret_cast<float*>(v_out)[ev] = val;
      else if (out_dt == 1) reinterpret_cast<__nv_bfloat16*>(v_out)[ev] = __float2bfloat16_rn(val);
      else reinterpret_cast<__half*>(v_out)[ev] = __float2half_rn(val);
    }
  }
}

__global__ void inv_s_kernel(const float* __restrict__ s, float* __restrict__ inv_s, long long d_in,
                             long long d_in_pad) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d_in_pad;
       c += (long long)gridDim.x * blockDim.x)
    inv_s[c] = c < d_in ? 1.0f / s[c] : 0.0f;
}

__device__ __forceinline__ float ld_dev_factor(const void* p, long long idx, int dt) {   // 0 f32, 1 bf16, 2 f16
  if (dt == 0) return reinterpret_cast<const float*>(p)[idx];
  if (dt == 1) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return __half2float(reinterpret_cast<const __half*>(p)[idx]);
}
__device__ __forceinline__ float ld_act(const void* p, long long idx, int dt) {
  if (dt == 0) return reinterpret_cast<const float*>(p)[idx];
  if (dt == 1) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
  return __half2float(reinterpret_cast<const __half*>(p)[idx]);
}

// K0: one CTA = one 128-row tile x one batch column; one thread = one row.
// T_r = sum_c S[j,c] Z[c,r] in FP32 FMA, then y += sum_r U'[j,r] T_r per block.
__global__ void __launch_bounds__(128) matmul_simt_kernel(
    const uint4* __restrict__ signs, const void* __restrict__ u, const void* __restrict__ v,
    const float* __restrict__ inv_s, const void* __restrict__ x, void* __restrict__ y, int n,
    int nq, int rows_pad, long long rows_local, long long d_in, long long d_in_pad, int f_dt,
    int x_dt, int y_dt, long long x_stride, long long y_stride, int layout, int ksh) {
  __shared__ float zs[128][17];
  const int tile = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int row = tile * 128 + tid;
  float yv = 0.f;
  for (int i = 0; i < n; ++i) {
    float t[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) t[r] = 0.f;
    for (int q = 0; q < nq; ++q) {
      __syncthreads();
      {
        const long long c = (long long)q * 128 + tid;
        const float xs = c < d_in ? ld_act(x, b * x_stride + c, x_dt) * inv_s[c] : 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          zs[tid][r] = ld_dev_factor(v, ((long long)i * d_in_pad + c) * 16 + r, f_dt) * xs;
      }
      __syncthreads();
      const uint4 sw = signs[((long long)(i >> ksh) * nq + q) * rows_pad + row];   // rank half i of block i >> ksh
      const uint32_t words[4] = {sw.x, sw.y, sw.z, sw.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        for (int pb = 0; pb < 32; ++pb) {
          const float sg = ((words[w] >> pb) & 1u) ? 1.f : -1.f;
          const int c = dev_bit_to_col(layout, w, pb);
#pragma unroll
          for (int r = 0; r < 16; ++r) t[r] = fmaf(sg, zs[c][r], t[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) yv = fmaf(ld_dev_factor(u, ((long long)i * rows_pad + row) * 16 + r, f_dt), t[r], yv);
  }
  if (row < rows_local) {
    const long long o = b * y_stride + row;
    if (y_dt == 0) reinterpret_cast<float*>(y)[o] = yv;
    else reinterpret_cast<__nv_bfloat16*>(y)[o] = __float2bfloat16_rn(yv);
  }
}

// K2: one thread per output element, 32x8 tiles; U'/V' of the tile cached in SMEM per block.
__global__ void __launch_bounds__(256) reconstruct_kernel(
    const uint4* __restrict__ signs, const void* __restrict__ u, const void* __restrict__ v,
    const float* __restrict__ inv_s, void* __restrict__ w, int n, int nq, int rows_pad,
    long long rows_local, long long d_in, long long d_in_pad, int f_dt, int w_dt, int layout, int ksh) {
  __shared__ float us[8][16];
  __shared__ float vs[32][17];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long c = (long long)blockIdx.x * 32 + tx;
  const long long row = (long long)blockIdx.y * 8 + ty;
  float acc = 0.f;
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    if (threadIdx.x < 128) {
      const int rr = threadIdx.x / 16, r = threadIdx.x % 16;
      const long long rw = (long long)blockIdx.y * 8 + rr;
      us[rr][r] = rw < rows_pad ? ld_dev_factor(u, ((long long)i * rows_pad + rw) * 16 + r, f_dt) : 0.f;
    }
    for (int e = threadIdx.x; e < 32 * 16; e += 256) {
      const int cc = e / 16, r = e % 16;
      const long long cg = (long long)blockIdx.x * 32 + cc;
      vs[cc][r] = cg < d_in_pad ? ld_dev_factor(v, ((long long)i * d_in_pad + cg) * 16 + r, f_dt) : 0.f;
    }
    __syncthreads();
    if (row < rows_local && c < d_in) {
      float m = 0.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) m = fmaf(us[ty][r], vs[tx][r], m);
      const int q = (int)(c / 128), cl = (int)(c % 128);
      const uint4 sw = signs[((long long)(i >> ksh) * nq + q) * rows_pad + row];
      const uint32_t words[4] = {sw.x, sw.y, sw.z, sw.w};
      const uint32_t word = words[cl / 32];
      const int pb = col_to_dev_bit(layout, cl % 32);
      acc += ((word >> pb) & 1u) ? m : -m;
    }
  }
  if (row < rows_local && c < d_in) {
    const float val = acc * inv_s[c];
    const long long o = row * d_in + c;
    if (w_dt == 0) reinterpret_cast<float*>(w)[o] = val;
    else if (w_dt == 1) reinterpret_cast<__nv_bfloat16*>(w)[o] = __float2bfloat16_rn(val);
    else reinterpret_cast<__half*>(w)[o] = __float2half_rn(val);
  }
}

}  // namespace bs
