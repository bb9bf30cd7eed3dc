// Device kernels of the GPU compression loop (bitstack_compress):
// Alg.1 P:423-445 for one weight matrix -- activation-aware scaling (Eq.3-4) once, then n
// absolute-value decompositions (Eq.5-7) of the running residual.  The skinny GEMMs with |R|
// and the tall-skinny products run in cuBLAS (fp32 SGEMM); these
// kernels are the element-wise and reduction steps around it, plus the two ell x ell dense
// steps (CholeskyQR's Cholesky + triangular inverse, the Jacobi eigensolver of B B^T).
//   colsq_kernel        s_c^2 = sum_t x_cal[t, c]^2 (fp64 accumulation, Eq.3)
//   scale_clamp_kernel  s_c = max(sqrt(s_c^2), 1e-8 max s), R_0 = W diag(s) (Eq.4)
//   sign_abs_kernel     canonical packed S = sign(R) (sign(0) = +1) and M = |R| (Eq.5)
//   gauss_kernel        seeded standard-normal test matrix (counter-based Philox)
//   factor_out_kernel   U = a sqrt(sigma), V = b sqrt(sigma) with the sign convention, rounded
//                       to the storage dtype (Eq.2 split), written in the canonical layouts
//   residual_kernel     R -= S (.) (U V^T) with the ROUNDED factors, sum R^2 (Eq.7)
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <curand_kernel.h>
#include <cstdint>

namespace bs {

// x_cal [p, d_in] row-major; one thread per column, rows strided over blockIdx.y slices.
__global__ void colsq_kernel(const float* __restrict__ x, long long p, long long d_in, double* __restrict__ s2) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= d_in) return;
  double acc = 0.0;
  for (long long t = blockIdx.y; t < p; t += gridDim.y) {
    const double v = x[t * d_in + c];
    acc += v * v;
  }
  atomicAdd(s2 + c, acc);
}

// s = sqrt(s2) clamped at 1e-8 * max (reading R5 / SPEC S:116), written as fp32; smax holds
// max_c s2 as the bits of a non-negative double (monotone in its bits).
__global__ void colmax_kernel(const double* __restrict__ s2, long long d_in, unsigned long long* __restrict__ smax) {
  unsigned long long m = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d_in; c += (long long)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)__double_as_longlong(s2[c]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(smax, m);
}

__global__ void scale_clamp_kernel(const double* __restrict__ s2, const unsigned long long* __restrict__ smax,
                                   long long d_in, float* __restrict__ s_out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= d_in) return;
  const double top = sqrt(__longlong_as_double((long long)*smax));
  const double floor_ = top > 0.0 ? 1e-8 * top : 1e-8;
  s_out[c] = (float)fmax(sqrt(s2[c]), floor_);
}

// R = W diag(s): column c times s_c (fp32; "diag(s) W" in the paper's orientation).
__global__ void scale_w_kernel(const float* __restrict__ w, const float* __restrict__ s, long long d_out,
                               long long d_in, float* __restrict__ r) {
  const long long total = d_out * d_in;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
    r[e] = w[e] * s[e % d_in];
}

// Canonical packing (bit e = element e of the row-major [d_out, d_in] matrix, LSB first,
// 1 = +1): one thread per output byte; pad bits 0.  Also M = |R| for the SVD.
// Block-indexed outputs (signs, factors, sigma, residual norms) are addressed through the
// device-side block counter *bi, so one captured CUDA graph of a block's work serves every block.
__global__ void sign_abs_kernel(const float* __restrict__ r, long long total, uint8_t* __restrict__ signs_base,
                                const int* __restrict__ bi, float* __restrict__ m) {
  const long long nbytes = (total + 7) / 8;
  uint8_t* signs = signs_base + (long long)*bi * nbytes;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nbytes; b += (long long)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const long long e = 8 * b + i;
      if (e < total) {
        const float v = r[e];
        byte |= (v >= 0.f ? 1u : 0u) << i;   // sign(0) = +1 (reading R6)
        m[e] = fabsf(v);
      }
    }
    signs[b] = (uint8_t)byte;
  }
}

__global__ void gauss_kernel(float* __restrict__ out, long long count, unsigned long long seed0,
                             const int* __restrict__ bi) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const unsigned long long seed = seed0 + 7919ull * (unsigned long long)*bi;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, (unsigned long long)i, 0, &st);
  out[i] = curand_normal(&st);
}

// Column r < k of a (col-major [d_out, ld_a], orthonormal left vectors) and b (col-major
// [d_in, ld_b] = B^T w_r = sigma_r x the right vector) with sigma_r: the largest-|entry| of
// a[:, r] is made positive (ties -> lowest index) and
// U[j, r] = a[j, r] sqrt(sigma_r), V[c, r] = b[c, r] / sqrt(sigma_r) rounded to out_dt
// (0 f32, 1 bf16 RNE, 2 f16) into the row-major [rows, k] outputs; the rounded values are
// also kept as f32 ([rows, k]) for the residual update.  One CTA per r.
__global__ void factor_out_kernel(const float* __restrict__ a, long long lda, const float* __restrict__ b,
                                  long long ldb, const float* __restrict__ sigma, long long d_out, long long d_in,
                                  int k, int out_dt, void* __restrict__ u_base, void* __restrict__ v_base,
                                  const int* __restrict__ blk_i, float* __restrict__ u_f, float* __restrict__ v_f) {
  const int r = blockIdx.x;
  const int fsz = out_dt == 0 ? 4 : 2;
  void* u_out = reinterpret_cast<uint8_t*>(u_base) + (long long)*blk_i * d_out * k * fsz;
  void* v_out = reinterpret_cast<uint8_t*>(v_base) + (long long)*blk_i * d_in * k * fsz;
  __shared__ float best_v[32];
  __shared__ long long best_i[32];
  __shared__ float sgn_s;
  float bv = -1.f;
  long long bi = 0;
  for (long long j = threadIdx.x; j < d_out; j += blockDim.x) {
    const float v = fabsf(a[r * lda + j]);
    if (v > bv) { bv = v; bi = j; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { best_v[threadIdx.x >> 5] = bv; best_i[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (best_v[w] > bv || (best_v[w] == bv && best_i[w] < bi)) { bv = best_v[w]; bi = best_i[w]; }
    sgn_s = a[r * lda + bi] < 0.f ? -1.f : 1.f;
  }
  __syncthreads();
  // U = a sqrt(sigma); V = b sqrt(sigma) with b = (B^T w_r) / sigma given unnormalised in b
  const float sg = fmaxf(sigma[r], 0.f);
  const float root = sqrtf(sg) * sgn_s;
  const float broot = sg > 0.f ? sgn_s / sqrtf(sg) : 0.f;
  for (long long e = threadIdx.x; e < d_out + d_in; e += blockDim.x) {
    const bool is_u = e < d_out;
    const long long j = is_u ? e : e - d_out;
    const float x = is_u ? a[r * lda + j] * root : b[r * ldb + j] * broot;
    float xr;
    void* out = is_u ? u_out : v_out;
    const long long o = j * k + r;
    if (out_dt == 1) {
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      reinterpret_cast<__nv_bfloat16*>(out)[o] = h;
      xr = __bfloat162float(h);
    } else if (out_dt == 2) {
      const __half h = __float2half_rn(x);
      reinterpret_cast<__half*>(out)[o] = h;
      xr = __half2float(h);
    } else {
      reinterpret_cast<float*>(out)[o] = x;
      xr = x;
    }
    (is_u ? u_f : v_f)[o] = xr;
  }
}

// R[j, c] -= sign(R[j, c]) sum_r U[j, r] V[c, r] (k <= 32), and sum R_new^2 (fp64).  Tile of
// 16 rows x 256 columns per CTA: U rows in shared memory, each thread's V row in registers,
// coalesced along the row.
constexpr int kResRows = 16;
__global__ void __launch_bounds__(256) residual_kernel(float* __restrict__ r, const float* __restrict__ u_f,
                                                       const float* __restrict__ v_f, long long d_out, long long d_in,
                                                       int k, double* __restrict__ sumsq_base, const int* __restrict__ bi) {
  double* sumsq = sumsq_base + *bi + 1;
  __shared__ float us[kResRows][32];
  const long long c = blockIdx.x * 256LL + threadIdx.x;
  const long long j0 = (long long)blockIdx.y * kResRows;
  for (int e = threadIdx.x; e < kResRows * 32; e += 256) {
    const int jj = e / 32, q = e % 32;
    us[jj][q] = (q < k && j0 + jj < d_out) ? u_f[(j0 + jj) * k + q] : 0.f;
  }
  float vr[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) vr[q] = (q < k && c < d_in) ? v_f[c * k + q] : 0.f;
  __syncthreads();
  double acc = 0.0;
  if (c < d_in) {
    for (int jj = 0; jj < kResRows && j0 + jj < d_out; ++jj) {
      float dot = 0.f;
#pragma unroll
      for (int q = 0; q < 32; ++q) dot = fmaf(us[jj][q], vr[q], dot);
      const long long e = (j0 + jj) * d_in + c;
      const float v = r[e];
      const float nv = v >= 0.f ? v - dot : v + dot;
      r[e] = nv;
      acc += (double)nv * nv;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sumsq, acc);
}

// ---- small dense kernels (ell <= 64, one CTA of 1024 threads; G col-major [ell, ell]) ----
constexpr int kSmallMax = 64;

// Cholesky G = R^T R (R upper, col-major [ell, ell]) for CholeskyQR (A <- A R^-1 by a
// triangular solve).  Right-looking with every thread updating one trailing entry.  A pivot
// below 1e-12 of the largest diagonal entry marks a rank-deficient direction: that row of R is
// zero with R_jj = 1e30, so the column of A R^-1 becomes ~0 (e.g. for an all-zero |R|).
__global__ void __launch_bounds__(1024) chol_kernel(const float* __restrict__ g, int ell, float* __restrict__ rmat) {
  __shared__ float a[kSmallMax][kSmallMax + 1];
  __shared__ float dmax, rjj_s;
  __shared__ int ok_s;
  const int t = threadIdx.x;
  for (int e = t; e < ell * ell; e += blockDim.x) a[e % ell][e / ell] = g[e];
  __syncthreads();
  if (t == 0) {
    float m = 0.f;
    for (int i = 0; i < ell; ++i) m = fmaxf(m, a[i][i]);
    dmax = m;
  }
  __syncthreads();
  for (int j = 0; j < ell; ++j) {
    if (t == 0) {
      const float piv = a[j][j];
      ok_s = piv > 1e-12f * dmax && piv > 0.f;
      rjj_s = ok_s ? sqrtf(piv) : 1e30f;
    }
    __syncthreads();
    const bool ok = ok_s;
    const float rjj = rjj_s;
    if (t > j && t < ell) a[j][t] = ok ? a[j][t] / rjj : 0.f;   // row j of R (upper part)
    __syncthreads();
    if (t == 0) a[j][j] = rjj;
    const int w = ell - j - 1;
    for (int e = t; e < w * w; e += blockDim.x) {
      const int i = j + 1 + e / w, c = j + 1 + e % w;
      if (c >= i) a[i][c] -= a[j][i] * a[j][c];
    }
    __syncthreads();
  }
  for (int e = t; e < ell * ell; e += blockDim.x) {
    const int i = e % ell, c = e / ell;
    rmat[e] = c >= i ? a[i][c] : 0.f;
  }
}

// The same factorisation for ell <= 32 in one warp: lane l keeps column l of G in registers,
// R(j, i) is broadcast by shuffles (no shared memory, no block barriers).
__global__ void __launch_bounds__(32) chol_warp_kernel(const float* __restrict__ g, int ell, float* __restrict__ rmat) {
  const int l = threadIdx.x;
  float gc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) gc[i] = (i < ell && l < ell) ? g[l * ell + i] : 0.f;
  float dm = (l < ell) ? gc[0] : 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) if (i == l) dm = gc[i];                   // G(l, l)
  for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  const float tiny = 1e-12f * dm;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j < ell) {
      const float piv = __shfl_sync(0xffffffffu, gc[j], j);
      const bool ok = piv > tiny && piv > 0.f;
      const float rjj = ok ? sqrtf(piv) : 1e30f;
      const float rj = l > j ? (ok ? gc[j] / rjj : 0.f) : (l == j ? rjj : 0.f);   // R(j, l)
      if (l < ell) rmat[l * ell + j] = rj;
#pragma unroll
      for (int i = j + 1; i < 32; ++i) {
        const float rji = __shfl_sync(0xffffffffu, rj, i);             // R(j, i)
        if (l > j) gc[i] -= rji * rj;
      }
    }
  }
  // entries below the diagonal of R
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i > l && i < ell && l < ell) rmat[l * ell + i] = 0.f;
}

// Symmetric eigendecomposition G = W diag(lambda) W^T by parallel cyclic Jacobi (round-robin
// pairing: m/2 disjoint rotations per step, every thread one (rotation, index) update),
// eigenvalues sorted descending, sigma = sqrt(max(lambda, 0)) written to sig[ell] and W
// (col-major [ell, ell]) to w_out.  Odd ell is padded with a zero row / column.
__global__ void __launch_bounds__(1024) symeig_kernel(const float* __restrict__ g, int ell, float* __restrict__ sig,
                                                      float* __restrict__ w_out) {
  __shared__ float a[kSmallMax][kSmallMax + 1];
  __shared__ float v[kSmallMax][kSmallMax + 1];
  __shared__ float cs[kSmallMax / 2], sn[kSmallMax / 2];
  __shared__ int pp[kSmallMax / 2], qq[kSmallMax / 2];
  __shared__ int order[kSmallMax];
  __shared__ float red_off, red_dia;
  const int t = threadIdx.x;
  const int m = (ell + 1) & ~1;
  const int half = m / 2;
  for (int e = t; e < m * m; e += blockDim.x) {
    const int i = e % m, j = e / m;
    a[i][j] = (i < ell && j < ell) ? g[j * ell + i] : 0.f;
    v[i][j] = (i == j) ? 1.f : 0.f;
  }
  for (int sweep = 0; sweep < 15; ++sweep) {
    if (t == 0) { red_off = 0.f; red_dia = 0.f; }
    __syncthreads();
    float off = 0.f, dia = 0.f;
    for (int e = t; e < m * m; e += blockDim.x) {
      const int i = e % m, j = e / m;
      const float x = a[i][j] * a[i][j];
      if (i == j) dia += x; else off += x;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      dia += __shfl_xor_sync(0xffffffffu, dia, o);
    }
    if ((t & 31) == 0) { atomicAdd(&red_off, off); atomicAdd(&red_dia, dia); }
    __syncthreads();
    if (red_off <= 1e-13f * red_dia) break;
    for (int step = 0; step < m - 1; ++step) {
      if (t < half) {
        const int x = t == 0 ? 0 : 1 + (t - 1 + step) % (m - 1);
        const int y = 1 + (m - 2 - t + step) % (m - 1);
        const int p = min(x, y), q = max(x, y);
        pp[t] = p;
        qq[t] = q;
        const float apq = a[p][q];
        float c = 1.f, s_ = 0.f;
        if (fabsf(apq) > 1e-30f) {
          const float tau = (a[q][q] - a[p][p]) / (2.f * apq);
          const float tt = (tau >= 0.f ? 1.f : -1.f) / (fabsf(tau) + sqrtf(1.f + tau * tau));
          c = rsqrtf(1.f + tt * tt);
          s_ = tt * c;
        }
        cs[t] = c;
        sn[t] = s_;
      }
      __syncthreads();
      for (int e = t; e < half * m; e += blockDim.x) {     // rows p, q of a (a <- J^T a)
        const int r = e / m, col = e % m;
        const int p = pp[r], q = qq[r];
        const float ap = a[p][col], aq = a[q][col];
        a[p][col] = cs[r] * ap - sn[r] * aq;
        a[q][col] = sn[r] * ap + cs[r] * aq;
      }
      __syncthreads();
      for (int e = t; e < half * m; e += blockDim.x) {     // columns p, q of a and v (a <- a J)
        const int r = e / m, row = e % m;
        const int p = pp[r], q = qq[r];
        const float ap = a[row][p], aq = a[row][q];
        a[row][p] = cs[r] * ap - sn[r] * aq;
        a[row][q] = sn[r] * ap + cs[r] * aq;
        const float vp = v[row][p], vq = v[row][q];
        v[row][p] = cs[r] * vp - sn[r] * vq;
        v[row][q] = sn[r] * vp + cs[r] * vq;
      }
      __syncthreads();
    }
  }
  if (t == 0) {                                  // descending eigenvalues
    for (int i = 0; i < m; ++i) order[i] = i;
    for (int i = 1; i < m; ++i) {
      const int key = order[i];
      int j = i - 1;
      while (j >= 0 && a[order[j]][order[j]] < a[key][key]) { order[j + 1] = order[j]; --j; }
      order[j + 1] = key;
    }
  }
  __syncthreads();
  if (t < ell) sig[t] = sqrtf(fmaxf(a[order[t]][order[t]], 0.f));
  for (int e = t; e < ell * ell; e += blockDim.x) {
    const int i = e % ell, j = e / ell;
    w_out[e] = v[i][order[j]];
  }
}

// End of a block: sigma[:k] -> sigma_out + bi k (if any), then the block counter advances.
__global__ void block_done_kernel(const float* __restrict__ sig, float* __restrict__ sigma_out, int k, int* __restrict__ bi) {
  const int b = *bi;
  if (sigma_out && threadIdx.x < k) sigma_out[(long long)b * k + threadIdx.x] = sig[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) *bi = b + 1;
}

__global__ void sumsq_kernel(const float* __restrict__ r, long long total, double* __restrict__ sumsq) {
  double acc = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
    acc += (double)r[e] * r[e];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sumsq, acc);
}

}  // namespace bs
