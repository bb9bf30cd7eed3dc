/* Plain C use of the BitStack C ABI (include/bitstack.h): no Python, no torch.
 *
 *   gcc -O2 -I include examples/abi_demo.c -L paper_2410_23918_b200 -lbitstack \
 *       -Wl,-rpath,$PWD/paper_2410_23918_b200 -o abi_demo && ./abi_demo
 *
 * Builds one random 512 x 1024 weight stack of n = 4 residual blocks in host memory (canonical
 * packed signs, bf16 factors given as uint16 bit patterns, s = 1), pushes it with
 * bitstack_load_blocks, and evaluates y = W_hat_n x from HOST x / y buffers at every level n,
 * comparing with a straightforward host evaluation of the factored formula (Eq.8 + Eq.4).
 * Exit status 0 on agreement (relative L2 <= 1e-3), 1 on a mismatch, 2 on an ABI error.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bitstack.h"

enum { D_OUT = 512, D_IN = 1024, K = 16, N = 4, B = 2 };

static uint32_t rng_state = 12345u;
static float frand(void) {                       /* uniform in [-1, 1) */
  rng_state = rng_state * 1664525u + 1013904223u;
  return (float)((rng_state >> 8) & 0xFFFFFF) / 8388608.0f - 1.0f;
}
static uint16_t to_bf16(float f) {               /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  const size_t sbytes = ((size_t)D_OUT * D_IN + 7) / 8;
  uint8_t* signs = malloc(N * sbytes);
  uint16_t* u = malloc(sizeof(uint16_t) * N * D_OUT * K);
  uint16_t* v = malloc(sizeof(uint16_t) * N * D_IN * K);
  float* s = malloc(sizeof(float) * D_IN);
  float* x = malloc(sizeof(float) * B * D_IN);
  float* y = malloc(sizeof(float) * B * D_OUT);
  double* ref = malloc(sizeof(double) * B * D_OUT);
  for (size_t e = 0; e < N * sbytes; ++e) signs[e] = (uint8_t)(frand() * 128.0f + 128.0f);
  for (size_t e = 0; e < (size_t)N * D_OUT * K; ++e) u[e] = to_bf16(frand());
  for (size_t e = 0; e < (size_t)N * D_IN * K; ++e) v[e] = to_bf16(frand());
  for (int c = 0; c < D_IN; ++c) s[c] = 1.0f;
  for (int e = 0; e < B * D_IN; ++e) x[e] = frand();

  bitstack_layer layer = NULL;
  bitstack_status st = bitstack_create(D_OUT, D_IN, K, N, BITSTACK_BF16, 0, D_OUT, 0, &layer);
  if (st != BITSTACK_OK) {
    printf("bitstack_create: status %d (%s)\n", (int)st, bitstack_last_error());
    return 2;
  }
  st = bitstack_load_blocks(layer, 0, N, signs, u, v, s, NULL);
  if (st != BITSTACK_OK) {
    printf("bitstack_load_blocks: status %d (%s)\n", (int)st, bitstack_last_error());
    return 2;
  }
  int bad = 0;
  for (int n = 1; n <= N; ++n) {
    bitstack_set_num_blocks(layer, n);
    st = bitstack_matmul(layer, x, BITSTACK_F32, y, BITSTACK_F32, B, NULL);   /* host x / y */
    if (st != BITSTACK_OK) {
      printf("bitstack_matmul: status %d (%s)\n", (int)st, bitstack_last_error());
      return 2;
    }
    /* host reference: y[b, j] = sum_i sum_r U_i[j, r] sum_c S_i[j, c] V_i[c, r] x[b, c] / s_c */
    memset(ref, 0, sizeof(double) * B * D_OUT);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < D_OUT; ++j)
        for (int b = 0; b < B; ++b) {
          double t[K] = {0};
          for (int c = 0; c < D_IN; ++c) {
            const size_t bit = (size_t)j * D_IN + c;
            const double sg = ((signs[i * sbytes + bit / 8] >> (bit % 8)) & 1u) ? 1.0 : -1.0;
            const double xs = x[b * D_IN + c] / s[c];
            for (int r = 0; r < K; ++r) t[r] += sg * from_bf16(v[((size_t)i * D_IN + c) * K + r]) * xs;
          }
          for (int r = 0; r < K; ++r) ref[b * D_OUT + j] += from_bf16(u[((size_t)i * D_OUT + j) * K + r]) * t[r];
        }
    double num = 0.0, den = 0.0;
    for (int e = 0; e < B * D_OUT; ++e) {
      num += (y[e] - ref[e]) * (y[e] - ref[e]);
      den += ref[e] * ref[e];
    }
    const double rel = sqrt(num / den);
    printf("n=%d  relative L2 vs host reference = %.3e\n", n, rel);
    bad |= !(rel <= 1e-3);
  }
  bitstack_info info;
  bitstack_get_info(layer, &info);
  printf("device bytes held by the handle: %lld (%lld per block)\n", (long long)info.device_bytes,
         (long long)info.block_bytes_device);
  bitstack_destroy(layer);
  printf(bad ? "MISMATCH\n" : "OK\n");
  return bad;
}
