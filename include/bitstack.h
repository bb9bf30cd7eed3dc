/*
 * bitstack.h -- C ABI of the B200-native BitStack hot path (arXiv 2410.23918).
 *
 * One handle = one weight stack of one linear layer (optionally one row shard of
 * it for tensor parallelism).  The weight is held ONLY as n stacked residual
 * blocks, block i being a packed sign matrix S_i with rank-k magnitude factors
 * U_i [d_out,k] (paper's B'), V_i [d_in,k] (paper's A'):
 *
 *     W_iavd^(i) = S_i (.) (U_i V_i^T)                 PAPER.md Eq.7
 *     W_hat_n    = (sum_{i<n} W_iavd^(i)) diag(1/s)    Eq.8 + Eq.4
 *     y          = W_hat_n x
 *                = sum_i sum_r u_{i,r} (.) (S_i (v_{i,r} (.) (x / s)))   (north star)
 *
 * Orientation: [d_out, d_in], y = W x (reading R1; the paper writes
 * X W with W in R^{m x n}, m = input channels).  s indexes input channels.
 *
 * Conventions for every entry point
 *   - returns bitstack_status: 0 = OK, < 0 = error; bitstack_last_error() gives a
 *     thread-local message for the last non-OK status of the calling thread.
 *   - no exception or abort crosses the ABI.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - the library owns the device block store; the caller owns x, y, w.
 *   - calls on one handle never overlap: each handle reuses its workspaces (Zq
 *     units, split-K slots, staging), so a call arriving on a different stream
 *     than the handle's previous call first makes its stream wait for everything
 *     already submitted to the previous one (an event; no host blocking).  Under
 *     CUDA-graph capture that ordering is the caller's (capture one stream per
 *     handle).  Handles are not safe for concurrent mutation from host threads.
 *   - a CUDA fault inside an asynchronous kernel surfaces at a later call (or
 *     cudaStreamSynchronize) as BITSTACK_E_CUDA.
 */
#ifndef BITSTACK_H_
#define BITSTACK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BITSTACK_ABI_VERSION 1

#if defined(__GNUC__)
#define BITSTACK_API __attribute__((visibility("default")))
#else
#define BITSTACK_API
#endif

typedef struct bitstack_layer_s* bitstack_layer;

typedef enum {
  BITSTACK_F32 = 0,
  BITSTACK_BF16 = 1,
  BITSTACK_F16 = 2
} bitstack_dtype;

typedef enum {
  BITSTACK_OK = 0,
  BITSTACK_E_INVALID_ARG = -1,        /* null pointer, k<1, k>min(d_out,d_in), bad dtype */
  BITSTACK_E_DIM_MISMATCH = -2,       /* row range outside [0,d_out), empty shard */
  BITSTACK_E_LEVEL_OUT_OF_RANGE = -3, /* n > resident, first_block > resident */
  BITSTACK_E_MALFORMED_BUFFER = -4,   /* non-zero pad bits in a packed sign buffer */
  BITSTACK_E_CAPACITY = -5,           /* first_block + count > n_capacity */
  BITSTACK_E_OOM = -6,                /* device allocation failed */
  BITSTACK_E_CUDA = -7,               /* CUDA runtime error (message has the CUDA string) */
  BITSTACK_E_UNSUPPORTED = -8,        /* not an sm_100 device, a forced path that cannot run, ... */
  BITSTACK_E_IO = -9                  /* block store: file error, bad magic / version, corrupt or
                                         truncated record (SPEC S:465 BadMagic / CorruptRecord / ...) */
} bitstack_status;

/* Kernel selection for bitstack_matmul (bitstack_set_kernel). */
typedef enum {
  BITSTACK_KERNEL_AUTO = 0,   /* bf16 / f16 factors: 1-5 tokens the tcgen05 e4m3 decode kernel; with
                                 >= 128 local rows, 6-32 tokens the restore-and-multiply kernel and
                                 more the restored-tile GEMM (prefill), else the decode
                                 kernel; fp32 factors the tcgen05 fp16 decode kernel when supported,
                                 else SIMT */
  BITSTACK_KERNEL_TC = 1,     /* force the tcgen05/TMEM decode kernel (E_UNSUPPORTED if not possible) */
  BITSTACK_KERNEL_SIMT = 2,   /* force the CUDA-core FP32 reference kernel (any shape) */
  BITSTACK_KERNEL_PREFILL = 3,/* force the prefill path: W' = sum_i S_i (.) U_i V_i^T restored per
                                 128 x 128 unit on tcgen05 into an fp16 operand image, then Y = (X diag(1/s)) W'^T on tcgen05 with fp16
                                 operands (E_UNSUPPORTED unless bf16 / f16 factors) */
  BITSTACK_KERNEL_RGEMV = 4   /* force the restore-and-multiply path: W' restored per 128 x 128 unit
                                 inside the SM (tcgen05 U'V'^T + sign application), y += W' X'^T on
                                 tcgen05 in tf32; W' never reaches HBM (E_UNSUPPORTED unless bf16 /
                                 f16 factors and batch <= 32) */
} bitstack_kernel;

typedef struct {
  int64_t d_out, d_in, row_begin, row_end;
  int32_t k, n_capacity, n_resident, n_active;
  bitstack_dtype factor_dtype;
  int32_t device;
  int64_t device_bytes;          /* bytes of device memory owned by the handle */
  int64_t block_bytes_device;    /* device bytes per resident block (signs + factors, padded) */
} bitstack_info;

/* Create an empty weight stack for a [d_out, d_in] matrix, keeping rows
 * [row_begin, row_end) (row sharding); capacity n_capacity blocks,
 * rank k, factors stored as factor_dtype (Q7: the paper stores FP16).
 * Allocates all device memory up front on `device`.
 * k <= 16 is stored zero-padded to 16 ranks; 16 < k <= 32 (the paper's k ablation)
 * is stored as two 16-rank halves that share the block's sign tile (at batch 1 the e4m3 decode
 * contracts both halves in one pass over that tile; the other paths handle a half as a block).
 * Errors: E_INVALID_ARG (k<1, k>min(d_out,d_in), k>32, n_capacity<1, bad dtype, out==NULL),
 *         E_DIM_MISMATCH (bad row range), E_UNSUPPORTED (device not sm_100), E_OOM, E_CUDA. */
BITSTACK_API bitstack_status bitstack_create(int64_t d_out, int64_t d_in, int32_t k, int32_t n_capacity,
                                bitstack_dtype factor_dtype, int64_t row_begin, int64_t row_end,
                                int32_t device, bitstack_layer* out);

/* Free the handle and its device memory (waits for the device). NULL is a no-op. */
BITSTACK_API bitstack_status bitstack_destroy(bitstack_layer layer);

/* Push blocks [first_block, first_block+count) onto the stack -- "load more
 * weight residuals from storage when available memory increases" (Fig.2,
 * P:72).  first_block <= resident; afterwards resident = first_block + count
 * (re-pushing after an offload overwrites).  All buffers describe the FULL
 * matrix, in host or device memory (detected per pointer):
 *   signs : count x ceil(d_out*d_in/8) bytes, canonical packing (R11):
 *           bit j*d_in + c is S[j,c], LSB-first, 1 = +1, 0 = -1, pad bits 0
 *   u     : count x d_out x k   (factor_dtype, row-major)
 *   v     : count x d_in  x k   (factor_dtype, row-major)
 *   s     : d_in float32 > 0 (Eq.3 scaling vector); required iff first_block == 0,
 *           must be NULL otherwise.
 * The library copies its row shard and repacks signs into its device tile
 * layout (stream-ordered on `stream`); the call returns after the host-side
 * copies are done, so caller buffers are reusable on return.  active n is
 * clamped to the new resident count.
 * Errors: E_INVALID_ARG, E_CAPACITY, E_LEVEL_OUT_OF_RANGE (first_block > resident),
 *         E_MALFORMED_BUFFER (pad bits), E_CUDA. */
BITSTACK_API bitstack_status bitstack_load_blocks(bitstack_layer layer, int32_t first_block, int32_t count,
                                     const uint8_t* signs, const void* u, const void* v,
                                     const float* s, void* stream);

/* bitstack_load_blocks without the host synchronisation: block streaming, "load more weight
 * residuals from storage when available memory increases" (Fig.2) overlapped with
 * compute on other streams.  Same arguments, layouts, validation and errors.  Per block, the
 * canonical sign bytes of this handle's rows (only the shard when d_in % 8 == 0), its U rows
 * and V are copied with cudaMemcpyAsync into a per-device staging area (two slots, grown once
 * to the largest block seen; each slot is reused only after an event says its last reader
 * finished) on the library's copy stream, which first waits for `stream`; `stream` then waits
 * for each copy and repacks / rebalances on the device.  The call returns once this is
 * enqueued: from PINNED host memory or device memory the copies are asynchronous and the caller
 * must keep the buffers unchanged until `stream` passes this point (e.g. an event recorded
 * after the call); from pageable host memory cudaMemcpyAsync returns after the data is staged,
 * so the call is effectively synchronous.  The resident/active counts change immediately:
 * matmul calls enqueued later on `stream` see the new blocks; calls on other streams must wait
 * for an event recorded on `stream` after this call.  Not capturable into a CUDA graph.
 * bitstack_load_blocks is this call followed by a synchronisation of `stream`. */
BITSTACK_API bitstack_status bitstack_load_blocks_async(bitstack_layer layer, int32_t first_block, int32_t count,
                                           const uint8_t* signs, const void* u, const void* v,
                                           const float* s, void* stream);

/* Select how many resident blocks take part in matmul/reconstruct: 0 <= n <= resident.
 * Host-side O(1) ("dynamically load or offload"); affects calls enqueued
 * after it.  Blocks >= n stay resident until overwritten ("offload ... in
 * reverse order").  Errors: E_LEVEL_OUT_OF_RANGE, E_INVALID_ARG. */
BITSTACK_API bitstack_status bitstack_set_num_blocks(bitstack_layer layer, int32_t n);

/* y[b, :] = W_hat_n[row_begin:row_end, :] x[b, :]  for b < batch.
 *   x : [batch, d_in] row-major, dtype F32 | BF16 | F16
 *   y : [batch, row_end-row_begin] row-major, dtype F32 | BF16, overwritten
 * x and y may be device or host memory.  Small (<= 1 MiB) pinned host buffers are read /
 * written in place by the decode and restore-and-multiply kernels (their PCIe traffic is the
 * transfer); other host
 * buffers are staged through device memory with cudaMemcpyAsync on `stream` (pageable host
 * memory makes those copies synchronous).  Staging and path workspaces (Zq units, prefill and
 * restore-and-multiply images, TMA descriptors) are allocated on the first call that needs them
 * (which therefore must not be under CUDA-graph capture).
 * x and y must not alias.  batch == 0 is a no-op; n == 0 writes y = 0.
 * Asynchronous on `stream`; argument errors are reported synchronously.
 * Numerics, tensor-core paths, accumulation in fp32 throughout:
 *   - BF16/F16 factors, decode (batch <= 5, or any batch on < 128 local rows): S as exact e4m3 +-1, the product
 *     Z = V (.) (x/s) as three e4m3 digits per (rank, token) with power-of-two
 *     scales per 32-channel block (MX block scaling: digit 0 puts the block
 *     maximum in [128, 256), digit d is scaled 2^-4d further): error <= 2^-13 of
 *     the block maximum per element, whatever the range of x, s or the batch.
 *   - F32 factors: Z as two fp16 digits after a per-token power-of-two scale of
 *     x/s (~22 bits).
 *   - BF16/F16 factors, 6..32 tokens (restore-and-multiply): W' summed in fp32,
 *     W' and x/s rounded once to tf32 for the tcgen05 MMA (~1e-4 .. 4e-4).
 *   - BF16/F16 factors, batch > 32 (prefill): the restored tile W' = W diag(s)
 *     and x/s as fp16 GEMM operands, each with power-of-two scales (per row of W',
 *     per token of x/s) so that neither overflows nor underflows.
 *   Every scale is exact; non-finite x propagates to y.
 * Errors: E_INVALID_ARG, E_UNSUPPORTED (forced TC kernel not possible), E_CUDA. */
BITSTACK_API bitstack_status bitstack_matmul(bitstack_layer layer, const void* x, bitstack_dtype x_dtype,
                                void* y, bitstack_dtype y_dtype, int64_t batch, void* stream);

/* Several independent bitstack_matmul calls at one batch size, e.g. the q/k/v or gate/up
 * projections of a transformer layer that read the same token (Fig.2: every linear
 * layer of the model is a BitStack stack):  ys[i] = W_hat_{n_i}(layers[i]) xs[i], i < count.
 * Each member keeps its own level n_i, dtypes of x / y are shared, xs[i] / ys[i] follow
 * bitstack_matmul's layouts (xs[i] may be the same buffer for several members).
 * When count <= 8, 1 <= batch <= 5, the members are distinct handles on one device on the
 * MX e4m3 decode path (bf16/f16 factors, d_in % 8 == 0, AUTO or TC kernel) and all xs / ys are
 * 16-byte aligned device buffers, the whole group runs as ONE Zq launch and ONE decode launch,
 * whose CTAs are shared out among the members in proportion to their
 * work; members at level n_i == 0 get ys[i] = 0 (a memset) and no share of the launches (no
 * launch at all when every member is at level 0); otherwise the members run one after another through
 * bitstack_matmul (from 6 tokens that is the restore-and-multiply path of each member).  Results are
 * identical to the individual calls either way.  With profiling enabled the fused pair is
 * bracketed once.  count == 0 or batch == 0 is a no-op.
 * Errors: E_INVALID_ARG (NULL arrays) and every error of bitstack_matmul. */
BITSTACK_API bitstack_status bitstack_matmul_grouped(const bitstack_layer* layers, int32_t count,
                                        const void* const* xs, bitstack_dtype x_dtype, void* const* ys,
                                        bitstack_dtype y_dtype, int64_t batch, void* stream);

/* w = W_hat_n[row_begin:row_end, :] = sum_{i<n} (S_i (.) U_i V_i^T) diag(1/s)
 * (Eq.8 + Eq.4) written densely to device w [row_end-row_begin, d_in] row-major,
 * dtype F32 | BF16 | F16.  A test / export path ("restoration").
 * Errors: E_INVALID_ARG, E_CUDA. */
BITSTACK_API bitstack_status bitstack_reconstruct(bitstack_layer layer, void* w, bitstack_dtype w_dtype,
                                     void* stream);

/* Handle metadata and memory accounting.  Errors: E_INVALID_ARG. */
BITSTACK_API bitstack_status bitstack_get_info(bitstack_layer layer, bitstack_info* out);

/* Kernel selection for subsequent matmul calls.  Errors: E_INVALID_ARG. */
BITSTACK_API bitstack_status bitstack_set_kernel(bitstack_layer layer, bitstack_kernel kernel);

/* Eq.9: delta_W = m*n + factor_bits*k*(m+n) bits (factor_bits = 16 in
 * the paper).  Pure host arithmetic, never fails. */
BITSTACK_API int64_t bitstack_block_size_bits(int64_t m, int64_t n, int32_t k, int32_t factor_bits);

/* ---------------------------------------------------------------- block store (on disk)
 * Residual blocks as "basic transmission units" between storage and the device (PAPER.md
 * abstract P:8; Fig.2 P:64 "load more weight residuals from storage when available memory
 * increases"; SPEC S:446-497 store).  A store is a file of block records in the order they were
 * appended -- the caller's universal stack order (budget.py), so a memory-budget prefix is a
 * contiguous byte range -- with an offset index, so any record range is read without touching
 * the rest of the file.  Format v1 (little-endian, written once, no in-place mutation) in
 * csrc/store.cuh.  Host code only: usable without a GPU except bitstack_store_load_range.
 * A store handle is used by one host thread at a time. */
typedef struct bitstack_store_s* bitstack_store;

typedef struct {
  int32_t stack;                 /* caller's stack id (e.g. the weight matrix index) */
  int32_t block;                 /* block index i of that stack (Eq.8 order) */
  int64_t d_out, d_in;
  int32_t k;
  bitstack_dtype factor_dtype;
  int64_t size_bits;             /* declared Eq.9 size at the dtype's factor bits */
  int64_t sign_bytes, u_bytes, v_bytes, s_bytes;   /* payload parts; s only with block 0 */
  int64_t offset;                /* record byte offset in the file */
  uint32_t crc32;                /* CRC-32 (IEEE) of the payload */
} bitstack_store_record;

/* Create (truncate) a store file for writing.  Errors: E_INVALID_ARG, E_IO. */
BITSTACK_API bitstack_status bitstack_store_create(const char* path, bitstack_store* out);
/* Append one block record: the canonical layouts of bitstack_load_blocks for ONE block (host
 * buffers), s (d_in float32) given with block 0 and only there.
 * Errors: E_INVALID_ARG, E_MALFORMED_BUFFER (pad bits), E_IO. */
BITSTACK_API bitstack_status bitstack_store_append(bitstack_store store, int32_t stack, int32_t block,
                                                   int64_t d_out, int64_t d_in, int32_t k,
                                                   bitstack_dtype factor_dtype, const uint8_t* signs,
                                                   const void* u, const void* v, const float* s);
/* Open a store for reading (header + index only; record headers and payloads are read on demand).
 * Errors: E_INVALID_ARG, E_IO (cannot open, bad magic, version / endianness mismatch, truncated
 * or corrupt index). */
BITSTACK_API bitstack_status bitstack_store_open(const char* path, bitstack_store* out);
BITSTACK_API bitstack_status bitstack_store_count(bitstack_store store, int64_t* n_records);
/* Record metadata (reads its 64-byte header).  Errors: E_LEVEL_OUT_OF_RANGE, E_IO. */
BITSTACK_API bitstack_status bitstack_store_record_info(bitstack_store store, int64_t record,
                                                        bitstack_store_record* out);
/* Payload of one record into host buffers sized by record_info (NULL skips a part; the CRC is
 * checked when every part is read).  Errors: E_LEVEL_OUT_OF_RANGE, E_IO (truncated, CRC). */
BITSTACK_API bitstack_status bitstack_store_read(bitstack_store store, int64_t record, uint8_t* signs, void* u,
                                                 void* v, float* s);
/* Stream records [first_record, first_record + count) -- consecutive blocks of the stack the
 * layer holds -- from the file into the layer: each record is read into one of two pinned
 * buffers of the store (the read of record j+1 overlaps the DMA and repack of record j) and
 * pushed with bitstack_load_blocks_async at its block index (so the range must continue the
 * layer's resident prefix).  Returns once enqueued on `stream`.
 * Errors: E_LEVEL_OUT_OF_RANGE, E_DIM_MISMATCH (shape / rank / dtype), E_IO, and the errors of
 * bitstack_load_blocks. */
BITSTACK_API bitstack_status bitstack_store_load_range(bitstack_store store, bitstack_layer layer,
                                                       int64_t first_record, int64_t count, void* stream);
/* Writer: write the index and header, fsync.  Reader: release (waits for pending loads).
 * NULL is a no-op.  Errors: E_IO. */
BITSTACK_API bitstack_status bitstack_store_close(bitstack_store store);

/* Thread-local message of the last error on this thread ("" if none). */
BITSTACK_API const char* bitstack_last_error(void);

/* ---- GPU compression (Alg.1 P:423-445 for one weight matrix) ----
 * Produces the stored form that bitstack_load_blocks takes, on the device:
 *   s_c = ||x_cal[:, c]||_2 clamped at 1e-8 max_c s_c (Eq.3; reading R5),
 *   R_0 = W diag(s) (Eq.4), and for i < n (Eq.5-7):
 *     S_i = sign(R_i) with sign(0) = +1 (reading R6), packed canonically,
 *     |R_i| ~= a diag(sigma) b^T, the top-k singular triplets by seeded randomized subspace
 *       iteration (ell = min(k + oversample, d_out, d_in) columns, `power_iters` power
 *       iterations each re-orthonormalised by QR; reading of §8(c) "SVD method"),
 *     U_i = a sqrt(sigma), V_i = b sqrt(sigma) (Eq.2 balanced split), the largest-|entry| of
 *       each a_r made positive, rounded to factor_dtype (RNE),
 *     R_{i+1} = R_i - S_i (.) U_i V_i^T with the ROUNDED factors (reading R8).
 * All buffers are device memory on one device (E_INVALID_ARG otherwise):
 *   w      [d_out, d_in] f32 row-major         x_cal [p, d_in] f32 row-major (calibration X)
 *   signs  out [n][ceil(d_out d_in / 8)] u8    u out [n][d_out][k], v out [n][d_in][k] (factor_dtype)
 *   s      out [d_in] f32                      sigma out [n][k] f32 (may be NULL)
 *   resid  out [n + 1] f32 = ||R_0||_F .. ||R_n||_F (may be NULL)
 * 1 <= k <= min(d_out, d_in, 32), ell <= 64.  The skinny GEMMs with |R| and the tall-skinny
 * products run in cuBLAS (fp32 SGEMM, no TF32); the QR is CholeskyQR2 and the SVD of the
 * small projected matrix goes through its ell x ell Gram matrix (Jacobi eigensolver): those
 * ell x ell steps and the element-wise / reduction steps run in this library's kernels.
 * The Gaussian test matrix of block i is Philox(seed + 7919 i) (so factor values
 * differ from the CPU oracle's numpy generator; SVD outputs are compared by invariants).
 * Workspace ~2 d_out d_in x 4 bytes, allocated per call.  Returns after `stream` has
 * finished the work.  Errors: E_INVALID_ARG, E_OOM, E_CUDA. */
BITSTACK_API bitstack_status bitstack_compress(const float* w, const float* x_cal, int64_t p, int64_t d_out,
                                  int64_t d_in, int32_t n, int32_t k, bitstack_dtype factor_dtype,
                                  int32_t oversample, int32_t power_iters, uint64_t seed, uint8_t* signs,
                                  void* u, void* v, float* s, float* sigma, float* resid, void* stream);

/* ---- measurement hooks (used by bench.py; not part of the paper's problem) ----
 * While enabled, the dominant kernel launch of every bitstack_matmul call (decode:
 * the Zq + decode kernel pair; SIMT: its kernel; prefill: the GEMM) is bracketed
 * by a pair of CUDA events recorded on the launching stream.  profile_end
 * synchronises those events and returns the number of bracketed launches and the
 * sum of their device durations in milliseconds.  Errors: E_INVALID_ARG, E_CUDA. */
BITSTACK_API bitstack_status bitstack_profile_begin(int32_t max_launches);
BITSTACK_API bitstack_status bitstack_profile_end(int32_t* launches, double* total_ms);

/* Number of kernel launches issued by this library since process start
 * (monotonic counter; bench.py reports the difference as gpu_launches). */
BITSTACK_API int64_t bitstack_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* BITSTACK_H_ */
