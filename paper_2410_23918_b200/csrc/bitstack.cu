// Host side of the BitStack C ABI (include/bitstack.h): handle lifetime,
// validation, the device block store, and stream-ordered kernel launches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared (see build.py).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bitstack.h"
#include <cublas_v2.h>

#include "aux_kernels.cuh"
#include "compress.cuh"
#include "decode_mx.cuh"
#include "decode_tc.cuh"
#include "prefill.cuh"
#include "rgemv.cuh"
#include "wrestore.cuh"

struct bitstack_layer_s {
  int64_t d_out = 0, d_in = 0, row_begin = 0, row_end = 0, rows_local = 0;
  int rows_pad = 0, nq = 0, row_tiles = 0;
  int64_t d_in_pad = 0;
  int32_t k = 0, n_cap = 0, n_res = 0, n_act = 0;
  int32_t kh = 1;          // 16-rank halves per block (k > 16: 2, sharing the block's sign tile)
  cudaStream_t pf_side = nullptr;              // prefill: xprep runs here, concurrent with wtile
  cudaEvent_t pf_fork = nullptr, pf_join = nullptr;
  bitstack_dtype fdt = BITSTACK_BF16;
  int dev_fdt = 1;  // device factor storage: 0 f32, 1 bf16, 2 f16 (the user's 16-bit dtype, kept as is)
  int layout = 1;   // device sign layout: 0 = F16 (fp32 factors, fp16 MMA), 1 = F8 (e4m3 MMA)
  int device = 0;
  int sm_count = 148;
  bitstack_kernel kernel = BITSTACK_KERNEL_AUTO;
  uint4* signs = nullptr;
  void* u = nullptr;
  void* v = nullptr;
  float* inv_s = nullptr;
  float* zscale = nullptr;
  float* vmaxr = nullptr;  // [n_cap x kh][16] max_c |V'[c, r]| (prefill W' range bound)
  float* y_part = nullptr; // [max(2 sm_count, row_tiles)][kPartStride] split-K partial slots (<= 2 CTAs/SM)
  uint8_t* zq = nullptr;   // e4m3 path: Zq units of the current call (grown on demand)
  int64_t zq_bytes = 0;
  int* counters = nullptr; // [row_tiles]
  unsigned* xmax = nullptr; // fp16 paths: [batch] bits of max_c |x_bc / s_c| of the call (absmax_xs_kernel)
  int64_t xmax_cap = 0;
  int* pf_rowexp = nullptr; // prefill: W' row scale exponents [rows_pad]
  uint8_t* pf_w = nullptr; // prefill path: W' operand image (transient workspace, grown on demand)
  uint8_t* pf_x = nullptr; // prefill path: X' operand image
  int64_t pf_w_bytes = 0, pf_x_bytes = 0;
  CUtensorMap rg_tmu, rg_tmv;  // restore-and-multiply path: TMA maps of U' and V' (built once)
  bool rg_maps = false;
  uint8_t* rg_x = nullptr;     // restore-and-multiply path: X' unit images (grown on demand)
  uint8_t* rg_part = nullptr;  // restore-and-multiply path: per-CTA partial y slots
  int64_t rg_x_bytes = 0, rg_part_bytes = 0;
  uint8_t* stage_x = nullptr;  // host-buffer calls: device staging of x / y (grown on demand)
  uint8_t* stage_y = nullptr;
  int64_t stage_x_bytes = 0, stage_y_bytes = 0;
  int64_t bytes = 0;
  int64_t block_bytes = 0;
  cudaStream_t last_stream = nullptr;   // stream of the previous call (order_after_last)
  bool has_last = false;
  cudaEvent_t order_ev = nullptr;
};

namespace {

float* g_dbg_acc = nullptr;     // test hook (bitstack_debug_set), not part of the ABI
uint32_t* g_dbg_z = nullptr;
thread_local std::string g_err;
std::atomic<long long> g_launches{0};

struct Profiler {
  std::mutex mu;
  bool on = false;
  int cap = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  int used = 0;
} g_prof;

bitstack_status fail(bitstack_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? BITSTACK_E_OOM : BITSTACK_E_CUDA,     \
                  "%s failed: %s", #call, cudaGetErrorString(e_));                        \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int dsize(bitstack_dtype d) { return d == BITSTACK_F32 ? 4 : 2; }
bool valid_dtype(int d) { return d == BITSTACK_F32 || d == BITSTACK_BF16 || d == BITSTACK_F16; }

enum MemKind { kMemDevice, kMemPinned, kMemPageable };
MemKind mem_kind(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return kMemPageable;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return kMemDevice;
  return a.type == cudaMemoryTypeHost ? kMemPinned : kMemPageable;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// cudaFuncSetAttribute is per device context: apply `set` once per (call site, device).  Two
// threads racing here both apply the (idempotent) attributes, which is harmless.
template <typename F>
bitstack_status once_per_device(std::atomic<unsigned long long>& done, F&& set) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return BITSTACK_OK;
  const bitstack_status rs = set();
  if (rs) return rs;
  done.fetch_or(bit, std::memory_order_acq_rel);
  return BITSTACK_OK;
}


template <int NB, int NDIG>
bitstack_status launch_decode(const bs::DecodeParams& prm, int grid, cudaStream_t st) {
  using C = bs::DecodeCfg<NB, NDIG>;
  static std::atomic<unsigned long long> attr_done{0};
  bitstack_status attr_rs = once_per_device(attr_done, [&]() -> bitstack_status {
    CK(cudaFuncSetAttribute(bs::decode_tc_kernel<NB, NDIG>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    return BITSTACK_OK;
  });
  if (attr_rs) return attr_rs;
  bs::decode_tc_kernel<NB, NDIG><<<grid, bs::kDecodeThreads, C::kSmemBytes, st>>>(prm);
  count_launch();
  CK(cudaGetLastError());
  return BITSTACK_OK;
}

constexpr int64_t kPrefillMinBatch = 33;   // AUTO: restored-tile GEMM path from this batch on

// AUTO takes the restored-tile GEMM (fp16 operands, ~3e-4 relative error) above the
// restore-and-multiply path's 32 tokens, for shards of at least one full 128-row tile; tiny shards
// stay on the decode path (one tile of GEMM work is not worth the restore, and y over a handful of
// rows is where the fp16 operand rounding shows most).
bool prefill_auto(bitstack_layer L, int64_t batch) { return batch >= kPrefillMinBatch && L->rows_local >= 128; }

// AUTO takes the restore-and-multiply path (rgemv.cuh) for kRgMinBatch..32 tokens with 16-bit
// factors: there the e4m3 decode's tensor work (48 Zq columns per token) exceeds restoring W'
// inside the SM, and the prefill path's W' round trip and 128-token GEMM tiles are not paid back
// (measured crossovers on C2 and C5).
constexpr int64_t kRgMinBatch = 6;
enum MatmulPath { kPathDecode, kPathRgemv, kPathPrefill };
MatmulPath choose_path(bitstack_layer L, int64_t batch) {
  const bool fp16ok = L->dev_fdt != 0 && L->layout == 1;
  if (L->kernel == BITSTACK_KERNEL_PREFILL) return kPathPrefill;
  if (L->kernel == BITSTACK_KERNEL_RGEMV) return kPathRgemv;
  if (L->kernel != BITSTACK_KERNEL_AUTO || !fp16ok) return kPathDecode;
  // (shards of >= one 128-row tile: over a handful of rows the tf32 operand rounding shows most)
  if (batch >= kRgMinBatch && batch <= bs::kRgMaxBatch && L->rows_local >= 128) return kPathRgemv;
  if (prefill_auto(L, batch)) return kPathPrefill;
  return kPathDecode;
}

// A handle's workspaces (Zq units, split-K slots and counters, staging, prefill images) are
// reused by every call.  Calls on one stream are ordered by the stream; when a call arrives on a
// different stream than the handle's previous call, the new stream first waits for everything
// submitted to the old one (an event recorded now on the old stream), so calls on one handle never
// overlap.  Under CUDA-graph capture the capture order is the caller's to keep (an event recorded
// outside a capture cannot be waited on inside it).
bitstack_status order_after_last(bitstack_layer L, cudaStream_t st) {
  if (L->has_last && L->last_stream != st) {
    cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &a));
    CK(cudaStreamIsCapturing(L->last_stream, &b));
    if (a == cudaStreamCaptureStatusNone && b == cudaStreamCaptureStatusNone) {
      if (!L->order_ev) CK(cudaEventCreateWithFlags(&L->order_ev, cudaEventDisableTiming));
      CK(cudaEventRecord(L->order_ev, L->last_stream));
      CK(cudaStreamWaitEvent(st, L->order_ev, 0));
    }
  }
  L->last_stream = st;
  L->has_last = true;
  return BITSTACK_OK;
}

// Per-token max_c |x_bc / s_c| of a call into L->xmax (the power-of-two operand scales of the
// fp16 paths); the buffer grows with the largest batch seen.
bitstack_status launch_absmax(bitstack_layer L, const void* x, int xdt, int64_t batch, cudaStream_t st) {
  if (batch > L->xmax_cap) {
    CK(cudaStreamSynchronize(st));
    cudaFree(L->xmax);
    L->xmax = nullptr;
    const int64_t cap = std::max<int64_t>(batch, 64);
    CK(cudaMalloc((void**)&L->xmax, (size_t)cap * 4));
    L->bytes += (cap - L->xmax_cap) * 4;
    L->xmax_cap = cap;
  }
  const int grid = (int)std::min<int64_t>(batch, (int64_t)L->sm_count * 8);
  const bool vec = L->d_in % 8 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  bs::absmax_xs_kernel<<<grid, 256, 0, st>>>(x, xdt, L->d_in, L->inv_s, (int)batch, (int)L->d_in, L->xmax, vec);
  count_launch();
  CK(cudaGetLastError());
  return BITSTACK_OK;
}

// ------------------------------------------------------------------ MX e4m3 decode (decode_mx.cuh)
// Zq workspace for batch class NB: one unit per (block half, 128-column chunk) of the capacity.
template <int NB>
bitstack_status ensure_zq_mx(bitstack_layer L, cudaStream_t st) {
  const int64_t cap = (int64_t)L->n_cap * L->kh * L->nq * bs::MxCfg<NB>::kUnit;
  if (cap <= L->zq_bytes) return BITSTACK_OK;
  CK(cudaStreamSynchronize(st));
  cudaFree(L->zq);
  L->zq = nullptr;
  CK(cudaMalloc((void**)&L->zq, (size_t)cap));
  L->bytes += cap - L->zq_bytes;
  L->zq_bytes = cap;
  return BITSTACK_OK;
}

bs::ZqMxParams zq_mx_params(bitstack_layer L, const bs::DecodeParams& p) {
  bs::ZqMxParams zp;
  zp.v = p.v;
  zp.inv_s = p.inv_s;
  zp.x = p.x;
  zp.zq = L->zq;
  zp.x_stride = p.x_stride;
  zp.nq = p.nq;
  zp.d_in = p.d_in;
  zp.batch = p.batch;
  zp.x_dtype = p.x_dtype;
  zp.f_dtype = p.f_dtype;
  zp.kfuse = p.kfuse;
  return zp;
}

// Zq CTAs resident per SM (persistent grid = SMs x this), per batch class; the same on every
// device of one architecture (the library is built for sm_100a only).
template <int NB>
std::atomic<int>& zq_occ() {
  static std::atomic<int> occ{1};
  return occ;
}
template <int NB>
constexpr int zq_smem() { return 2 * bs::MxCfg<NB>::kUnit; }

template <int NB>
bitstack_status mx_attrs() {
  static std::atomic<unsigned long long> done{0};
  return once_per_device(done, [&]() -> bitstack_status {
    using C = bs::DecodeMxCfg<NB>;
    constexpr int zs = zq_smem<NB>();
    CK(cudaFuncSetAttribute(bs::zq_mx_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, zs));
    CK(cudaFuncSetAttribute(bs::zq_mx_grouped_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, zs));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bs::zq_mx_grouped_kernel<NB>, bs::zq_threads<NB>(), zs));
    zq_occ<NB>().store(occ > 0 ? occ : 1);
    CK(cudaFuncSetAttribute(bs::decode_mx_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    CK(cudaFuncSetAttribute(bs::decode_mx_grouped_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            C::kSmemBytes));
    return BITSTACK_OK;
  });
}

cudaLaunchConfig_t pdl_config(int grid, int threads, int smem, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// One zq_mx + one decode_mx (PDL) launch for one layer and one batch chunk of NB tokens.
template <int NB>
bitstack_status launch_decode_mx(bitstack_layer L, const bs::DecodeParams& prm_in, int grid, cudaStream_t st) {
  using C = bs::DecodeMxCfg<NB>;
  bitstack_status rs = mx_attrs<NB>();
  if (rs) return rs;
  rs = ensure_zq_mx<NB>(L, st);
  if (rs) return rs;
  const int64_t units = (int64_t)prm_in.n * prm_in.nq;
  const int zgrid = (int)std::min<int64_t>(units, (int64_t)L->sm_count * zq_occ<NB>().load());
  bs::zq_mx_kernel<NB><<<(unsigned)zgrid, bs::zq_threads<NB>(), zq_smem<NB>(), st>>>(zq_mx_params(L, prm_in), (int)units);
  count_launch();
  CK(cudaGetLastError());
  bs::DecodeParams prm = prm_in;
  prm.zq = L->zq;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = pdl_config(grid, C::kThreads, C::kSmemBytes, st, attr);
  CK(cudaLaunchKernelEx(&cfg, bs::decode_mx_kernel<NB>, prm));
  count_launch();
  return BITSTACK_OK;
}

int mx_occ(int nb) { return nb == 1 ? bs::MxGeom<1>::OCC : 1; }
int mx_rows(int nb) {
  switch (nb) {
    case 1: return bs::MxGeom<1>::R;
    case 2: return bs::MxGeom<2>::R;
    case 3: return bs::MxGeom<3>::R;
    default: return bs::MxGeom<4>::R;
  }
}

bitstack_status dispatch_mx(int nb, bitstack_layer L, const bs::DecodeParams& prm, int grid, cudaStream_t st) {
  switch (nb) {
    case 1: return launch_decode_mx<1>(L, prm, grid, st);
    case 2: return launch_decode_mx<2>(L, prm, grid, st);
    case 3: return launch_decode_mx<3>(L, prm, grid, st);
    case 4: return launch_decode_mx<4>(L, prm, grid, st);
    case 5: return launch_decode_mx<5>(L, prm, grid, st);
    case 6: return launch_decode_mx<6>(L, prm, grid, st);
    case 7: return launch_decode_mx<7>(L, prm, grid, st);
    case 8: return launch_decode_mx<8>(L, prm, grid, st);
    default: return fail(BITSTACK_E_INVALID_ARG, "internal: batch chunk %d", nb);
  }
}

bitstack_status record_prof(cudaStream_t st, bool begin, int* slot) {
  if (!g_prof.on) return BITSTACK_OK;
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (begin) {
    if (g_prof.used >= g_prof.cap) {
      *slot = -1;
      return BITSTACK_OK;
    }
    *slot = g_prof.used++;
    CK(cudaEventRecord(g_prof.ev[*slot].first, st));
  } else if (*slot >= 0) {
    CK(cudaEventRecord(g_prof.ev[*slot].second, st));
  }
  return BITSTACK_OK;
}

#ifndef BS_WTILE_G
#define BS_WTILE_G 2
#endif
constexpr int kWtileG = BS_WTILE_G;   // blocks per wtile MMA step (2: 2 CTAs/SM; 4: 1 CTA/SM)

// GEMM tile shape: BN tokens (256, or 128 for small batches) x 128 MH rows.  MH = 2 reuses each
// X' stage for two MMAs (higher operand reuse, one accumulator set); MH = 1 doubles the tile
// count (better wave fill on the persistent grid) and double-buffers the accumulators so the
// epilogue overlaps the next tile.  Measured (C3, B = 2048): up/gate [14336, 4096] MH=1 207 us
// vs MH=2 231 us; down [4096, 14336] MH=2 182 us vs MH=1 203 us -- modelled as rounds of
// ceil(tiles / SMs) x per-tile cost (MH=1 tiles cost ~0.56 of MH=2 tiles).
void prefill_shape(int64_t row_tiles, int64_t batch, int sms, int* bn, int* mh) {
  *bn = batch <= 128 ? 128 : 256;
  const int64_t nt = (batch + *bn - 1) / *bn;
  const int64_t t2 = (row_tiles + 1) / 2 * nt, t1 = row_tiles * nt;
  const double c2 = (double)((t2 + sms - 1) / sms) * 2.0, c1 = (double)((t1 + sms - 1) / sms) * 1.12;
  *mh = c1 < c2 ? 1 : 2;
}

bitstack_status grow(bitstack_layer L, uint8_t** buf, int64_t* have, int64_t need, cudaStream_t st) {
  if (need <= *have) return BITSTACK_OK;
  CK(cudaStreamSynchronize(st));
  cudaFree(*buf);
  *buf = nullptr;
  L->bytes -= *have;
  *have = 0;
  cudaError_t e = cudaMalloc((void**)buf, (size_t)need);
  if (e != cudaSuccess) return fail(BITSTACK_E_OOM, "prefill workspace (%lld bytes): %s", (long long)need, cudaGetErrorString(e));
  *have = need;
  L->bytes += need;
  return BITSTACK_OK;
}

bitstack_status launch_wrestore(bitstack_layer L, int kc, int rt_img, cudaStream_t st);

// Large-batch path (prefill.cuh): X' image, W' image, GEMM -- three launches on `st`.
template <int BN, int MH>
bitstack_status launch_prefill(bitstack_layer L, const void* x, int xdt, void* y, int ydt, int64_t batch,
                               cudaStream_t st) {
  using GC = bs::GemmCfg<BN, MH>;
  using WC = bs::WtileCfg<kWtileG>;
  static std::atomic<unsigned long long> attr_done{0};
  bitstack_status attr_rs = once_per_device(attr_done, [&]() -> bitstack_status {
    CK(cudaFuncSetAttribute(bs::prefill_gemm_kernel<BN, MH>, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::kSmemBytes));
    CK(cudaFuncSetAttribute(bs::wtile_kernel<kWtileG>, cudaFuncAttributeMaxDynamicSharedMemorySize, WC::kSmem(16) + 1024));
    CK(cudaFuncSetAttribute(bs::wtile_kernel<kWtileG>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    return BITSTACK_OK;
  });
  if (attr_rs) return attr_rs;
  const int kc = (int)(L->d_in_pad / bs::kPK);
  const int rt_img = (L->row_tiles + 1) / 2 * 2;
  const int nt = (int)((batch + BN - 1) / BN);
  bitstack_status rs = grow(L, &L->pf_w, &L->pf_w_bytes, (int64_t)rt_img * kc * bs::kImgTileA, st);
  if (rs) return rs;
  rs = grow(L, &L->pf_x, &L->pf_x_bytes, (int64_t)nt * kc * BN * bs::kPK * 2, st);
  if (rs) return rs;

  // xprep (X' image) and wtile (W' image) are independent: xprep runs on a side stream forked
  // from `st` (fork / join by events, capturable into CUDA graphs), the GEMM waits for both
  if (!L->pf_side) {
    CK(cudaStreamCreateWithFlags(&L->pf_side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&L->pf_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&L->pf_join, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(L->pf_fork, st));
  CK(cudaStreamWaitEvent(L->pf_side, L->pf_fork, 0));
  const long long pieces = (long long)nt * kc * BN * 8;
  const int xgrid = (int)std::min<long long>((pieces + 255) / 256, (long long)L->sm_count * 16);
  const bool xvec = L->d_in % 8 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  rs = launch_absmax(L, x, xdt, batch, L->pf_side);
  if (rs) return rs;
  bs::xprep_kernel<<<xgrid, 256, 0, L->pf_side>>>(x, xdt, L->d_in, L->inv_s, (int)batch, (int)L->d_in, kc, BN,
                                                  pieces, reinterpret_cast<uint4*>(L->pf_x), xvec, L->xmax);
  count_launch();
  CK(cudaGetLastError());
  CK(cudaEventRecord(L->pf_join, L->pf_side));

  // W' restore: the rgemv pipeline in W'-output mode (TMA operands, balanced ranges), or the
  // original wtile kernel (BS_PREFILL_WTILE=1, A/B)
  static const int wtile_env = [] { const char* e = getenv("BS_PREFILL_WTILE"); return e ? atoi(e) : 0; }();
  if (wtile_env && L->n_act * L->kh > 16)
    return fail(BITSTACK_E_UNSUPPORTED, "wtile restore supports n <= 16 active blocks (n <= 8 for k > 16)");
  if (!wtile_env) {
    rs = launch_wrestore(L, kc, rt_img, st);
    if (rs) return rs;
  } else {
  bs::WtileParams wp;
  wp.signs = L->signs;
  wp.u = reinterpret_cast<const uint16_t*>(L->u);
  wp.v = reinterpret_cast<const uint16_t*>(L->v);
  wp.vmaxr = L->vmaxr;
  wp.f16 = L->dev_fdt == 2 ? 1 : 0;
  wp.img = L->pf_w;
  wp.rowexp = L->pf_rowexp;
  wp.n = L->n_act * L->kh;
  wp.ksh = L->kh == 2 ? 1 : 0;
  wp.nq = L->nq;
  wp.rows_pad = L->rows_pad;
  wp.row_tiles = L->row_tiles;
  wp.kc = kc;
  wp.row_tiles_img = rt_img;
  // persistent: 512 / kTmemCols CTAs per SM (G = 2: two CTAs of 256 TMEM columns each)
  const int wgrid = (int)std::min<int64_t>((int64_t)rt_img * kc, (int64_t)L->sm_count * (512 / WC::kTmemCols));
  bs::wtile_kernel<kWtileG><<<wgrid, WC::kThreads, WC::kSmem(wp.n), st>>>(wp);
  count_launch();
  CK(cudaGetLastError());
  }
  CK(cudaStreamWaitEvent(st, L->pf_join, 0));

  bs::GemmParams gp;
  gp.a_img = L->pf_w;
  gp.b_img = L->pf_x;
  gp.y = y;
  gp.rowexp = L->pf_rowexp;
  gp.xmax = L->xmax;
  gp.y_dtype = ydt;
  gp.y_stride = L->rows_local;
  gp.batch = (int)batch;
  gp.rows_local = (int)L->rows_local;
  gp.row_tiles = L->row_tiles;
  gp.m2_count = (L->row_tiles + MH - 1) / MH;
  gp.nt_count = nt;
  gp.kc = kc;
  const int tiles = gp.m2_count * nt;
  int slot = -1;   // measurement hooks bracket the dominant kernel of the path: the GEMM
  bitstack_status ps = record_prof(st, true, &slot);
  if (ps) return ps;
  bs::prefill_gemm_kernel<BN, MH><<<std::min(tiles, L->sm_count), GC::kThreads, GC::kSmemBytes, st>>>(gp);
  count_launch();
  CK(cudaGetLastError());
  return record_prof(st, false, &slot);
}

// TMA maps of a [rows][16] 16-bit factor array: box 128 rows x 16, 32-byte swizzle (the UMMA
// K-major SW32 layout).  The encoder comes from the driver at run time (no libcuda link).
bitstack_status encode_factor_map(CUtensorMap* map, const void* base, int64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(BITSTACK_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {16, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {16, 128};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BITSTACK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BITSTACK_OK;
}

// Work partition of the rgemv kernel (rgemv.cuh): either each row tile split into `splits` unit
// ranges (whole row tiles per CTA), or one CTA per SM over a balanced contiguous range of the
// row_tiles x nq (row tile, unit) pairs, whichever has the shorter longest range (a range that
// spans row tiles costs about one unit more: a drain and a partial slot per segment); kmax =
// partial slots per CTA.  Also builds the TMA maps of U' and V' once per handle.
bitstack_status rg_setup(bitstack_layer L, int* grid, int* kmax, int* splits) {
  const int64_t W = (int64_t)L->row_tiles * L->nq;
  const int splits_r = (int)std::max<int64_t>(1, std::min<int64_t>(L->sm_count / std::max(1, L->row_tiles), L->nq));
  const int64_t span_r = (L->nq + splits_r - 1) / splits_r;
  const int grid_b = (int)std::min<int64_t>(W, L->sm_count);
  const int64_t span_b = (W + grid_b - 1) / grid_b + 1;
  static const int mode_env = [] { const char* e = getenv("BS_RG_MODE"); return e ? atoi(e) : 0; }();   // A/B override
  const bool balanced = mode_env == 2 || (mode_env != 1 && span_b < span_r);
  *grid = balanced ? grid_b : L->row_tiles * splits_r;
  *kmax = balanced ? (int)((span_b - 1 + L->nq - 1) / L->nq + 1) : 1;
  *splits = balanced ? 0 : splits_r;
  if (*kmax > 32) return fail(BITSTACK_E_UNSUPPORTED, "restore-and-multiply: too many row tiles per CTA");
  if (!L->rg_maps) {
    bitstack_status rs = encode_factor_map(&L->rg_tmu, L->u, (int64_t)L->n_cap * L->kh * L->rows_pad);
    if (rs) return rs;
    rs = encode_factor_map(&L->rg_tmv, L->v, (int64_t)L->n_cap * L->kh * L->d_in_pad);
    if (rs) return rs;
    L->rg_maps = true;
  }
  return BITSTACK_OK;
}

bs::RgParams rg_params(bitstack_layer L, int kmax, int splits) {
  bs::RgParams rp = {};
  rp.tmu = L->rg_tmu;
  rp.tmv = L->rg_tmv;
  rp.signs = L->signs;
  rp.u = reinterpret_cast<const uint16_t*>(L->u);
  rp.v = reinterpret_cast<const uint16_t*>(L->v);
  rp.counters = L->counters;
  rp.n = L->n_act * L->kh;
  rp.ksh = L->kh == 2 ? 1 : 0;
  rp.nq = L->nq;
  rp.rows_pad = L->rows_pad;
  rp.rows_local = (int)L->rows_local;
  rp.row_tiles = L->row_tiles;
  rp.kmax = kmax;
  rp.splits = splits;
  rp.f16 = L->dev_fdt == 2 ? 1 : 0;
  rp.trace = reinterpret_cast<long long*>(g_dbg_acc);
  return rp;
}

// Restore-and-multiply path (rgemv.cuh): X' images, then one kernel; 2 launches on `st`.
// Restore-and-multiply channel half 1 with register products (mma.sync) instead of TMEM reads:
// BS_RG_HYB=1 (opt-in; measured slower -- C5 at 8 tokens 631 -> 777 us)
static bool rg_hybrid() {
  static const int v = [] { const char* e = getenv("BS_RG_HYB"); return e ? atoi(e) : 0; }();
  return v != 0;
}

template <int BP>
bitstack_status launch_rgemv_bp(bitstack_layer L, const void* x, int xdt, void* y, int ydt, int64_t batch,
                                cudaStream_t st) {
  using C = bs::RgCfg<BP>;
  static std::atomic<unsigned long long> attr_done{0};
  bitstack_status rs = once_per_device(attr_done, [&]() -> bitstack_status {
    CK(cudaFuncSetAttribute(bs::rgemv_kernel<BP, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    CK(cudaFuncSetAttribute(bs::rgemv_kernel<BP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    return BITSTACK_OK;
  });
  if (rs) return rs;
  int grid = 0, kmax = 0, splits = 0;
  rs = rg_setup(L, &grid, &kmax, &splits);
  if (rs) return rs;
  rs = grow(L, &L->rg_x, &L->rg_x_bytes, (int64_t)L->nq * C::kXImg, st);
  if (rs) return rs;
  rs = grow(L, &L->rg_part, &L->rg_part_bytes, (int64_t)grid * kmax * BP * 128 * 4, st);
  if (rs) return rs;
  const long long pieces = (long long)L->nq * BP * 32;
  const int xgrid = (int)std::min<long long>((pieces + 255) / 256, (long long)L->sm_count * 8);
  bs::rg_xprep_kernel<<<xgrid, 256, 0, st>>>(x, xdt, L->d_in, L->inv_s, (int)batch, (int)L->d_in, L->nq, BP,
                                            reinterpret_cast<uint4*>(L->rg_x));
  count_launch();
  CK(cudaGetLastError());
  bs::RgParams rp = rg_params(L, kmax, splits);
  rp.ximg = L->rg_x;
  rp.part = reinterpret_cast<float*>(L->rg_part);
  rp.y = y;
  rp.y_stride = L->rows_local;
  rp.y_dtype = ydt;
  rp.batch = (int)batch;
  int slot = -1;   // measurement hooks bracket the dominant kernel
  bitstack_status ps = record_prof(st, true, &slot);
  if (ps) return ps;
  // programmatic dependent launch after rg_xprep (BS_RG_PDL=0: plain launch): the U' / V' / sign
  // stages stream in while the X' image is written; only the X' loads wait
  static const int pdl_env = [] { const char* e = getenv("BS_RG_PDL"); return e ? atoi(e) : 1; }();
  if (pdl_env) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = pdl_config(grid, bs::kRgWarps * 32, C::kSmem, st, attr);
    if (rg_hybrid()) CK(cudaLaunchKernelEx(&cfg, bs::rgemv_kernel<BP, false, true>, rp));
    else CK(cudaLaunchKernelEx(&cfg, bs::rgemv_kernel<BP, false, false>, rp));
  } else if (rg_hybrid()) {
    bs::rgemv_kernel<BP, false, true><<<grid, bs::kRgWarps * 32, C::kSmem, st>>>(rp);
  } else {
    bs::rgemv_kernel<BP, false, false><<<grid, bs::kRgWarps * 32, C::kSmem, st>>>(rp);
  }
  count_launch();
  CK(cudaGetLastError());
  return record_prof(st, false, &slot);
}

// The prefill's W' restore on the rgemv pipeline (W'-output mode): every (row tile, unit) of W'
// as the GEMM's scaled fp16 operand image, row scales into pf_rowexp.  Padding row tiles of the
// image (rt_img > row_tiles) are zeroed.
bitstack_status launch_wrestore(bitstack_layer L, int kc, int rt_img, cudaStream_t st) {
  using C = bs::RgCfg<16>;
  static std::atomic<unsigned long long> attr_done{0};
  bitstack_status rs = once_per_device(attr_done, [&]() -> bitstack_status {
    CK(cudaFuncSetAttribute(bs::rgemv_kernel<16, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    CK(cudaFuncSetAttribute(bs::rgemv_kernel<16, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    return BITSTACK_OK;
  });
  if (rs) return rs;
  int grid = 0, kmax = 0, splits = 0;
  rs = rg_setup(L, &grid, &kmax, &splits);
  if (rs) return rs;
  if (rt_img > L->row_tiles)
    CK(cudaMemsetAsync(L->pf_w + (int64_t)L->row_tiles * kc * bs::kImgTileA, 0,
                       (size_t)(rt_img - L->row_tiles) * kc * bs::kImgTileA, st));
  bs::RgParams rp = rg_params(L, kmax, splits);
  rp.wimg = L->pf_w;
  rp.rowexp = L->pf_rowexp;
  rp.vmaxr = L->vmaxr;
  rp.kc = kc;
  // default: tcgen05 products read back from TMEM (rgemv_kernel<16, true>); BS_WRESTORE_HMMA=1: the
  // products in registers (wrestore.cuh, mma.sync) -- measured slower (C3 up/gate restore 130 vs 106
  // us: ALU-issue bound at ~2 instructions per element and block), kept for A/B runs
  static const int hm_env = [] { const char* e = getenv("BS_WRESTORE_HMMA"); return e ? atoi(e) : 0; }();
  if (hm_env) {
    static std::atomic<unsigned long long> hm_done{0};
    rs = once_per_device(hm_done, [&]() -> bitstack_status {
      CK(cudaFuncSetAttribute(bs::wrestore_hmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs::kWrSmem));
      CK(cudaFuncSetAttribute(bs::wrestore_hmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs::kWrSmem));
      return BITSTACK_OK;
    });
    if (rs) return rs;
    const int hgrid = (int)std::min<int64_t>((int64_t)L->row_tiles * L->nq, (int64_t)L->sm_count * 2);
    if (rp.f16) bs::wrestore_hmma_kernel<false><<<hgrid, bs::kWrThreads, bs::kWrSmem, st>>>(rp);
    else bs::wrestore_hmma_kernel<true><<<hgrid, bs::kWrThreads, bs::kWrSmem, st>>>(rp);
    count_launch();
    CK(cudaGetLastError());
    return BITSTACK_OK;
  }
  if (rg_hybrid()) bs::rgemv_kernel<16, true, true><<<grid, bs::kRgWarps * 32, C::kSmem, st>>>(rp);
  else bs::rgemv_kernel<16, true, false><<<grid, bs::kRgWarps * 32, C::kSmem, st>>>(rp);
  count_launch();
  CK(cudaGetLastError());
  return BITSTACK_OK;
}

bitstack_status launch_rgemv(bitstack_layer L, const void* x, int xdt, void* y, int ydt, int64_t batch,
                             cudaStream_t st) {
  if (batch <= 16) return launch_rgemv_bp<16>(L, x, xdt, y, ydt, batch, st);
  return launch_rgemv_bp<32>(L, x, xdt, y, ydt, batch, st);
}

bitstack_status launch_prefill(bitstack_layer L, const void* x, int xdt, void* y, int ydt, int64_t batch,
                               cudaStream_t st) {
  int bn = 256, mh = 2;
  prefill_shape(L->row_tiles, batch, L->sm_count, &bn, &mh);
  static const int bn_env = [] { const char* e = getenv("BS_PREFILL_BN"); return e ? atoi(e) : 0; }();
  static const int mh_env = [] { const char* e = getenv("BS_PREFILL_MH"); return e ? atoi(e) : 0; }();
  if (bn_env) bn = bn_env;   // A/B overrides (scripts/exp_bn.sh)
  if (mh_env) mh = mh_env;
  if (mh == 1) {
    switch (bn) {
      case 128: return launch_prefill<128, 1>(L, x, xdt, y, ydt, batch, st);
      default: return launch_prefill<256, 1>(L, x, xdt, y, ydt, batch, st);
    }
  }
  switch (bn) {
    case 128: return launch_prefill<128, 2>(L, x, xdt, y, ydt, batch, st);
    case 192: return launch_prefill<192, 2>(L, x, xdt, y, ydt, batch, st);
    case 224: return launch_prefill<224, 2>(L, x, xdt, y, ydt, batch, st);
    default: return launch_prefill<256, 2>(L, x, xdt, y, ydt, batch, st);
  }
}

template <int NDIG>
bitstack_status dispatch_decode(int nb, const bs::DecodeParams& prm, int grid, cudaStream_t st) {
  switch (nb) {
    case 1: return launch_decode<1, NDIG>(prm, grid, st);
    case 2: return launch_decode<2, NDIG>(prm, grid, st);
    case 4: return launch_decode<4, NDIG>(prm, grid, st);
    case 8: return launch_decode<8, NDIG>(prm, grid, st);
    default:
      return fail(BITSTACK_E_INVALID_ARG, "internal: batch chunk %d", nb);
  }
}

int r_tiles_for(int nb, int ndig) {
  const int N = 16 * nb * ndig;
  return std::min(8, 256 / N);
}

// Kernel parameters of one batch chunk [b0, b0 + bc) of layer L on the tcgen05 decode paths.
bs::DecodeParams decode_params(bitstack_layer L, const void* x, int xdt, int xsz, void* y, int ydt, int ysz,
                                      int64_t b0, int bc, int n_groups, int cpg) {
  bs::DecodeParams prm;
  prm.signs = L->signs;
  prm.u = L->u;
  prm.v = L->v;
  prm.inv_s = L->inv_s;
  prm.x = reinterpret_cast<const uint8_t*>(x) + b0 * L->d_in * xsz;
  prm.y = reinterpret_cast<uint8_t*>(y) + b0 * L->rows_local * ysz;
  prm.y_part = L->y_part;
  prm.counters = L->counters;
  prm.x_stride = L->d_in;
  prm.y_stride = L->rows_local;
  prm.n = L->n_act * L->kh;               // 16-rank halves
  prm.ksh = L->kh == 2 ? 1 : 0;
  prm.nq = L->nq;
  prm.rows_pad = L->rows_pad;
  prm.rows_local = (int)L->rows_local;
  prm.d_in = (int)L->d_in;
  prm.d_in_pad = (int)L->d_in_pad;
  prm.row_tiles = L->row_tiles;
  prm.n_groups = n_groups;
  prm.ctas_per_group = cpg;
  prm.batch = bc;
  prm.x_dtype = xdt;
  prm.y_dtype = ydt;
  prm.f_dtype = L->dev_fdt;
  prm.one2 = 0x3C003C00u;
  prm.one = 1u;
  prm.xmax = L->xmax ? L->xmax + b0 : nullptr;
  prm.dbg_acc = g_dbg_acc;
  prm.dbg_z = g_dbg_z;
  prm.zq = nullptr;
  prm.kfuse = 0;
  return prm;
}

// One zq_mx_grouped + one decode_mx_grouped launch (PDL) for `count` layers sharing a batch
// chunk of NB tokens.  SMs are shared out in proportion to work: every layer starts at one CTA
// per row group, then CTAs go one row group's worth at a time to the layer with the most work
// per CTA while the total stays within one wave (one resident CTA per SM).
template <int NB>
bitstack_status launch_grouped_mx(const bitstack_layer* layers, int count, const void* const* xs, int xdt, int xsz,
                                  void* const* ys, int ydt, int ysz, int bc, cudaStream_t st) {
  using C = bs::DecodeMxCfg<NB>;
  constexpr int R = C::R;
  bitstack_status rs = mx_attrs<NB>();
  if (rs) return rs;
  int n_groups[bs::kMaxMxGroup], cpg[bs::kMaxMxGroup];
  int64_t units[bs::kMaxMxGroup];
  double work[bs::kMaxMxGroup];
  int total = 0;
  for (int i = 0; i < count; ++i) {
    bitstack_layer L = layers[i];
    n_groups[i] = (L->row_tiles + R - 1) / R;
    units[i] = (int64_t)L->n_act * L->kh * L->nq;
    work[i] = (double)units[i] * L->row_tiles;
    cpg[i] = 1;
    total += n_groups[i];
  }
  const int budget = layers[0]->sm_count * C::OCC;
  for (;;) {
    int best = -1;
    double best_w = 0.0;
    for (int i = 0; i < count; ++i) {
      if (cpg[i] >= units[i] || total + n_groups[i] > budget) continue;
      const double w = work[i] / ((double)n_groups[i] * cpg[i]);
      if (w > best_w) { best_w = w; best = i; }
    }
    if (best < 0) break;
    ++cpg[best];
    total += n_groups[best];
  }
  bs::ZqMxGroup zg;
  bs::DecodeMxGroup dg;
  zg.count = dg.count = count;
  zg.unit_start[0] = dg.cta_start[0] = 0;
  for (int i = 0; i < count; ++i) {
    bitstack_layer L = layers[i];
    rs = ensure_zq_mx<NB>(L, st);
    if (rs) return rs;
    bs::DecodeParams prm = decode_params(L, xs[i], xdt, xsz, ys[i], ydt, ysz, 0, bc, n_groups[i], cpg[i]);
    prm.zq = L->zq;
    zg.prm[i] = zq_mx_params(L, prm);
    dg.prm[i] = prm;
    zg.unit_start[i + 1] = zg.unit_start[i] + (int)units[i];
    dg.cta_start[i + 1] = dg.cta_start[i] + n_groups[i] * cpg[i];
  }
  for (int i = count; i < bs::kMaxMxGroup; ++i) zg.unit_start[i + 1] = dg.cta_start[i + 1] = 0;
  int slot = -1;
  bitstack_status ps = record_prof(st, true, &slot);
  if (ps) return ps;
  const int zgrid = std::min(zg.unit_start[count], layers[0]->sm_count * zq_occ<NB>().load());
  bs::zq_mx_grouped_kernel<NB><<<(unsigned)zgrid, bs::zq_threads<NB>(), zq_smem<NB>(), st>>>(zg);
  count_launch();
  CK(cudaGetLastError());
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = pdl_config(dg.cta_start[count], C::kThreads, C::kSmemBytes, st, attr);
  CK(cudaLaunchKernelEx(&cfg, bs::decode_mx_grouped_kernel<NB>, dg));
  count_launch();
  return record_prof(st, false, &slot);
}

bitstack_status dispatch_grouped_mx(int nb, const bitstack_layer* layers, int count, const void* const* xs, int xdt,
                                    int xsz, void* const* ys, int ydt, int ysz, cudaStream_t st) {
  switch (nb) {
    case 1: return launch_grouped_mx<1>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 2: return launch_grouped_mx<2>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 3: return launch_grouped_mx<3>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 4: return launch_grouped_mx<4>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 5: return launch_grouped_mx<5>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 6: return launch_grouped_mx<6>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 7: return launch_grouped_mx<7>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    case 8: return launch_grouped_mx<8>(layers, count, xs, xdt, xsz, ys, ydt, ysz, nb, st);
    default: return fail(BITSTACK_E_INVALID_ARG, "internal: batch chunk %d", nb);
  }
}

// Per-device cuBLAS handles (created on first use).
struct LinalgHandles {
  std::mutex mu;
  cublasHandle_t blas = nullptr;
  void* ws = nullptr;          // cuBLAS workspace (set explicitly: required under stream capture)
  uint8_t* arena = nullptr;    // compression scratch (Arena), grow-only
  int64_t arena_bytes = 0;
};
constexpr size_t kBlasWorkspace = 64ull << 20;
LinalgHandles g_linalg[64];

// Bump allocator over the per-device compression arena (grow-only, kept across calls: large
// cudaMalloc / cudaFree pairs per call made the call time erratic).  Run once with base ==
// nullptr to size it, then again over the arena.
struct Arena {
  uint8_t* base = nullptr;
  int64_t off = 0;
  template <typename T>
  void take(T** out, int64_t count) {
    *out = reinterpret_cast<T*>(base + off);
    off += (std::max<int64_t>(count, 1) * (int64_t)sizeof(T) + 255) / 256 * 256;
  }
};
}  // namespace

extern "C" {

const char* bitstack_last_error(void) { return g_err.c_str(); }

// Test hook (not declared in bitstack.h): device buffers that the decode kernel
// fills with CTA 0's first on-chip Z tile and raw TMEM accumulators.
BITSTACK_API void bitstack_debug_set(void* acc, void* z) {
  g_dbg_acc = reinterpret_cast<float*>(acc);
  g_dbg_z = reinterpret_cast<uint32_t*>(z);
}

int64_t bitstack_launch_count(void) { return g_launches.load(); }

int64_t bitstack_block_size_bits(int64_t m, int64_t n, int32_t k, int32_t factor_bits) {
  return m * n + (int64_t)factor_bits * k * (m + n);
}

bitstack_status bitstack_create(int64_t d_out, int64_t d_in, int32_t k, int32_t n_capacity,
                                bitstack_dtype factor_dtype, int64_t row_begin, int64_t row_end,
                                int32_t device, bitstack_layer* out) {
  if (!out) return fail(BITSTACK_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (d_out < 1 || d_in < 1) return fail(BITSTACK_E_INVALID_ARG, "dims must be positive");
  if (k < 1 || k > std::min<int64_t>(d_out, d_in) || k > 32)
    return fail(BITSTACK_E_INVALID_ARG, "k=%d outside [1, min(d_out, d_in, 32)]", k);
  if (n_capacity < 1) return fail(BITSTACK_E_INVALID_ARG, "n_capacity must be >= 1");
  if (!valid_dtype(factor_dtype)) return fail(BITSTACK_E_INVALID_ARG, "bad factor dtype");
  if (row_begin < 0 || row_end > d_out || row_begin >= row_end)
    return fail(BITSTACK_E_DIM_MISMATCH, "row range [%lld,%lld) outside [0,%lld)",
                (long long)row_begin, (long long)row_end, (long long)d_out);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(BITSTACK_E_INVALID_ARG, "bad device %d", device);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(BITSTACK_E_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                device, prop.major, prop.minor);
  DeviceGuard guard(device);

  auto* L = new bitstack_layer_s();
  L->d_out = d_out;
  L->d_in = d_in;
  L->row_begin = row_begin;
  L->row_end = row_end;
  L->rows_local = row_end - row_begin;
  L->rows_pad = (int)((L->rows_local + 127) / 128 * 128);
  L->row_tiles = L->rows_pad / 128;
  L->d_in_pad = (d_in + 127) / 128 * 128;
  L->nq = (int)(L->d_in_pad / 128);
  L->k = k;
  L->kh = k > 16 ? 2 : 1;
  L->n_cap = n_capacity;
  L->fdt = factor_dtype;
  L->dev_fdt = factor_dtype == BITSTACK_BF16 ? 1 : (factor_dtype == BITSTACK_F16 ? 2 : 0);
  L->layout = factor_dtype == BITSTACK_F32 ? 0 : 1;
  L->device = device;
  L->sm_count = prop.multiProcessorCount;

  const int64_t fs = L->dev_fdt ? 2 : 4;
  const int64_t sign_bytes = (int64_t)L->nq * L->rows_pad * 16;
  const int64_t u_bytes = (int64_t)L->rows_pad * 16 * fs;   // per 16-rank half
  const int64_t v_bytes = L->d_in_pad * 16 * fs;
  L->block_bytes = sign_bytes + L->kh * (u_bytes + v_bytes);
  auto alloc = [&](void** p, int64_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, (size_t)bytes);
    if (e == cudaSuccess) {
      L->bytes += bytes;
      e = cudaMemset(*p, 0, (size_t)bytes);
    }
    return e;
  };
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = alloc((void**)&L->signs, sign_bytes * n_capacity);
  if (e == cudaSuccess) e = alloc(&L->u, u_bytes * n_capacity * L->kh);
  if (e == cudaSuccess) e = alloc(&L->v, v_bytes * n_capacity * L->kh);
  if (e == cudaSuccess) e = alloc((void**)&L->inv_s, L->d_in_pad * 4);
  if (e == cudaSuccess) e = alloc((void**)&L->zscale, (int64_t)n_capacity * L->kh * 16 * 4);
  if (e == cudaSuccess) e = alloc((void**)&L->vmaxr, (int64_t)n_capacity * L->kh * 16 * 4);
  if (e == cudaSuccess) e = alloc((void**)&L->y_part, (int64_t)std::max(2 * L->sm_count, L->row_tiles) * bs::kPartStride * 4);
  if (e == cudaSuccess) e = alloc((void**)&L->counters, (int64_t)L->row_tiles * 4);
  if (e == cudaSuccess) e = alloc((void**)&L->pf_rowexp, (int64_t)L->rows_pad * 4);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    bitstack_destroy(L);
    return fail(e == cudaErrorMemoryAllocation ? BITSTACK_E_OOM : BITSTACK_E_CUDA,
                "bitstack_create: %s", cudaGetErrorString(e));
  }
  *out = L;
  return BITSTACK_OK;
}

bitstack_status bitstack_destroy(bitstack_layer L) {
  if (!L) return BITSTACK_OK;
  DeviceGuard guard(L->device);
  cudaDeviceSynchronize();
  cudaFree(L->signs);
  cudaFree(L->u);
  cudaFree(L->v);
  cudaFree(L->inv_s);
  cudaFree(L->zscale);
  cudaFree(L->vmaxr);
  if (L->pf_side) cudaStreamDestroy(L->pf_side);
  if (L->pf_fork) cudaEventDestroy(L->pf_fork);
  if (L->pf_join) cudaEventDestroy(L->pf_join);
  if (L->order_ev) cudaEventDestroy(L->order_ev);
  cudaFree(L->y_part);
  cudaFree(L->counters);
  cudaFree(L->xmax);
  cudaFree(L->pf_rowexp);
  cudaFree(L->zq);
  cudaFree(L->pf_w);
  cudaFree(L->pf_x);
  cudaFree(L->stage_x);
  cudaFree(L->stage_y);
  cudaFree(L->rg_x);
  cudaFree(L->rg_part);
  delete L;
  return BITSTACK_OK;
}

bitstack_status bitstack_get_info(bitstack_layer L, bitstack_info* out) {
  if (!L || !out) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  out->d_out = L->d_out;
  out->d_in = L->d_in;
  out->row_begin = L->row_begin;
  out->row_end = L->row_end;
  out->k = L->k;
  out->n_capacity = L->n_cap;
  out->n_resident = L->n_res;
  out->n_active = L->n_act;
  out->factor_dtype = L->fdt;
  out->device = L->device;
  out->device_bytes = L->bytes;
  out->block_bytes_device = L->block_bytes;
  return BITSTACK_OK;
}

bitstack_status bitstack_set_kernel(bitstack_layer L, bitstack_kernel kernel) {
  if (!L) return fail(BITSTACK_E_INVALID_ARG, "NULL layer");
  if (kernel != BITSTACK_KERNEL_AUTO && kernel != BITSTACK_KERNEL_TC && kernel != BITSTACK_KERNEL_SIMT &&
      kernel != BITSTACK_KERNEL_PREFILL && kernel != BITSTACK_KERNEL_RGEMV)
    return fail(BITSTACK_E_INVALID_ARG, "bad kernel selector %d", (int)kernel);
  L->kernel = kernel;
  return BITSTACK_OK;
}

bitstack_status bitstack_set_num_blocks(bitstack_layer L, int32_t n) {
  if (!L) return fail(BITSTACK_E_INVALID_ARG, "NULL layer");
  if (n < 0 || n > L->n_res)
    return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "n=%d outside [0, resident=%d]", n, L->n_res);
  L->n_act = n;
  return BITSTACK_OK;
}

// Validation shared by the two load entry points (before any device state changes).
// Argument checks of a block load.  Device-resident buffers are read back on `st` (ordered after
// whatever produced them there, e.g. bitstack_compress on a side stream), then `st` is synchronised
// for those few bytes.
static bitstack_status check_load_args(bitstack_layer L, int32_t first_block, int32_t count, const uint8_t* signs,
                                       const void* u, const void* v, const float* s, cudaStream_t st) {
  if (!L) return fail(BITSTACK_E_INVALID_ARG, "NULL layer");
  if (count < 0) return fail(BITSTACK_E_INVALID_ARG, "count < 0");
  if (first_block < 0 || first_block > L->n_res)
    return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "first_block=%d outside [0, resident=%d]",
                first_block, L->n_res);
  if ((int64_t)first_block + count > L->n_cap)
    return fail(BITSTACK_E_CAPACITY, "first_block+count=%d > capacity %d", first_block + count, L->n_cap);
  if (first_block == 0 && !s) return fail(BITSTACK_E_INVALID_ARG, "s is required when first_block == 0");
  if (first_block > 0 && s) return fail(BITSTACK_E_INVALID_ARG, "s must be NULL when first_block > 0");
  if (count > 0 && (!signs || !u || !v)) return fail(BITSTACK_E_INVALID_ARG, "NULL block buffer");
  DeviceGuard guard(L->device);
  const int64_t nbits = L->d_out * L->d_in;
  const int64_t cbytes = (nbits + 7) / 8;
  const int pad = (int)(cbytes * 8 - nbits);
  // pad-bit validation (SPEC S:203 MalformedBuffer): one byte per block
  if (count > 0 && pad) {
    const uint8_t mask = (uint8_t)(0xFFu << (8 - pad));
    const bool dev = is_device_ptr(signs);
    for (int b = 0; b < count; ++b) {
      uint8_t last = 0;
      if (dev) {
        CK(cudaMemcpyAsync(&last, signs + (int64_t)b * cbytes + cbytes - 1, 1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      } else {
        last = signs[(int64_t)b * cbytes + cbytes - 1];
      }
      if (last & mask) return fail(BITSTACK_E_MALFORMED_BUFFER, "block %d: non-zero pad bits", first_block + b);
    }
  }
  if (s) {
    std::vector<float> hs;
    const float* sp = s;
    if (is_device_ptr(s)) {
      hs.resize(L->d_in);
      CK(cudaMemcpyAsync(hs.data(), s, L->d_in * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      sp = hs.data();
    }
    for (int64_t c = 0; c < L->d_in; ++c)
      if (!(sp[c] > 0.f) || !std::isfinite(sp[c]))
        return fail(BITSTACK_E_INVALID_ARG, "s[%lld] = %g is not a positive finite scale", (long long)c, sp[c]);
  }
  return BITSTACK_OK;
}

// Per-device staging for block loads: two slots used alternately, each guarded by an event
// recorded after the kernels that read it, so a slot is refilled (on any stream) only after
// its previous contents were consumed.  Grow-only; growth waits for the slot's event.
struct StagePool {
  std::mutex mu;
  uint8_t* buf[2] = {nullptr, nullptr};
  int64_t bytes[2] = {0, 0};
  cudaEvent_t ev[2] = {nullptr, nullptr};      // slot's last reader (kernels) done
  cudaEvent_t copied[2] = {nullptr, nullptr};  // slot's copies done
  cudaEvent_t entry = nullptr;                 // the caller's stream at entry
  cudaStream_t copy = nullptr;                 // DMA stream: block b+1's copies overlap block b's kernels
  int next = 0;
};

// Lazily created per-device pool objects (under pool.mu); grows slot sl to `need` bytes.
static bitstack_status pool_slot(StagePool& pool, int sl, int64_t need) {
  if (!pool.copy) {
    CK(cudaStreamCreateWithFlags(&pool.copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&pool.entry, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&pool.ev[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&pool.copied[i], cudaEventDisableTiming));
    }
  }
  if (pool.bytes[sl] < need) {
    CK(cudaEventSynchronize(pool.ev[sl]));
    cudaFree(pool.buf[sl]);
    pool.buf[sl] = nullptr;
    pool.bytes[sl] = 0;
    CK(cudaMalloc((void**)&pool.buf[sl], (size_t)need));
    pool.bytes[sl] = need;
  }
  return BITSTACK_OK;
}
static StagePool g_stage[64];

// Enqueue the transfer + repack of blocks [first_block, first_block + count): per block, the
// canonical sign bytes of this handle's rows, its U rows and all of V are copied into a staging
// slot on the pool's DMA stream (cudaMemcpyAsync: asynchronous from pinned host or device
// memory; pageable host memory makes the copy synchronous), then `st` waits for the copy and
// repacks / rebalances from the slot.  Two slots: the copies of block b+1 overlap the kernels
// of block b.  The DMA stream first waits for `st` (the sources may be produced there).
static bitstack_status enqueue_blocks(bitstack_layer L, int32_t first_block, int32_t count, const uint8_t* signs,
                                      const void* u, const void* v, cudaStream_t st) {
  const int64_t nbits = L->d_out * L->d_in;
  const int64_t cbytes = (nbits + 7) / 8;
  const int fs = dsize(L->fdt);
  const bool rows_aligned = L->d_in % 8 == 0;     // every row starts on a byte: copy the shard only
  const int64_t sb0 = rows_aligned ? L->row_begin * (L->d_in / 8) : 0;
  const int64_t sbytes = rows_aligned ? L->rows_local * (L->d_in / 8) : cbytes;
  const int64_t ubytes = L->rows_local * L->k * fs;
  const int64_t vbytes = L->d_in * L->k * fs;
  auto up = [](int64_t x) { return (x + 255) / 256 * 256; };
  const int64_t need = up(sbytes) + up(ubytes) + up(vbytes) + 128;   // + vmax[32]
  const int64_t words_per_block = (int64_t)L->nq * L->rows_pad * 4;
  const int64_t fsd = L->dev_fdt ? 2 : 4;
  const int in_dt = L->fdt == BITSTACK_F32 ? 0 : (L->fdt == BITSTACK_BF16 ? 1 : 2);
  StagePool& pool = g_stage[L->device & 63];
  std::lock_guard<std::mutex> lk(pool.mu);
  bitstack_status rs = pool_slot(pool, 0, 0);
  if (rs) return rs;
  CK(cudaEventRecord(pool.entry, st));
  CK(cudaStreamWaitEvent(pool.copy, pool.entry, 0));
  for (int b = 0; b < count; ++b) {
    const int sl = pool.next;
    pool.next ^= 1;
    rs = pool_slot(pool, sl, need);
    if (rs) return rs;
    uint8_t* st_signs = pool.buf[sl];
    uint8_t* st_u = st_signs + up(sbytes);
    uint8_t* st_v = st_u + up(ubytes);
    unsigned int* vmax = reinterpret_cast<unsigned int*>(st_v + up(vbytes));
    const int64_t blk = first_block + b;
    CK(cudaStreamWaitEvent(pool.copy, pool.ev[sl], 0));          // slot's previous readers done
    CK(cudaMemcpyAsync(st_signs, signs + b * cbytes + sb0, (size_t)sbytes, cudaMemcpyDefault, pool.copy));
    CK(cudaMemcpyAsync(st_u, reinterpret_cast<const uint8_t*>(u) + (b * L->d_out + L->row_begin) * L->k * fs,
                       (size_t)ubytes, cudaMemcpyDefault, pool.copy));
    CK(cudaMemcpyAsync(st_v, reinterpret_cast<const uint8_t*>(v) + b * vbytes, (size_t)vbytes, cudaMemcpyDefault,
                       pool.copy));
    CK(cudaMemsetAsync(vmax, 0, 128, pool.copy));
    CK(cudaEventRecord(pool.copied[sl], pool.copy));
    CK(cudaStreamWaitEvent(st, pool.copied[sl], 0));
    uint32_t* dst = reinterpret_cast<uint32_t*>(L->signs) + blk * words_per_block;
    const int threads = 256;
    const int cap = L->sm_count * 8;
    if (rows_aligned) {
      const int64_t total = (int64_t)L->rows_pad * L->nq;
      const int grid = (int)std::min<int64_t>((total + threads - 1) / threads, cap);
      bs::repack_rows_kernel<<<grid, threads, 0, st>>>(st_signs, sbytes, reinterpret_cast<uint4*>(dst), 1, L->d_in,
                                                       L->nq, L->rows_pad, L->rows_local, L->layout);
    } else {
      const int grid = (int)std::min<int64_t>((words_per_block + threads - 1) / threads, 65536);
      bs::repack_signs_kernel<<<grid, threads, 0, st>>>(st_signs, dst, 1, cbytes, L->d_in, L->nq, L->rows_pad,
                                                        L->rows_local, L->row_begin, L->layout);
    }
    count_launch();
    CK(cudaGetLastError());
    // factors of rank half h (columns [16h, 16h + 16) of the stored [rows, k] U, V) -> internal
    // block blk * kh + h; one vmax[16] per half
    for (int h = 0; h < L->kh; ++h) {
      const int64_t vb = blk * L->kh + h;
      const int kc = std::min(16, L->k - 16 * h);
      uint8_t* u_dst = reinterpret_cast<uint8_t*>(L->u) + vb * L->rows_pad * 16 * fsd;
      uint8_t* v_dst = reinterpret_cast<uint8_t*>(L->v) + vb * L->d_in_pad * 16 * fsd;
      const int mgrid = (int)std::min<int64_t>((L->d_in + threads - 1) / threads, L->sm_count);
      bs::factor_max_kernel<<<mgrid, threads, 0, st>>>(st_v, in_dt, L->k, 16 * h, kc, L->d_in, vmax + 16 * h);
      count_launch();
      CK(cudaGetLastError());
      const int64_t elems = ((int64_t)L->rows_pad + L->d_in_pad) * 16;
      const int sgrid = (int)std::min<int64_t>((elems + threads - 1) / threads, cap);
      bs::factor_scale_kernel<<<sgrid, threads, 0, st>>>(st_u, st_v, in_dt, L->k, 16 * h, kc, L->rows_local,
                                                          L->rows_pad, L->d_in, L->d_in_pad, vmax + 16 * h, u_dst,
                                                          v_dst, L->dev_fdt, L->zscale + vb * 16, L->vmaxr + vb * 16);
      count_launch();
      CK(cudaGetLastError());
    }
    CK(cudaEventRecord(pool.ev[sl], st));
  }
  return BITSTACK_OK;
}

// 1/s into the handle (Eq.4), staged like the blocks (on `st` only: it is tiny).
static bitstack_status enqueue_scale(bitstack_layer L, const float* s, cudaStream_t st) {
  StagePool& pool = g_stage[L->device & 63];
  std::lock_guard<std::mutex> lk(pool.mu);
  const int sl = pool.next;
  pool.next ^= 1;
  bitstack_status rs = pool_slot(pool, sl, L->d_in * 4);
  if (rs) return rs;
  CK(cudaStreamWaitEvent(st, pool.ev[sl], 0));
  float* st_s = reinterpret_cast<float*>(pool.buf[sl]);
  CK(cudaMemcpyAsync(st_s, s, (size_t)(L->d_in * 4), cudaMemcpyDefault, st));
  bs::inv_s_kernel<<<(int)((L->d_in_pad + 255) / 256), 256, 0, st>>>(st_s, L->inv_s, L->d_in, L->d_in_pad);
  count_launch();
  CK(cudaGetLastError());
  CK(cudaEventRecord(pool.ev[sl], st));
  return BITSTACK_OK;
}

static bitstack_status load_blocks_impl(bitstack_layer L, int32_t first_block, int32_t count, const uint8_t* signs,
                                        const void* u, const void* v, const float* s, void* stream, bool wait) {
  DeviceGuard guard(L ? L->device : 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bitstack_status rs = check_load_args(L, first_block, count, signs, u, v, s, st);
  if (rs) return rs;
  rs = order_after_last(L, st);
  if (rs) return rs;
  if (count > 0) {
    rs = enqueue_blocks(L, first_block, count, signs, u, v, st);
    if (rs) return rs;
  }
  if (s) {
    rs = enqueue_scale(L, s, st);
    if (rs) return rs;
  }
  if (wait) CK(cudaStreamSynchronize(st));
  L->n_res = first_block + count;
  L->n_act = std::min(L->n_act, L->n_res);
  if (first_block == 0 && count > 0 && L->n_act == 0) L->n_act = L->n_res;
  return BITSTACK_OK;
}

bitstack_status bitstack_load_blocks(bitstack_layer L, int32_t first_block, int32_t count,
                                     const uint8_t* signs, const void* u, const void* v,
                                     const float* s, void* stream) {
  return load_blocks_impl(L, first_block, count, signs, u, v, s, stream, true);
}

bitstack_status bitstack_load_blocks_async(bitstack_layer L, int32_t first_block, int32_t count,
                                           const uint8_t* signs, const void* u, const void* v,
                                           const float* s, void* stream) {
  return load_blocks_impl(L, first_block, count, signs, u, v, s, stream, false);
}

// bitstack_matmul with device-accessible x / y (device memory, or pinned host memory read /
// written in place by the kernels); arguments already validated.
static bitstack_status matmul_device(bitstack_layer L, const void* x, bitstack_dtype x_dtype, void* y,
                                     bitstack_dtype y_dtype, int64_t batch, cudaStream_t st) {
  const int ysz = y_dtype == BITSTACK_F32 ? 4 : 2;
  if (L->n_act == 0) {
    CK(cudaMemsetAsync(y, 0, (size_t)(batch * L->rows_local * ysz), st));
    return BITSTACK_OK;
  }
  const int xdt = x_dtype == BITSTACK_F32 ? 0 : (x_dtype == BITSTACK_BF16 ? 1 : 2);
  const int ydt = y_dtype == BITSTACK_F32 ? 0 : 1;
  const int xsz = dsize(x_dtype);
  // small / large batches with 16-bit factors: restore-and-multiply or restored-tile GEMM
  // (forced with BITSTACK_KERNEL_RGEMV / BITSTACK_KERNEL_PREFILL)
  const MatmulPath path = choose_path(L, batch);
  const bool fp16ok = L->dev_fdt != 0 && L->layout == 1;
  if (path == kPathPrefill) {
    if (!fp16ok)
      return fail(BITSTACK_E_UNSUPPORTED, "prefill path needs bf16 / f16 factors");
    return launch_prefill(L, x, xdt, y, ydt, batch, st);
  }
  if (path == kPathRgemv) {
    if (!fp16ok || batch > bs::kRgMaxBatch)
      return fail(BITSTACK_E_UNSUPPORTED, "restore-and-multiply path needs bf16 / f16 factors and batch <= 32");
    return launch_rgemv(L, x, xdt, y, ydt, batch, st);
  }

  // tcgen05 path: k <= 16 (zero-padded columns of U', V'), x rows bulk-copied by the
  // TMA engine -> 16-byte aligned x and d_in % 8 == 0.
  const bool tc_ok = L->d_in % 8 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  const bool use_tc = L->kernel == BITSTACK_KERNEL_TC || (L->kernel == BITSTACK_KERNEL_AUTO && tc_ok);
  if (L->kernel == BITSTACK_KERNEL_TC && !tc_ok)
    return fail(BITSTACK_E_UNSUPPORTED, "tcgen05 decode kernel needs k <= 16, d_in %% 8 == 0 and a 16-byte aligned x");

  if (!use_tc) {
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int nb = (int)std::min<int64_t>(65535, batch - b0);
      int slot = -1;
      bitstack_status ps = record_prof(st, true, &slot);
      if (ps) return ps;
      dim3 grid(L->row_tiles, nb);
      bs::matmul_simt_kernel<<<grid, 128, 0, st>>>(
          L->signs, L->u, L->v, L->inv_s, reinterpret_cast<const uint8_t*>(x) + b0 * L->d_in * xsz,
          reinterpret_cast<uint8_t*>(y) + b0 * L->rows_local * ysz, L->n_act * L->kh, L->nq, L->rows_pad,
          L->rows_local, L->d_in, L->d_in_pad, L->dev_fdt, xdt, ydt, L->d_in, L->rows_local, L->layout,
          L->kh == 2 ? 1 : 0);
      count_launch();
      CK(cudaGetLastError());
      ps = record_prof(st, false, &slot);
      if (ps) return ps;
    }
    return BITSTACK_OK;
  }

  const bool f8 = L->layout == 1;          // MX e4m3 kernel (bf16/f16 factors); fp16 kernel for fp32 factors
  const int nbmax = 8;
  if (!f8) {   // fp16 digits: the call's x / s scale first
    bitstack_status rs = launch_absmax(L, x, xdt, batch, st);
    if (rs) return rs;
  }
  for (int64_t b0 = 0; b0 < batch; b0 += nbmax) {
    const int bc = (int)std::min<int64_t>(nbmax, batch - b0);
    int slot = -1;
    bitstack_status ps;
    if (f8) {
      // k > 16 with one token: both 16-rank halves of a block in ONE N = 96 contraction (the
      // batch-2 geometry, column group b = rank half b), so each sign tile is streamed once
      const bool kfuse = L->kh == 2 && bc == 1;
      const int nb = kfuse ? 2 : bc;
      const int R = mx_rows(nb);
      const int n_groups = (L->row_tiles + R - 1) / R;
      const int64_t units = (int64_t)L->n_act * (kfuse ? 1 : L->kh) * L->nq;
      int cpg = std::max(1, mx_occ(nb) * L->sm_count / n_groups);
      cpg = (int)std::min<int64_t>(cpg, units);
      bs::DecodeParams prm = decode_params(L, x, xdt, xsz, y, ydt, ysz, b0, bc, n_groups, cpg);
      if (kfuse) {
        prm.n = L->n_act;
        prm.ksh = 0;
        prm.kfuse = 1;
      }
      ps = record_prof(st, true, &slot);
      if (ps) return ps;
      bitstack_status rs = dispatch_mx(nb, L, prm, n_groups * cpg, st);
      if (rs) return rs;
    } else {
      int nb = 1;
      while (nb < bc) nb <<= 1;
      const int R = r_tiles_for(nb, 2);
      const int n_groups = (L->row_tiles + R - 1) / R;
      const int64_t units = (int64_t)L->n_act * L->kh * L->nq;
      int cpg = std::max(1, L->sm_count / n_groups);
      cpg = (int)std::min<int64_t>(cpg, units);
      const bs::DecodeParams prm = decode_params(L, x, xdt, xsz, y, ydt, ysz, b0, bc, n_groups, cpg);
      ps = record_prof(st, true, &slot);
      if (ps) return ps;
      bitstack_status rs = dispatch_decode<2>(nb, prm, n_groups * cpg, st);
      if (rs) return rs;
    }
    ps = record_prof(st, false, &slot);
    if (ps) return ps;
  }
  return BITSTACK_OK;
}

bitstack_status bitstack_matmul(bitstack_layer L, const void* x, bitstack_dtype x_dtype, void* y,
                                bitstack_dtype y_dtype, int64_t batch, void* stream) {
  if (!L) return fail(BITSTACK_E_INVALID_ARG, "NULL layer");
  if (batch < 0) return fail(BITSTACK_E_INVALID_ARG, "batch < 0");
  if (batch == 0) return BITSTACK_OK;
  if (!x || !y) return fail(BITSTACK_E_INVALID_ARG, "NULL x or y");
  if (!valid_dtype(x_dtype)) return fail(BITSTACK_E_INVALID_ARG, "bad x dtype");
  if (y_dtype != BITSTACK_F32 && y_dtype != BITSTACK_BF16)
    return fail(BITSTACK_E_INVALID_ARG, "y dtype must be F32 or BF16");
  if (L->n_res == 0 || L->n_act > L->n_res)
    return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "no resident blocks (load_blocks first)");
  DeviceGuard guard(L->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bitstack_status ors = order_after_last(L, st);
  if (ors) return ors;
  const int64_t xbytes = batch * L->d_in * dsize(x_dtype);
  const int64_t ybytes = batch * L->rows_local * (y_dtype == BITSTACK_F32 ? 4 : 2);
  const MemKind kx = mem_kind(x), ky = mem_kind(y);
  if (kx == kMemDevice && ky == kMemDevice) return matmul_device(L, x, x_dtype, y, y_dtype, batch, st);

  // Host buffers (the e2e path).  Small pinned buffers on the decode paths whose kernels read x
  // and write y with plain loads / stores (e4m3 decode, SIMT) are used in place: the transfer
  // is the kernels' own PCIe traffic.  Everything else is staged through device memory with
  // cudaMemcpyAsync on `stream` (synchronous with respect to pageable host memory).
  const bool pf = choose_path(L, batch) == kPathPrefill;
  const bool plain_io = !pf && (L->layout == 1 || L->kernel == BITSTACK_KERNEL_SIMT) && L->n_act > 0;
  const bool small = xbytes <= (1 << 20) && ybytes <= (1 << 20);
  const void* xd = x;
  void* yd = y;
  if (kx != kMemDevice) {
    if (kx == kMemPinned && plain_io && small) {
      void* dp = nullptr;
      CK(cudaHostGetDevicePointer(&dp, const_cast<void*>(x), 0));
      xd = dp;
    } else {
      bitstack_status rs = grow(L, &L->stage_x, &L->stage_x_bytes, xbytes, st);
      if (rs) return rs;
      CK(cudaMemcpyAsync(L->stage_x, x, (size_t)xbytes, cudaMemcpyHostToDevice, st));
      xd = L->stage_x;
    }
  }
  bool copy_back = false;
  if (ky != kMemDevice) {
    if (ky == kMemPinned && plain_io && small) {
      void* dp = nullptr;
      CK(cudaHostGetDevicePointer(&dp, y, 0));
      yd = dp;
    } else {
      bitstack_status rs = grow(L, &L->stage_y, &L->stage_y_bytes, ybytes, st);
      if (rs) return rs;
      yd = L->stage_y;
      copy_back = true;
    }
  }
  bitstack_status rs = matmul_device(L, xd, x_dtype, yd, y_dtype, batch, st);
  if (rs) return rs;
  if (copy_back) CK(cudaMemcpyAsync(y, L->stage_y, (size_t)ybytes, cudaMemcpyDeviceToHost, st));
  return BITSTACK_OK;
}

bitstack_status bitstack_matmul_grouped(const bitstack_layer* layers, int32_t count, const void* const* xs,
                                        bitstack_dtype x_dtype, void* const* ys, bitstack_dtype y_dtype,
                                        int64_t batch, void* stream) {
  if (count < 0 || (count > 0 && (!layers || !xs || !ys))) return fail(BITSTACK_E_INVALID_ARG, "bad group arrays");
  if (count == 0 || batch == 0) return BITSTACK_OK;
  // One launch pair when every member can take the e4m3 decode kernel on device buffers;
  // otherwise the members run one after another through bitstack_matmul (same results).
  bool fused = count <= bs::kMaxMxGroup && batch >= 1 && batch < kRgMinBatch &&
               valid_dtype(x_dtype) && (y_dtype == BITSTACK_F32 || y_dtype == BITSTACK_BF16);
  // members at level 0 (possible under any budget below one level, and common under the Random
  // and Greedy sortings) get y = 0 and stay out of the launches; the rest run fused
  bitstack_layer fl[bs::kMaxMxGroup];
  const void* fx[bs::kMaxMxGroup];
  void* fy[bs::kMaxMxGroup];
  int fc = 0, zero[bs::kMaxMxGroup], zc = 0;
  for (int i = 0; fused && i < count; ++i) {
    bitstack_layer L = layers[i];
    fused = L && xs[i] && ys[i] && L->device == layers[0]->device && mem_kind(ys[i]) == kMemDevice;
    for (int j = 0; fused && j < i; ++j) fused = layers[j] != L;   // each member owns its workspaces
    if (fused && L->n_act == 0) {
      zero[zc++] = i;
      continue;
    }
    fused = fused && L->layout == 1 && L->n_res > 0 && L->n_act <= L->n_res && L->d_in % 8 == 0 &&
            (L->kernel == BITSTACK_KERNEL_AUTO || L->kernel == BITSTACK_KERNEL_TC) &&
            (reinterpret_cast<uintptr_t>(xs[i]) % 16) == 0 && mem_kind(xs[i]) == kMemDevice;
    if (fused) {
      fl[fc] = L;
      fx[fc] = xs[i];
      fy[fc] = ys[i];
      ++fc;
    }
  }
  if (!fused) {
    for (int i = 0; i < count; ++i) {
      bitstack_status rs = bitstack_matmul(layers[i], xs[i], x_dtype, ys[i], y_dtype, batch, stream);
      if (rs) return rs;
    }
    return BITSTACK_OK;
  }
  DeviceGuard guard(layers[0]->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < fc; ++i) {
    bitstack_status ors = order_after_last(fl[i], st);
    if (ors) return ors;
  }
  const int xdt = x_dtype == BITSTACK_F32 ? 0 : (x_dtype == BITSTACK_BF16 ? 1 : 2);
  const int ydt = y_dtype == BITSTACK_F32 ? 0 : 1;
  const int xsz = dsize(x_dtype), ysz = y_dtype == BITSTACK_F32 ? 4 : 2;
  for (int z = 0; z < zc; ++z)
    CK(cudaMemsetAsync(ys[zero[z]], 0, (size_t)(batch * layers[zero[z]]->rows_local * ysz), st));
  // batch chunks of <= 8 tokens (the decode kernel's widest batch class), one launch pair each
  for (int64_t b0 = 0; fc > 0 && b0 < batch; b0 += 8) {
    const int bc = (int)std::min<int64_t>(8, batch - b0);
    const void* xc[bs::kMaxMxGroup];
    void* yc[bs::kMaxMxGroup];
    for (int i = 0; i < fc; ++i) {
      xc[i] = reinterpret_cast<const uint8_t*>(fx[i]) + b0 * fl[i]->d_in * xsz;
      yc[i] = reinterpret_cast<uint8_t*>(fy[i]) + b0 * fl[i]->rows_local * ysz;
    }
    bitstack_status rs = dispatch_grouped_mx(bc, fl, fc, xc, xdt, xsz, yc, ydt, ysz, st);
    if (rs) return rs;
  }
  return BITSTACK_OK;
}

bitstack_status bitstack_reconstruct(bitstack_layer L, void* w, bitstack_dtype w_dtype, void* stream) {
  if (!L || !w) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  if (!valid_dtype(w_dtype)) return fail(BITSTACK_E_INVALID_ARG, "bad w dtype");
  if (L->n_res == 0) return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "no resident blocks");
  DeviceGuard guard(L->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bitstack_status ors = order_after_last(L, st);
  if (ors) return ors;
  const int wdt = w_dtype == BITSTACK_F32 ? 0 : (w_dtype == BITSTACK_BF16 ? 1 : 2);
  dim3 grid((unsigned)((L->d_in + 31) / 32), (unsigned)((L->rows_local + 7) / 8));
  bs::reconstruct_kernel<<<grid, 256, 0, st>>>(L->signs, L->u, L->v, L->inv_s, w, L->n_act * L->kh, L->nq,
                                                L->rows_pad, L->rows_local, L->d_in, L->d_in_pad,
                                                L->dev_fdt, wdt, L->layout, L->kh == 2 ? 1 : 0);
  count_launch();
  CK(cudaGetLastError());
  return BITSTACK_OK;
}

// ---------------------------------------------------------------- GPU compression

#define CKB(call)                                                                         \
  do {                                                                                    \
    cublasStatus_t b_ = (call);                                                           \
    if (b_ != CUBLAS_STATUS_SUCCESS) return fail(BITSTACK_E_CUDA, "%s failed: cuBLAS status %d", #call, (int)b_); \
  } while (0)
bitstack_status bitstack_compress(const float* w, const float* x_cal, int64_t p, int64_t d_out, int64_t d_in,
                                  int32_t n, int32_t k, bitstack_dtype factor_dtype, int32_t oversample,
                                  int32_t power_iters, uint64_t seed, uint8_t* signs, void* u, void* v, float* s,
                                  float* sigma, float* resid, void* stream) {
  if (!w || !x_cal || !s || (n > 0 && (!signs || !u || !v))) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  if (d_out < 1 || d_in < 1 || p < 1 || n < 0 || oversample < 0 || power_iters < 0)
    return fail(BITSTACK_E_INVALID_ARG, "bad sizes");
  if (k < 1 || k > std::min<int64_t>(d_out, d_in) || k > 32)
    return fail(BITSTACK_E_INVALID_ARG, "k=%d outside [1, min(d_out, d_in, 32)]", k);
  if (!valid_dtype(factor_dtype)) return fail(BITSTACK_E_INVALID_ARG, "bad factor dtype");
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, w) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(BITSTACK_E_INVALID_ARG, "w must be device memory");
  }
  const void* outs[] = {x_cal, s, signs, u, v, sigma, resid};
  for (const void* q : outs)
    if (q && !is_device_ptr(q)) return fail(BITSTACK_E_INVALID_ARG, "all buffers must be device memory");
  DeviceGuard guard(pa.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LinalgHandles& H = g_linalg[pa.device & 63];
  std::lock_guard<std::mutex> lk(H.mu);
  if (!H.blas) CKB(cublasCreate(&H.blas));
  CKB(cublasSetStream(H.blas, st));
  CKB(cublasSetMathMode(H.blas, CUBLAS_DEFAULT_MATH));   // fp32 FFMA GEMMs (no TF32)

  const int ell = (int)std::min<int64_t>(k + oversample, std::min(d_out, d_in));
  if (ell > bs::kSmallMax) return fail(BITSTACK_E_INVALID_ARG, "k + oversample = %d > %d", ell, bs::kSmallMax);
  const int64_t total = d_out * d_in;
  const int fs = dsize(factor_dtype);
  const int out_dt = factor_dtype == BITSTACK_F32 ? 0 : (factor_dtype == BITSTACK_BF16 ? 1 : 2);
  float *R, *M, *Om, *Y, *Z, *G, *Rinv, *Wv, *Acol, *Bb, *sig, *uf, *vf;
  double *s2, *sumsq;
  unsigned long long* smax;
  int* bi = nullptr;               // device block counter of the block graph
  auto carve = [&](Arena& ar) {
    ar.take(&R, total);
    ar.take(&M, total);
    ar.take(&Om, d_in * ell);
    ar.take(&Y, d_out * ell);
    ar.take(&Z, d_in * ell);
    ar.take(&G, (int64_t)ell * ell);
    ar.take(&Rinv, (int64_t)ell * ell);
    ar.take(&Wv, (int64_t)ell * ell);
    ar.take(&Acol, d_out * k);
    ar.take(&Bb, d_in * k);
    ar.take(&sig, ell);
    ar.take(&uf, d_out * k);
    ar.take(&vf, d_in * k);
    ar.take(&s2, d_in);
    ar.take(&sumsq, n + 1);
    ar.take(&smax, 1);
    ar.take(&bi, 1);
  };
  {
    Arena sizing;
    carve(sizing);
    if (sizing.off > H.arena_bytes) {
      CK(cudaDeviceSynchronize());
      cudaFree(H.arena);
      H.arena = nullptr;
      H.arena_bytes = 0;
      CK(cudaMalloc((void**)&H.arena, (size_t)sizing.off));
      H.arena_bytes = sizing.off;
    }
    Arena ar;
    ar.base = H.arena;
    carve(ar);
  }
  // The ~100 launches per block (many of them tiny) are recorded once into a CUDA graph: issued
  // one by one, host launch overhead doubled the wall time of a 4096 x 4096 block.
  if (!H.ws) {
    CK(cudaMalloc(&H.ws, kBlasWorkspace));
    CKB(cublasSetWorkspace(H.blas, H.ws, kBlasWorkspace));
  }
  auto body = [&](cudaStream_t st, int part) -> bitstack_status {   // part 0: prologue, 1: one block
    const float one = 1.f, zero = 0.f;
    // CholeskyQR: A [m, ell] col-major <- an orthonormal basis of its range (G = A^T A,
    // G = R^T R, A <- A R^-1 by a triangular solve; rank-deficient directions become ~zero
    // columns).  One pass inside the power iteration (only the subspace matters there), two
    // (CholeskyQR2) for the final basis Q.
    auto qr = [&](float* A, int64_t m, int passes) -> bitstack_status {
      for (int pass = 0; pass < passes; ++pass) {
        CKB(cublasSgemm(H.blas, CUBLAS_OP_T, CUBLAS_OP_N, ell, ell, (int)m, &one, A, (int)m, A, (int)m, &zero, G, ell));
        if (ell <= 32) bs::chol_warp_kernel<<<1, 32, 0, st>>>(G, ell, Rinv);
        else bs::chol_kernel<<<1, 1024, 0, st>>>(G, ell, Rinv);
        count_launch();
        CK(cudaGetLastError());
        CKB(cublasStrsm(H.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)m, ell,
                        &one, Rinv, ell, A, (int)m));                                    // A <- A R^-1
      }
      return BITSTACK_OK;
    };
    const int T = 256;
    const int egrid = (int)std::min<int64_t>((total + T - 1) / T, 148 * 16);

    if (part == 0) {
    // Eq.3-4: s (fp64 sums of squares, clamped), R_0 = W diag(s)
    CK(cudaMemsetAsync(s2, 0, d_in * sizeof(double), st));
    CK(cudaMemsetAsync(smax, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(sumsq, 0, (n + 1) * sizeof(double), st));
    bs::colsq_kernel<<<dim3((unsigned)((d_in + T - 1) / T), (unsigned)std::min<int64_t>(p, 64)), T, 0, st>>>(x_cal, p, d_in, s2);
    bs::colmax_kernel<<<(int)std::min<int64_t>((d_in + T - 1) / T, 148), T, 0, st>>>(s2, d_in, smax);
    bs::scale_clamp_kernel<<<(int)((d_in + T - 1) / T), T, 0, st>>>(s2, smax, d_in, s);
    bs::scale_w_kernel<<<egrid, T, 0, st>>>(w, s, d_out, d_in, R);
    bs::sumsq_kernel<<<egrid, T, 0, st>>>(R, total, sumsq);
    for (int i = 0; i < 5; ++i) count_launch();
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(bi, 0, sizeof(int), st));
    return BITSTACK_OK;
    }

    {   // one block (block-indexed outputs through the device counter bi)
      // Eq.5: S_i = sign(R), M = |R|
      bs::sign_abs_kernel<<<egrid, T, 0, st>>>(R, total, signs, bi, M);
      bs::gauss_kernel<<<(int)((d_in * ell + T - 1) / T), T, 0, st>>>(Om, d_in * ell, seed, bi);
      count_launch();
      count_launch();
      CK(cudaGetLastError());
      // top-k SVD of M by randomized subspace iteration (row-major M = col-major M^T, ld d_in)
      CKB(cublasSgemm(H.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)d_out, ell, (int)d_in, &one, M, (int)d_in, Om, (int)d_in,
                      &zero, Y, (int)d_out));                                              // Y = M Om
      bitstack_status rs = qr(Y, d_out, power_iters > 0 ? 1 : 2);
      if (rs) return rs;
      for (int it = 0; it < power_iters; ++it) {
        CKB(cublasSgemm(H.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)d_in, ell, (int)d_out, &one, M, (int)d_in, Y,
                        (int)d_out, &zero, Z, (int)d_in));                                 // Z = M^T Q
        rs = qr(Z, d_in, 1);
        if (rs) return rs;
        CKB(cublasSgemm(H.blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)d_out, ell, (int)d_in, &one, M, (int)d_in, Z,
                        (int)d_in, &zero, Y, (int)d_out));                                 // Y = M Z
        rs = qr(Y, d_out, it + 1 == power_iters ? 2 : 1);
        if (rs) return rs;
      }
      CKB(cublasSgemm(H.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)d_in, ell, (int)d_out, &one, M, (int)d_in, Y, (int)d_out,
                      &zero, Z, (int)d_in));                                               // Bt = (Q^T M)^T
      // SVD of B = Q^T M through its Gram matrix: B B^T = Bt^T Bt = W diag(sigma^2) W^T; left
      // vectors a = Q W, right vectors B^T w / sigma = Bt W / sigma (factor_out divides)
      CKB(cublasSgemm(H.blas, CUBLAS_OP_T, CUBLAS_OP_N, ell, ell, (int)d_in, &one, Z, (int)d_in, Z, (int)d_in, &zero, G,
                      ell));
      bs::symeig_kernel<<<1, 1024, 0, st>>>(G, ell, sig, Wv);
      count_launch();
      CK(cudaGetLastError());
      CKB(cublasSgemm(H.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)d_out, k, ell, &one, Y, (int)d_out, Wv, ell, &zero, Acol,
                      (int)d_out));                                                        // a = Q W[:, :k]
      CKB(cublasSgemm(H.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)d_in, k, ell, &one, Z, (int)d_in, Wv, ell, &zero, Bb,
                      (int)d_in));                                                         // Bt W[:, :k]
      // Eq.2 split + sign convention + storage rounding; Eq.7 residual with the rounded factors
      bs::factor_out_kernel<<<k, T, 0, st>>>(Acol, d_out, Bb, d_in, sig, d_out, d_in, k, out_dt, u, v, bi, uf, vf);
      bs::residual_kernel<<<dim3((unsigned)((d_in + 255) / 256), (unsigned)((d_out + bs::kResRows - 1) / bs::kResRows)),
                            256, 0, st>>>(R, uf, vf, d_out, d_in, k, sumsq, bi);
      count_launch();
      count_launch();
      CK(cudaGetLastError());
      bs::block_done_kernel<<<1, 32, 0, st>>>(sig, sigma, k, bi);   // sigma out, ++bi
      count_launch();
      CK(cudaGetLastError());
    }
    return BITSTACK_OK;
  };
  // Two captured graphs: the prologue and one block's ~60 launches; the block graph is
  // replayed n times (host launch overhead of the many small kernels is paid once per call).
  cudaStream_t cap = nullptr;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  CKB(cublasSetStream(H.blas, cap));
  cudaGraph_t graphs[2] = {nullptr, nullptr};
  cudaGraphExec_t execs[2] = {nullptr, nullptr};
  bitstack_status rs0 = BITSTACK_OK;
  cudaError_t ce = cudaSuccess;
  int64_t block_launches = 0;        // our kernels in the block graph (counted once at capture)
  for (int g = 0; g < 2 && ce == cudaSuccess && rs0 == BITSTACK_OK; ++g) {
    ce = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) break;
    const int64_t l0 = g_launches.load();
    rs0 = body(cap, g);
    if (g == 1) block_launches = g_launches.load() - l0;
    const cudaError_t ee = cudaStreamEndCapture(cap, &graphs[g]);
    if (ce == cudaSuccess) ce = ee;
    if (ce == cudaSuccess && rs0 == BITSTACK_OK) ce = cudaGraphInstantiate(&execs[g], graphs[g], 0);
  }
  if (ce == cudaSuccess && rs0 == BITSTACK_OK) ce = cudaGraphLaunch(execs[0], st);
  for (int i = 0; i < n && ce == cudaSuccess && rs0 == BITSTACK_OK; ++i) ce = cudaGraphLaunch(execs[1], st);
  if (n > 1) g_launches.fetch_add((n - 1) * block_launches, std::memory_order_relaxed);   // the replays
  for (int g = 0; g < 2; ++g) {
    if (execs[g]) cudaGraphExecDestroy(execs[g]);
    if (graphs[g]) cudaGraphDestroy(graphs[g]);
  }
  cudaStreamDestroy(cap);
  cublasSetStream(H.blas, st);
  if (rs0) return rs0;
  if (ce != cudaSuccess) return fail(BITSTACK_E_CUDA, "compress graph: %s", cudaGetErrorString(ce));
  std::vector<double> hs(n + 1);
  CK(cudaMemcpyAsync(hs.data(), sumsq, (n + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (resid) {
    std::vector<float> hr(n + 1);
    for (int i = 0; i <= n; ++i) hr[i] = (float)std::sqrt(hs[i]);
    CK(cudaMemcpy(resid, hr.data(), (n + 1) * sizeof(float), cudaMemcpyHostToDevice));
  }
  return BITSTACK_OK;
}

bitstack_status bitstack_profile_begin(int32_t max_launches) {
  if (max_launches < 1) return fail(BITSTACK_E_INVALID_ARG, "max_launches < 1");
  std::lock_guard<std::mutex> lk(g_prof.mu);
  while ((int)g_prof.ev.size() < max_launches) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    g_prof.ev.emplace_back(a, b);
  }
  g_prof.cap = max_launches;
  g_prof.used = 0;
  g_prof.on = true;
  return BITSTACK_OK;
}

bitstack_status bitstack_profile_end(int32_t* launches, double* total_ms) {
  if (!launches || !total_ms) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = false;
  double tot = 0.0;
  for (int i = 0; i < g_prof.used; ++i) {
    CK(cudaEventSynchronize(g_prof.ev[i].second));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, g_prof.ev[i].first, g_prof.ev[i].second));
    tot += ms;
  }
  *launches = g_prof.used;
  *total_ms = tot;
  g_prof.used = 0;
  return BITSTACK_OK;
}

}  // extern "C"

#include "store.cuh"
