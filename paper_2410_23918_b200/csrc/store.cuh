// Block container on disk: BitStack's residual blocks as "basic transmission units" between
// storage and device memory (PAPER.md abstract P:8, Fig.2: "load more weight residuals
// from storage when available memory increases").  Host code of the C ABI
// (include/bitstack.h, bitstack_store_*), compiled into libbitstack.so with the kernels.
//
// Format v1 (little-endian; written once, read many times, no in-place mutation):
//   header  32 B   "BSTK" | u32 version 1 | u32 endian marker 0x01020304 | u32 0 |
//                  u64 n_records | u64 index_offset
//   record  64 B   "BREC" | u32 64 | i32 stack | i32 block | i64 d_out | i64 d_in | i32 k |
//                  i32 factor dtype | i64 declared size bits (Eq.9, factor bits of the
//                  dtype) | u64 payload bytes | u32 CRC-32 of the payload | u32 0
//           then   payload = canonical packed signs (ceil(d_out d_in / 8) B, R11) |
//                  U [d_out, k] | V [d_in, k] (factor dtype) | s [d_in] f32 (block 0 only)
//   index          n_records x u64 record offsets (at index_offset)
// Records are stored in the order they were appended -- the universal stack order of the
// caller (budget.py) -- so a memory-budget prefix of the stack is a contiguous byte range and
// any block range is read without touching the rest of the file (pread at indexed offsets).
#pragma once
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

struct bitstack_store_s {
  int fd = -1;
  bool writer = false;
  std::string path;
  std::vector<uint64_t> offsets;   // record offsets (reader: from the index; writer: as appended)
  uint64_t end = 0;                // writer: next record offset
  uint8_t* pin[2] = {nullptr, nullptr};   // load_range: pinned read buffers (ping-pong)
  int64_t pin_bytes[2] = {0, 0};
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  int device = -1;
};

namespace {

constexpr uint32_t kStoreVersion = 1;
constexpr uint32_t kEndianMarker = 0x01020304u;
constexpr int kHeaderBytes = 32, kRecordBytes = 64;

uint32_t crc32_update(uint32_t crc, const uint8_t* p, size_t n) {
  static uint32_t table[256];
  static bool init = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    return true;
  }();
  (void)init;
  crc = ~crc;
  for (size_t i = 0; i < n; ++i) crc = table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
  return ~crc;
}

template <typename T>
void put(std::vector<uint8_t>& b, T v) {
  const size_t o = b.size();
  b.resize(o + sizeof(T));
  std::memcpy(b.data() + o, &v, sizeof(T));
}
template <typename T>
T get(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

bool write_all(int fd, const void* p, size_t n, uint64_t off) {
  const uint8_t* c = static_cast<const uint8_t*>(p);
  while (n > 0) {
    const ssize_t w = pwrite(fd, c, n, (off_t)off);
    if (w <= 0) return false;
    c += w;
    n -= (size_t)w;
    off += (uint64_t)w;
  }
  return true;
}
bool read_all(int fd, void* p, size_t n, uint64_t off) {
  uint8_t* c = static_cast<uint8_t*>(p);
  while (n > 0) {
    const ssize_t r = pread(fd, c, n, (off_t)off);
    if (r <= 0) return false;
    c += r;
    n -= (size_t)r;
    off += (uint64_t)r;
  }
  return true;
}

struct RecordSizes {
  int64_t sign, u, v, s;
  int64_t total() const { return sign + u + v + s; }
};
RecordSizes record_sizes(int64_t d_out, int64_t d_in, int32_t k, int dtype, int32_t block) {
  const int fs = dtype == BITSTACK_F32 ? 4 : 2;
  return {(d_out * d_in + 7) / 8, d_out * k * fs, d_in * k * fs, block == 0 ? d_in * 4 : 0};
}

bitstack_status store_header(bitstack_store S, uint64_t n, uint64_t index_offset) {
  std::vector<uint8_t> h;
  h.insert(h.end(), {'B', 'S', 'T', 'K'});
  put<uint32_t>(h, kStoreVersion);
  put<uint32_t>(h, kEndianMarker);
  put<uint32_t>(h, 0);
  put<uint64_t>(h, n);
  put<uint64_t>(h, index_offset);
  if (!write_all(S->fd, h.data(), h.size(), 0)) return fail(BITSTACK_E_IO, "store %s: header write failed", S->path.c_str());
  return BITSTACK_OK;
}

// Reads and validates record r's 64-byte header.
bitstack_status store_record(bitstack_store S, int64_t r, bitstack_store_record* out) {
  if (r < 0 || r >= (int64_t)S->offsets.size())
    return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "record %lld outside [0, %zu)", (long long)r, S->offsets.size());
  uint8_t h[kRecordBytes];
  const uint64_t off = S->offsets[(size_t)r];
  if (!read_all(S->fd, h, sizeof(h), off))
    return fail(BITSTACK_E_IO, "store %s: record %lld truncated at offset %llu", S->path.c_str(), (long long)r,
                (unsigned long long)off);
  if (std::memcmp(h, "BREC", 4) != 0 || get<uint32_t>(h + 4) != kRecordBytes)
    return fail(BITSTACK_E_IO, "store %s: corrupt record %lld at offset %llu", S->path.c_str(), (long long)r,
                (unsigned long long)off);
  out->stack = get<int32_t>(h + 8);
  out->block = get<int32_t>(h + 12);
  out->d_out = get<int64_t>(h + 16);
  out->d_in = get<int64_t>(h + 24);
  out->k = get<int32_t>(h + 32);
  out->factor_dtype = (bitstack_dtype)get<int32_t>(h + 36);
  out->size_bits = get<int64_t>(h + 40);
  const uint64_t payload = get<uint64_t>(h + 48);
  out->crc32 = get<uint32_t>(h + 56);
  out->offset = (int64_t)off;
  if (out->d_out < 1 || out->d_in < 1 || out->k < 1 || out->k > 32 || out->block < 0 || !valid_dtype(out->factor_dtype))
    return fail(BITSTACK_E_IO, "store %s: corrupt record %lld header", S->path.c_str(), (long long)r);
  const RecordSizes rs = record_sizes(out->d_out, out->d_in, out->k, out->factor_dtype, out->block);
  if ((uint64_t)rs.total() != payload)
    return fail(BITSTACK_E_IO, "store %s: record %lld payload size mismatch", S->path.c_str(), (long long)r);
  out->sign_bytes = rs.sign;
  out->u_bytes = rs.u;
  out->v_bytes = rs.v;
  out->s_bytes = rs.s;
  return BITSTACK_OK;
}

// Payload of record r into caller buffers (any may be NULL to skip), CRC-checked when all parts
// are read.
bitstack_status store_payload(bitstack_store S, int64_t r, const bitstack_store_record& rec, uint8_t* signs,
                              void* u, void* v, float* s) {
  const uint64_t base = (uint64_t)rec.offset + kRecordBytes;
  uint8_t* parts[4] = {signs, static_cast<uint8_t*>(u), static_cast<uint8_t*>(v), reinterpret_cast<uint8_t*>(s)};
  const int64_t sizes[4] = {rec.sign_bytes, rec.u_bytes, rec.v_bytes, rec.s_bytes};
  uint64_t off = base;
  uint32_t crc = 0;
  bool all = true;
  for (int i = 0; i < 4; ++i) {
    if (sizes[i] > 0) {
      if (parts[i]) {
        if (!read_all(S->fd, parts[i], (size_t)sizes[i], off))
          return fail(BITSTACK_E_IO, "store %s: record %lld truncated", S->path.c_str(), (long long)r);
        crc = crc32_update(crc, parts[i], (size_t)sizes[i]);
      } else {
        all = false;
      }
    }
    off += (uint64_t)sizes[i];
  }
  if (all && crc != rec.crc32)
    return fail(BITSTACK_E_IO, "store %s: record %lld payload CRC mismatch", S->path.c_str(), (long long)r);
  return BITSTACK_OK;
}

}  // namespace

extern "C" {

bitstack_status bitstack_store_create(const char* path, bitstack_store* out) {
  if (!path || !out) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const int fd = open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return fail(BITSTACK_E_IO, "store %s: cannot create", path);
  auto* S = new bitstack_store_s();
  S->fd = fd;
  S->writer = true;
  S->path = path;
  S->end = kHeaderBytes;
  bitstack_status rs = store_header(S, 0, 0);
  if (rs) {
    close(fd);
    delete S;
    return rs;
  }
  *out = S;
  return BITSTACK_OK;
}

bitstack_status bitstack_store_append(bitstack_store S, int32_t stack, int32_t block, int64_t d_out, int64_t d_in,
                                      int32_t k, bitstack_dtype factor_dtype, const uint8_t* signs, const void* u,
                                      const void* v, const float* s) {
  if (!S || !S->writer) return fail(BITSTACK_E_INVALID_ARG, "not a store opened for writing");
  if (!signs || !u || !v) return fail(BITSTACK_E_INVALID_ARG, "NULL block buffer");
  if (d_out < 1 || d_in < 1 || k < 1 || k > 32 || k > std::min(d_out, d_in) || block < 0 || !valid_dtype(factor_dtype))
    return fail(BITSTACK_E_INVALID_ARG, "bad block shape / dtype");
  if ((block == 0) != (s != nullptr)) return fail(BITSTACK_E_INVALID_ARG, "s is stored with block 0 and only there");
  const RecordSizes rs = record_sizes(d_out, d_in, k, factor_dtype, block);
  const int pad = (int)(rs.sign * 8 - d_out * d_in);
  if (pad && (signs[rs.sign - 1] & (uint8_t)(0xFFu << (8 - pad))))
    return fail(BITSTACK_E_MALFORMED_BUFFER, "non-zero pad bits");
  const void* parts[4] = {signs, u, v, s};
  const int64_t sizes[4] = {rs.sign, rs.u, rs.v, rs.s};
  uint32_t crc = 0;
  for (int i = 0; i < 4; ++i)
    if (sizes[i]) crc = crc32_update(crc, static_cast<const uint8_t*>(parts[i]), (size_t)sizes[i]);
  std::vector<uint8_t> h;
  h.insert(h.end(), {'B', 'R', 'E', 'C'});
  put<uint32_t>(h, kRecordBytes);
  put<int32_t>(h, stack);
  put<int32_t>(h, block);
  put<int64_t>(h, d_out);
  put<int64_t>(h, d_in);
  put<int32_t>(h, k);
  put<int32_t>(h, (int32_t)factor_dtype);
  put<int64_t>(h, bitstack_block_size_bits(d_out, d_in, k, factor_dtype == BITSTACK_F32 ? 32 : 16));
  put<uint64_t>(h, (uint64_t)rs.total());
  put<uint32_t>(h, crc);
  put<uint32_t>(h, 0);
  uint64_t off = S->end;
  if (!write_all(S->fd, h.data(), h.size(), off)) return fail(BITSTACK_E_IO, "store %s: write failed", S->path.c_str());
  off += h.size();
  for (int i = 0; i < 4; ++i) {
    if (!sizes[i]) continue;
    if (!write_all(S->fd, parts[i], (size_t)sizes[i], off)) return fail(BITSTACK_E_IO, "store %s: write failed", S->path.c_str());
    off += (uint64_t)sizes[i];
  }
  S->offsets.push_back(S->end);
  S->end = off;
  return BITSTACK_OK;
}

bitstack_status bitstack_store_open(const char* path, bitstack_store* out) {
  if (!path || !out) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(BITSTACK_E_IO, "store %s: cannot open", path);
  auto* S = new bitstack_store_s();
  S->fd = fd;
  S->path = path;
  auto bad = [&](const char* why) {
    close(fd);
    delete S;
    return fail(BITSTACK_E_IO, "store %s: %s", path, why);
  };
  struct stat sb;
  if (fstat(fd, &sb) != 0) return bad("stat failed");
  uint8_t h[kHeaderBytes];
  if (!read_all(fd, h, sizeof(h), 0)) return bad("truncated header");
  if (std::memcmp(h, "BSTK", 4) != 0) return bad("bad magic");
  if (get<uint32_t>(h + 4) != kStoreVersion) return bad("format version mismatch");
  if (get<uint32_t>(h + 8) != kEndianMarker) return bad("endianness mismatch");
  const uint64_t n = get<uint64_t>(h + 16), idx = get<uint64_t>(h + 24);
  if (n == 0 && idx == 0) {   // header-only (an empty store, or a writer that never closed)
    *out = S;
    return BITSTACK_OK;
  }
  if (idx < kHeaderBytes || n > (uint64_t)sb.st_size / 8 || idx + n * 8 > (uint64_t)sb.st_size)
    return bad("truncated or corrupt index");
  S->offsets.resize(n);
  if (n && !read_all(fd, S->offsets.data(), n * 8, idx)) return bad("truncated index");
  for (uint64_t o : S->offsets)
    if (o < kHeaderBytes || o + kRecordBytes > idx) return bad("corrupt index offset");
  *out = S;
  return BITSTACK_OK;
}

bitstack_status bitstack_store_count(bitstack_store S, int64_t* n_records) {
  if (!S || !n_records) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  *n_records = (int64_t)S->offsets.size();
  return BITSTACK_OK;
}

bitstack_status bitstack_store_record_info(bitstack_store S, int64_t record, bitstack_store_record* out) {
  if (!S || !out) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  if (S->writer) return fail(BITSTACK_E_INVALID_ARG, "store is open for writing");
  return store_record(S, record, out);
}

bitstack_status bitstack_store_read(bitstack_store S, int64_t record, uint8_t* signs, void* u, void* v, float* s) {
  if (!S) return fail(BITSTACK_E_INVALID_ARG, "NULL store");
  if (S->writer) return fail(BITSTACK_E_INVALID_ARG, "store is open for writing");
  bitstack_store_record rec;
  bitstack_status rs = store_record(S, record, &rec);
  if (rs) return rs;
  return store_payload(S, record, rec, signs, u, v, s);
}

bitstack_status bitstack_store_load_range(bitstack_store S, bitstack_layer L, int64_t first_record, int64_t count,
                                          void* stream) {
  if (!S || !L) return fail(BITSTACK_E_INVALID_ARG, "NULL argument");
  if (S->writer) return fail(BITSTACK_E_INVALID_ARG, "store is open for writing");
  if (count < 0 || first_record < 0 || first_record + count > (int64_t)S->offsets.size())
    return fail(BITSTACK_E_LEVEL_OUT_OF_RANGE, "record range [%lld, %lld) outside [0, %zu)", (long long)first_record,
                (long long)(first_record + count), S->offsets.size());
  DeviceGuard guard(L->device);
  if (S->device >= 0 && S->device != L->device) {   // pinned buffers / events belong to one device
    for (int i = 0; i < 2; ++i) {
      if (S->pin_ev[i]) { cudaEventSynchronize(S->pin_ev[i]); cudaEventDestroy(S->pin_ev[i]); S->pin_ev[i] = nullptr; }
      cudaFreeHost(S->pin[i]);
      S->pin[i] = nullptr;
      S->pin_bytes[i] = 0;
    }
  }
  S->device = L->device;
  for (int64_t j = 0; j < count; ++j) {
    bitstack_store_record rec;
    bitstack_status rs = store_record(S, first_record + j, &rec);
    if (rs) return rs;
    if (rec.d_out != L->d_out || rec.d_in != L->d_in || rec.k != L->k || rec.factor_dtype != L->fdt)
      return fail(BITSTACK_E_DIM_MISMATCH, "record %lld does not match the layer's shape / rank / dtype",
                  (long long)(first_record + j));
    const int sl = (int)(j & 1);
    if (!S->pin_ev[sl]) CK(cudaEventCreateWithFlags(&S->pin_ev[sl], cudaEventDisableTiming));
    CK(cudaEventSynchronize(S->pin_ev[sl]));        // the buffer's previous load has been consumed
    const int64_t need = rec.sign_bytes + rec.u_bytes + rec.v_bytes + rec.s_bytes;
    if (S->pin_bytes[sl] < need) {
      cudaFreeHost(S->pin[sl]);
      S->pin[sl] = nullptr;
      CK(cudaHostAlloc((void**)&S->pin[sl], (size_t)need, cudaHostAllocDefault));
      S->pin_bytes[sl] = need;
    }
    uint8_t* b = S->pin[sl];
    uint8_t* pu = b + rec.sign_bytes;
    uint8_t* pv = pu + rec.u_bytes;
    float* ps = rec.s_bytes ? reinterpret_cast<float*>(pv + rec.v_bytes) : nullptr;
    rs = store_payload(S, first_record + j, rec, b, pu, pv, ps);   // disk -> pinned (overlaps the previous DMA)
    if (rs) return rs;
    rs = load_blocks_impl(L, rec.block, 1, b, pu, pv, ps, stream, false);   // pinned -> device, async
    if (rs) return rs;
    CK(cudaEventRecord(S->pin_ev[sl], reinterpret_cast<cudaStream_t>(stream)));
  }
  return BITSTACK_OK;
}

bitstack_status bitstack_store_close(bitstack_store S) {
  if (!S) return BITSTACK_OK;
  bitstack_status rs = BITSTACK_OK;
  if (S->writer) {
    const uint64_t idx = S->end;
    if (!write_all(S->fd, S->offsets.data(), S->offsets.size() * 8, idx))
      rs = fail(BITSTACK_E_IO, "store %s: index write failed", S->path.c_str());
    else
      rs = store_header(S, S->offsets.size(), idx);
    if (!rs && fsync(S->fd) != 0) rs = fail(BITSTACK_E_IO, "store %s: fsync failed", S->path.c_str());
  }
  for (int i = 0; i < 2; ++i) {
    if (S->pin_ev[i]) {
      cudaEventSynchronize(S->pin_ev[i]);
      cudaEventDestroy(S->pin_ev[i]);
    }
    if (S->pin[i]) cudaFreeHost(S->pin[i]);
  }
  close(S->fd);
  delete S;
  return rs;
}

}  // extern "C"
