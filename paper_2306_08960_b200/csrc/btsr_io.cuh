// BTSR container -> device memory.
//
// Format and checks follow the reference loader (tensor_io.hpp:14-20, tensor_io.cpp:139-215):
//   magic "BTSR" | version u32 = 1 | kind u8 | rows u64 | cols u64 | payload, little-endian
//   0 dense: rows*cols f32            1 bit: words_per_row u64, rows*wpr u64
//   2 csr:   nnz u64, row_ptr u64[rows+1], col_idx u64[nnz], vals f32[nnz]
// Errors carry the reference's IoError texts ("bad magic: <path>", "truncated file: <path>",
// "trailing bytes: <path>", "<validation message>: <path>", ...) in the reference's order:
// header, size (truncated before trailing), then the object validation of BitMatrix::from_words
// (tensor.cpp:62-89), CsrMatrix::create (tensor.cpp:91-123) or the DenseMatrix constructor
// (tensor.cpp:38-48).
//
// Loading streams the payload through two pinned host chunks: chunk i is read and validated on
// the host while chunk i-1 is copied to the device on the caller's stream.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace bitmm_dev {

constexpr uint64_t kBtsrMaxElems = uint64_t{1} << 40;  // tensor_io.cpp:17
constexpr size_t kBtsrChunk = size_t{8} << 20;          // pinned staging chunk (bytes)

struct BtsrFile {
  FILE* f = nullptr;
  std::string path;
  ~BtsrFile() {
    if (f) fclose(f);
  }
  bool read(void* p, size_t n) { return fread(p, 1, n, f) == n; }
};

struct BtsrHeader {
  int kind = 0;
  uint64_t rows = 0, cols = 0, wpr = 0, nnz = 0;
  uint64_t payload_bytes = 0;  // after the kind's count field
  long header_bytes = 0;
};

inline uint64_t le64(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

// Opens and validates everything the reference checks before touching the payload values.
// Returns an empty string on success, else the IoError text.
inline std::string btsr_open(const char* path, BtsrFile& bf, BtsrHeader& h) {
  bf.path = path;
  bf.f = fopen(path, "rb");
  if (!bf.f) return "cannot open for reading: " + bf.path;
  unsigned char hdr[4 + 4 + 1 + 8 + 8];
  if (!bf.read(hdr, 4)) return "truncated file: " + bf.path;
  if (hdr[0] != 'B' || hdr[1] != 'T' || hdr[2] != 'S' || hdr[3] != 'R') return "bad magic: " + bf.path;
  if (!bf.read(hdr + 4, sizeof(hdr) - 4)) return "truncated file: " + bf.path;
  const uint32_t version = hdr[4] | (hdr[5] << 8) | (hdr[6] << 16) | (static_cast<uint32_t>(hdr[7]) << 24);
  if (version != 1) return "unsupported container version " + std::to_string(version) + ": " + bf.path;
  const unsigned kind = hdr[8];
  if (kind > 2) return "unknown tensor kind " + std::to_string(kind) + ": " + bf.path;
  h.kind = static_cast<int>(kind);
  h.rows = le64(hdr + 9);
  h.cols = le64(hdr + 17);
  if (h.rows > kBtsrMaxElems || h.cols > kBtsrMaxElems ||
      (h.rows != 0 && h.cols > kBtsrMaxElems / h.rows))
    return "dimension overflow: " + bf.path;
  h.header_bytes = sizeof(hdr);
  unsigned char b8[8];
  if (h.kind == 0) {
    h.payload_bytes = h.rows * h.cols * 4;
  } else if (h.kind == 1) {
    if (!bf.read(b8, 8)) return "truncated file: " + bf.path;
    h.wpr = le64(b8);
    if (h.wpr > kBtsrMaxElems || (h.rows != 0 && h.wpr > kBtsrMaxElems / h.rows))
      return "dimension overflow: " + bf.path;
    h.payload_bytes = h.rows * h.wpr * 8;
    h.header_bytes += 8;
  } else {
    if (!bf.read(b8, 8)) return "truncated file: " + bf.path;
    h.nnz = le64(b8);
    if (h.nnz > kBtsrMaxElems) return "dimension overflow: " + bf.path;
    h.payload_bytes = (h.rows + 1) * 8 + h.nnz * 8 + h.nnz * 4;
    h.header_bytes += 8;
  }
  // the reference reads the payload value by value: a short file is "truncated", a longer one
  // "trailing bytes" (checked after the whole payload was read)
  if (fseek(bf.f, 0, SEEK_END) != 0) return "truncated file: " + bf.path;
  const long size = ftell(bf.f);
  const uint64_t want = static_cast<uint64_t>(h.header_bytes) + h.payload_bytes;
  if (size < 0 || static_cast<uint64_t>(size) < want) return "truncated file: " + bf.path;
  if (static_cast<uint64_t>(size) > want) return "trailing bytes: " + bf.path;
  if (fseek(bf.f, h.header_bytes, SEEK_SET) != 0) return "truncated file: " + bf.path;
  // constructor-level shape checks that need no payload values
  if (h.kind == 1 && h.wpr * 64 < h.cols)
    return "words_per_row too small for the column count: " + bf.path;
  return std::string();
}

// Streams `bytes` from the file to `dst` (device) through the pinned double buffer, calling
// check(host_ptr, offset, n) on every chunk before its copy is queued. check returns "" or
// the validation message.
template <class Check>
std::string btsr_stream(BtsrFile& bf, uint8_t* dst, uint64_t bytes, void* pinned[2],
                        cudaEvent_t ev[2], cudaStream_t s, Check&& check, cudaError_t* cerr) {
  uint64_t off = 0;
  int b = 0;
  // copies queued by an earlier call may still read the pinned chunks
  for (int i = 0; i < 2; ++i) {
    *cerr = cudaEventSynchronize(ev[i]);
    if (*cerr != cudaSuccess) return "cuda";
  }
  bool used[2] = {false, false};
  while (off < bytes) {
    const size_t n = static_cast<size_t>(std::min<uint64_t>(kBtsrChunk, bytes - off));
    if (used[b]) {
      *cerr = cudaEventSynchronize(ev[b]);
      if (*cerr != cudaSuccess) return "cuda";
    }
    if (!bf.read(pinned[b], n)) return "truncated file: " + bf.path;
    std::string msg = check(static_cast<const uint8_t*>(pinned[b]), off, n);
    if (!msg.empty()) return msg + ": " + bf.path;
    *cerr = cudaMemcpyAsync(dst + off, pinned[b], n, cudaMemcpyHostToDevice, s);
    if (*cerr != cudaSuccess) return "cuda";
    *cerr = cudaEventRecord(ev[b], s);
    if (*cerr != cudaSuccess) return "cuda";
    used[b] = true;
    off += n;
    b ^= 1;
  }
  return std::string();
}

}  // namespace bitmm_dev
