// tnsr.hpp -- the reference's TNSR tensor file format (tensor.hpp:76-139) over
// raw host buffers, with the bf16 / i32 extension codes.
//
// Layout, as save_tensor / load_tensor (tensor.hpp:80-133) define it:
//   "TNSR", u8 dtype code, u8 rank, u64 dims[rank] little-endian, raw LE data.
// Codes 0 (f32, 4 B) and 1 (f16, 2 B) are the reference's; 2 (bf16, 2 B) and
// 3 (i32, 4 B) are this backend's extension and equal the DType values of
// ext_ops.hpp / the TCB_* codes of tcb200.h.  An f32/f16 file written here is
// byte-identical to the reference's save_tensor of the same tensor, and the
// reference's load_tensor reads it (tests/test_tnsr.py pins both directions).
//
// The data section is written from / read into the caller's buffer as stored
// bytes: there is no float round trip, so f16/bf16 payloads move bit-exactly
// (the reference widens f16 to float in memory, which is also exact).  Errors
// carry the reference's messages ("bad tensor file magic", "bad tensor file
// header", "truncated tensor file", "cannot open <path>").
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "trainc/dtype.hpp"

namespace tb::tnsr {

inline int code_bytes(int code) {
  switch (code) {
    case 0: case 3: return 4;
    case 1: case 2: return 2;
    default: throw trainc::Error("bad tensor file header");
  }
}

struct Header {
  int code = 0;
  std::vector<int64_t> shape;
  int64_t numel() const {
    int64_t n = 1;
    for (auto d : shape) n *= d;
    return n;
  }
  int64_t data_bytes() const { return numel() * code_bytes(code); }
};

inline void save(const std::string& path, const Header& h, const void* data) {
  if (h.shape.size() > 255) throw trainc::Error("tensor rank exceeds the TNSR u8 rank field");
  for (auto d : h.shape)
    if (d < 0) throw trainc::Error("negative dimension in TNSR save");
  std::ofstream f(path, std::ios::binary);
  if (!f) throw trainc::Error("cannot open " + path + " for writing");
  f.write("TNSR", 4);
  f.put(static_cast<char>(static_cast<uint8_t>(h.code)));
  f.put(static_cast<char>(static_cast<uint8_t>(h.shape.size())));
  for (auto d : h.shape) {
    uint64_t u = static_cast<uint64_t>(d);
    f.write(reinterpret_cast<const char*>(&u), 8);  // x86/aarch64 hosts are LE
  }
  f.write(static_cast<const char*>(data), static_cast<std::streamsize>(h.data_bytes()));
  if (!f) throw trainc::Error("write failed: " + path);
}

/// Reads the header and leaves `f` positioned at the data section.
inline Header read_header(std::ifstream& f) {
  char magic[4];
  f.read(magic, 4);
  if (!f || std::memcmp(magic, "TNSR", 4) != 0) throw trainc::Error("bad tensor file magic");
  int code = f.get();
  int rank = f.get();
  if (code < 0 || code > 3 || rank < 0) throw trainc::Error("bad tensor file header");
  Header h;
  h.code = code;
  for (int i = 0; i < rank; ++i) {
    uint64_t u = 0;
    f.read(reinterpret_cast<char*>(&u), 8);
    h.shape.push_back(static_cast<int64_t>(u));
  }
  if (!f) throw trainc::Error("truncated tensor file");
  return h;
}

inline Header load_header(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw trainc::Error("cannot open " + path);
  return read_header(f);
}

/// Reads the data section into `data` (capacity `bytes`, which must equal the
/// header's data size) and returns the header.
inline Header load(const std::string& path, void* data, int64_t bytes) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw trainc::Error("cannot open " + path);
  Header h = read_header(f);
  if (h.data_bytes() != bytes)
    throw trainc::Error("TNSR size mismatch: file holds " + std::to_string(h.data_bytes()) +
                        " bytes, buffer " + std::to_string(bytes));
  f.read(static_cast<char*>(data), static_cast<std::streamsize>(bytes));
  if (!f) throw trainc::Error("truncated tensor file");
  return h;
}

}  // namespace tb::tnsr
