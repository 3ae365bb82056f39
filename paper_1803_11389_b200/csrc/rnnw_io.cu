// RNNW / RNNX files straight into the device layouts.
//
// Formats: rnnblock model_io.py:1-33 (little-endian, fixed headers,
// row-major payloads, canonical field order per layer).  Validation and
// error classes follow load_weights / load_sequence (model_io.py:209-308):
// every failure returns RNNB_EFORMAT with the message prefixed by the
// reference's exception class name, which the Python shim maps back to
// BadMagicError / UnsupportedVersionError / TruncatedFileError /
// ShapeConsistencyError.  Sizes are checked against the remaining file
// length before anything is allocated (model_io.py:246-248).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rnnb.h"
#include "abi_guard.h"

namespace {

using rnnb::set_error;

constexpr uint32_t kVersion = 1;

struct File {
  FILE* f = nullptr;
  int64_t size = 0;
  explicit File(const char* path) {
    f = path ? std::fopen(path, "rb") : nullptr;
    if (f) {
      std::fseek(f, 0, SEEK_END);
      size = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
    }
  }
  ~File() {
    if (f) std::fclose(f);
  }
  int64_t remaining() const { return size - std::ftell(f); }
  bool read(void* dst, size_t n) { return std::fread(dst, 1, n, f) == n; }
};

rnnb_status ferr(const char* cls, const std::string& msg) {
  return set_error(RNNB_EFORMAT, std::string(cls) + ": " + msg);
}

uint32_t rd32(const unsigned char* p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }

struct LayerDims {
  int64_t d_in, d_h;
};

// Payload bytes of one layer, or -1 when they exceed `limit` (the bytes left
// in the file).  The header fields are untrusted u32s: d_h * d_in alone can
// reach 2^64, so the arithmetic is done in 128 bits and compared with the
// limit before anything is sized from it (model_io.py:246-248: a lying
// header must fail as truncated, never trigger a huge allocation).
int64_t layer_bytes_capped(int kind, int64_t din, int64_t dh, int es, int64_t limit) {
  using u128 = unsigned __int128;
  const u128 mat = (u128)(uint64_t)din * (u128)(uint64_t)dh;
  const u128 vec = (u128)(uint64_t)dh;
  u128 n;
  if (kind == 0) n = 4 * mat + 4 * (u128)(uint64_t)dh * (u128)(uint64_t)dh + 4 * vec;  // LSTM
  else if (kind == 1) n = 3 * mat + 2 * vec;                                            // SRU
  else n = 6 * mat;                                                                      // QRNN
  const u128 bytes = n * (u128)es;
  return bytes > (u128)(limit < 0 ? 0 : limit) ? -1 : (int64_t)bytes;
}

// Canonical per-layer array sizes (model_io.py:133-139); only called once
// layer_bytes_capped has bounded the products
void layer_spec(int kind, int64_t din, int64_t dh, std::vector<int64_t>& sizes) {
  sizes.clear();
  if (kind == 0) {  // LSTM
    for (int i = 0; i < 4; ++i) sizes.push_back(dh * din);
    for (int i = 0; i < 4; ++i) sizes.push_back(dh * dh);
    for (int i = 0; i < 4; ++i) sizes.push_back(dh);
  } else if (kind == 1) {  // SRU
    for (int i = 0; i < 3; ++i) sizes.push_back(dh * din);
    for (int i = 0; i < 2; ++i) sizes.push_back(dh);
  } else {  // QRNN
    for (int i = 0; i < 6; ++i) sizes.push_back(dh * din);
  }
}

// Parse and fully validate an RNNW file; optionally keep the payloads
// (widened to double; the stack upload converts to its mode).
rnnb_status parse_rnnw(const char* path, int* kind, int* prec, std::vector<LayerDims>* dims,
                       std::vector<std::vector<double>>* payload) {
  File file(path);
  if (!file.f) return set_error(RNNB_EINVAL, std::string("cannot open ") + (path ? path : "(null)"));
  unsigned char h[16];
  if (!file.read(h, 16)) return ferr("TruncatedFileError", "file ends inside header");
  if (std::memcmp(h, "RNNW", 4) != 0) return ferr("BadMagicError", "bad magic, expected 'RNNW'");
  const uint32_t version = rd32(h + 4);
  if (version != kVersion)
    return ferr("UnsupportedVersionError", "format version " + std::to_string(version) + ", expected 1");
  const int k = h[8], p = h[9];
  const uint32_t n_layers = rd32(h + 12);
  if (k > 2) return ferr("ShapeConsistencyError", "unknown cell kind code " + std::to_string(k));
  if (p > 1) return ferr("ShapeConsistencyError", "unknown precision code " + std::to_string(p));
  if (n_layers < 1) return ferr("ShapeConsistencyError", "layer count must be >= 1");
  const int es = p == 1 ? 8 : 4;
  std::vector<int64_t> sizes;
  int64_t prev_dh = -1;
  for (uint32_t li = 0; li < n_layers; ++li) {
    const std::string lname = "layer " + std::to_string(li);
    unsigned char lh[8];
    if (!file.read(lh, 8)) return ferr("TruncatedFileError", "file ends inside " + lname + " header");
    const int64_t din = rd32(lh), dh = rd32(lh + 4);
    if (din < 1 || dh < 1) return ferr("ShapeConsistencyError", lname + " has zero dimension");
    if (k == 1 && din != dh) return ferr("ShapeConsistencyError", "SRU layer must have d_in == d_h");
    if (prev_dh >= 0 && din != prev_dh)
      return ferr("ShapeConsistencyError", lname + " input width does not match previous layer width");
    prev_dh = dh;
    const int64_t nbytes = layer_bytes_capped(k, din, dh, es, file.remaining());
    if (nbytes < 0) return ferr("TruncatedFileError", lname + " payload incomplete");
    const int64_t n = nbytes / es;
    if (dims) dims->push_back({din, dh});
    if (payload) {
      std::vector<unsigned char> raw((size_t)nbytes);
      if (!file.read(raw.data(), raw.size())) return ferr("TruncatedFileError", lname + " data");
      std::vector<double> vals((size_t)n);
      for (int64_t i = 0; i < n; ++i) {
        if (es == 8) {
          std::memcpy(&vals[(size_t)i], &raw[(size_t)i * 8], 8);
        } else {
          float f;
          std::memcpy(&f, &raw[(size_t)i * 4], 4);
          vals[(size_t)i] = f;
        }
      }
      payload->push_back(std::move(vals));
    } else {
      std::fseek(file.f, (long)(n * es), SEEK_CUR);
    }
  }
  if (file.remaining() != 0) return ferr("ShapeConsistencyError", "trailing bytes after final layer");
  *kind = k;
  *prec = p;
  return RNNB_OK;
}

std::vector<const void*> layer_ptrs(int kind, const LayerDims& d, const std::vector<double>& vals) {
  std::vector<int64_t> sizes;
  layer_spec(kind, d.d_in, d.d_h, sizes);
  std::vector<const void*> mats;
  size_t off = 0;
  for (int64_t s : sizes) {
    mats.push_back(vals.data() + off);
    off += (size_t)s;
  }
  return mats;
}

}  // namespace

extern "C" {

rnnb_status rnnb_rnnw_info(const char* path, int* kind, int* precision, int* n_layers, int64_t* d_in, int64_t* d_h,
                           int max_layers) {
  return rnnb::abi_guard("rnnb_rnnw_info", [&]() -> rnnb_status {
    if (!kind || !precision || !n_layers) return set_error(RNNB_EINVAL, "null output argument");
    std::vector<LayerDims> dims;
    int k = 0, p = 0;
    rnnb_status st = parse_rnnw(path, &k, &p, &dims, nullptr);
    if (st != RNNB_OK) return st;
    *kind = k;
    *precision = p;
    *n_layers = (int)dims.size();
    for (int i = 0; i < (int)dims.size() && i < max_layers; ++i) {
      if (d_in) d_in[i] = dims[(size_t)i].d_in;
      if (d_h) d_h[i] = dims[(size_t)i].d_h;
    }
    return RNNB_OK;
  });
}

rnnb_status rnnb_stack_load_rnnw(rnnb_stack_t* out, const char* path, int mode, int device) {
  return rnnb::abi_guard("rnnb_stack_load_rnnw", [&]() -> rnnb_status {
    if (!out) return set_error(RNNB_EINVAL, "null output handle");
    *out = nullptr;
    std::vector<LayerDims> dims;
    std::vector<std::vector<double>> payload;
    int k = 0, p = 0;
    rnnb_status st = parse_rnnw(path, &k, &p, &dims, &payload);
    if (st != RNNB_OK) return st;
    if (k == 0) return set_error(RNNB_EINVAL, "blocked execution covers SRU and QRNN; use rnnb_lstm_load_rnnw for LSTM");
    const int n = (int)dims.size();
    std::vector<int64_t> din(n), dh(n);
    for (int i = 0; i < n; ++i) din[i] = dims[i].d_in, dh[i] = dims[i].d_h;
    rnnb_stack_t h = nullptr;
    st = rnnb_stack_create(&h, k, n, din.data(), dh.data(), mode, device);
    if (st != RNNB_OK) return st;
    for (int li = 0; li < n; ++li) {
      std::vector<const void*> mats = layer_ptrs(k, dims[(size_t)li], payload[(size_t)li]);
      st = rnnb_stack_set_layer(h, li, mats.data(), (int)mats.size(), RNNB_DT_F64);
      if (st != RNNB_OK) {
        rnnb_stack_destroy(h);
        return st;
      }
    }
    *out = h;
    return RNNB_OK;
  });
}

rnnb_status rnnb_lstm_load_rnnw(rnnb_lstm_t* out, const char* path, int layer, int mode, int device) {
  return rnnb::abi_guard("rnnb_lstm_load_rnnw", [&]() -> rnnb_status {
    if (!out) return set_error(RNNB_EINVAL, "null output handle");
    *out = nullptr;
    std::vector<LayerDims> dims;
    std::vector<std::vector<double>> payload;
    int k = 0, p = 0;
    rnnb_status st = parse_rnnw(path, &k, &p, &dims, &payload);
    if (st != RNNB_OK) return st;
    if (k != 0) return set_error(RNNB_EINVAL, "file does not hold LSTM weights");
    if (layer < 0 || layer >= (int)dims.size()) return set_error(RNNB_EINVAL, "layer index out of range");
    const LayerDims& d = dims[(size_t)layer];
    rnnb_lstm_t h = nullptr;
    st = rnnb_lstm_create(&h, d.d_in, d.d_h, mode, device);
    if (st != RNNB_OK) return st;
    std::vector<const void*> mats = layer_ptrs(0, d, payload[(size_t)layer]);
    st = rnnb_lstm_set_weights(h, mats.data(), (int)mats.size(), RNNB_DT_F64);
    if (st != RNNB_OK) {
      rnnb_lstm_destroy(h);
      return st;
    }
    *out = h;
    return RNNB_OK;
  });
}

rnnb_status rnnb_rnnw_read(const char* path, void* dst, int64_t n, int dst_dtype) {
  return rnnb::abi_guard("rnnb_rnnw_read", [&]() -> rnnb_status {
    if (!dst) return set_error(RNNB_EINVAL, "null destination");
    if (dst_dtype != RNNB_DT_F32 && dst_dtype != RNNB_DT_F64) return set_error(RNNB_EINVAL, "dst dtype must be f32 or f64");
    std::vector<LayerDims> dims;
    std::vector<std::vector<double>> payload;
    int k = 0, p = 0;
    rnnb_status st = parse_rnnw(path, &k, &p, &dims, &payload);
    if (st != RNNB_OK) return st;
    int64_t total = 0;
    for (auto& v : payload) total += (int64_t)v.size();
    if (n != total)
      return set_error(RNNB_EINVAL, "destination holds " + std::to_string(n) + " elements, file has " +
                                        std::to_string(total));
    int64_t o = 0;
    for (auto& v : payload)
      for (double x : v) {
        if (dst_dtype == RNNB_DT_F64) static_cast<double*>(dst)[o++] = x;
        else static_cast<float*>(dst)[o++] = (float)x;
      }
    return RNNB_OK;
  });
}

rnnb_status rnnb_rnnx_info(const char* path, int* precision, int64_t* seq_len, int64_t* width) {
  return rnnb::abi_guard("rnnb_rnnx_info", [&]() -> rnnb_status {
    File file(path);
    if (!file.f) return set_error(RNNB_EINVAL, std::string("cannot open ") + (path ? path : "(null)"));
    unsigned char h[20];
    if (!file.read(h, 20)) return ferr("TruncatedFileError", "file ends inside header");
    if (std::memcmp(h, "RNNX", 4) != 0) return ferr("BadMagicError", "bad magic, expected 'RNNX'");
    const uint32_t version = rd32(h + 4);
    if (version != kVersion)
      return ferr("UnsupportedVersionError", "format version " + std::to_string(version) + ", expected 1");
    const int p = h[8];
    const int64_t L = rd32(h + 12), W = rd32(h + 16);
    if (p > 1) return ferr("ShapeConsistencyError", "unknown precision code " + std::to_string(p));
    if (L < 1 || W < 1) return ferr("ShapeConsistencyError", "sequence dimensions must be >= 1");
    // L, W < 2^32 each: L * W * 8 needs up to 67 bits, so compare in 128 bits
    const unsigned __int128 payload = (unsigned __int128)(uint64_t)L * (uint64_t)W * (unsigned)(p == 1 ? 8 : 4);
    const int64_t got = file.remaining();
    if ((unsigned __int128)(got < 0 ? 0 : got) < payload) return ferr("TruncatedFileError", "payload incomplete");
    if ((unsigned __int128)got > payload) return ferr("ShapeConsistencyError", "trailing bytes after payload");
    if (precision) *precision = p;
    if (seq_len) *seq_len = L;
    if (width) *width = W;
    return RNNB_OK;
  });
}

rnnb_status rnnb_rnnx_load(const char* path, void* dst, int dst_dtype, int dst_on_device, void* stream) {
  return rnnb::abi_guard("rnnb_rnnx_load", [&]() -> rnnb_status {
    int p = 0;
    int64_t L = 0, W = 0;
    rnnb_status st = rnnb_rnnx_info(path, &p, &L, &W);
    if (st != RNNB_OK) return st;
    if (!dst) return set_error(RNNB_EINVAL, "null destination");
    if (dst_dtype != RNNB_DT_F32 && dst_dtype != RNNB_DT_F64) return set_error(RNNB_EINVAL, "dst dtype must be f32 or f64");
    File file(path);
    std::fseek(file.f, 20, SEEK_SET);
    const int64_t n = L * W;
    const int ses = p == 1 ? 8 : 4, des = dst_dtype == RNNB_DT_F64 ? 8 : 4;
    constexpr int64_t kPiece = 1 << 20;  // elements per piece
    std::vector<unsigned char> raw((size_t)(kPiece * ses));
    unsigned char* stage = nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaEvent_t done[2] = {nullptr, nullptr};
    if (dst_on_device) {
      if (cudaMallocHost(&stage, (size_t)(2 * kPiece * des)) != cudaSuccess)
        return set_error(RNNB_ECUDA, "pinned staging allocation failed");
      cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
    }
    auto cleanup = [&]() {
      if (stage) cudaFreeHost(stage);
      for (auto& e : done)
        if (e) cudaEventDestroy(e);
    };
    int slot = 0;
    for (int64_t i0 = 0, piece = 0; i0 < n; i0 += kPiece, ++piece, slot ^= 1) {
      const int64_t m = (n - i0) < kPiece ? (n - i0) : kPiece;
      if (!file.read(raw.data(), (size_t)(m * ses))) {
        cleanup();
        return ferr("TruncatedFileError", "payload incomplete");
      }
      unsigned char* outp = dst_on_device ? stage + (size_t)slot * kPiece * des
                                          : static_cast<unsigned char*>(dst) + (size_t)i0 * des;
      if (dst_on_device && piece >= 2) cudaEventSynchronize(done[slot]);  // the copy out of this slot is done
      for (int64_t i = 0; i < m; ++i) {
        double v;
        if (ses == 8) {
          std::memcpy(&v, &raw[(size_t)i * 8], 8);
        } else {
          float f;
          std::memcpy(&f, &raw[(size_t)i * 4], 4);
          v = f;
        }
        if (des == 8) {
          std::memcpy(outp + (size_t)i * 8, &v, 8);
        } else {
          const float f = (float)v;
          std::memcpy(outp + (size_t)i * 4, &f, 4);
        }
      }
      if (dst_on_device) {
        cudaError_t e = cudaMemcpyAsync(static_cast<unsigned char*>(dst) + (size_t)i0 * des, outp, (size_t)(m * des),
                                        cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(done[slot], s);
        if (e != cudaSuccess) {
          cleanup();
          return set_error(RNNB_ECUDA, std::string("RNNX upload: ") + cudaGetErrorString(e));
        }
      }
    }
    if (dst_on_device) cudaStreamSynchronize(s);
    cleanup();
    return RNNB_OK;
  });
}

}  // extern "C"
