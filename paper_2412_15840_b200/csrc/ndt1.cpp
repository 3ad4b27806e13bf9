// NDT1 tensor container and the reference's seeded problem generator, host side.
//
// NDT1 (reference tensor_file.hpp:9-15, tensor_file.cpp:48-96): little-endian
//   "NDT1" | u32 version = 1 | u32 order N (1..64) | u64 n_1 .. n_N | f64 (re, im) x total,
// entries column-major; reading rejects bad magic, other versions, zero / overflowing extents and
// payloads shorter or longer than the header says (TensorFileError -> NDS_ERR_FILE).
// The payload moves in large blocks (the host is little-endian, like every CUDA host), and the
// chunked readers/writers below let the C ABI stream multi-GiB tensors through pinned buffers.
//
// Generator (reference rng.hpp:12-49, rng.cpp:5-33): xoshiro256++ seeded through splitmix64,
// uniforms from the top 53 bits, complex entries (re then im); random_problem draws A_1..A_N
// (column-major) then X_true from one stream; random_ode_system draws A_1..A_N, the forcing, then
// the initial state. Restated from the published algorithm.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "ndt1.h"

namespace nds {

namespace {

constexpr char kMagic[4] = {'N', 'D', 'T', '1'};

uint32_t le32(const unsigned char* b) { return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24; }
uint64_t le64(const unsigned char* b) { return (uint64_t)le32(b) | (uint64_t)le32(b + 4) << 32; }

}  // namespace

// Open + parse the header (tensor_file.cpp:67-88).
void ndt1_open(Ndt1Reader& r, const char* path) {
  r.path = path ? path : "";
  r.file.f = std::fopen(r.path.c_str(), "rb");
  if (!r.file.f) throw Error(NDS_ERR_FILE, "cannot open '" + r.path + "' for reading");
  unsigned char h[12];
  if (std::fread(h, 1, 4, r.file.f) != 4) throw Error(NDS_ERR_FILE, "'" + r.path + "': unexpected end of file");
  if (std::memcmp(h, kMagic, 4) != 0) throw Error(NDS_ERR_FILE, "'" + r.path + "': not a tensor container");
  if (std::fread(h, 1, 8, r.file.f) != 8) throw Error(NDS_ERR_FILE, "unexpected end of file");
  const uint32_t version = le32(h), order = le32(h + 4);
  if (version != 1) throw Error(NDS_ERR_FILE, "'" + r.path + "': unsupported format version " + std::to_string(version));
  if (order == 0 || order > 64) throw Error(NDS_ERR_FILE, "'" + r.path + "': invalid tensor order");
  r.n_modes = (int)order;
  int64_t total = 1;
  for (uint32_t j = 0; j < order; ++j) {
    unsigned char b[8];
    if (std::fread(b, 1, 8, r.file.f) != 8) throw Error(NDS_ERR_FILE, "unexpected end of file");
    const uint64_t n = le64(b);
    if (n == 0 || n > (uint64_t)INT64_MAX) throw Error(NDS_ERR_FILE, "'" + r.path + "': invalid extent");
    r.dims[j] = (int64_t)n;
    if (__builtin_mul_overflow(total, (int64_t)n, &total) || total > INT64_MAX / 16)
      throw Error(NDS_ERR_FILE, "'" + r.path + "': extents overflow");
  }
  r.total = total;
}

// Next `count` entries of the payload into out (complex128 = two little-endian f64).
void ndt1_read(Ndt1Reader& r, int64_t count, nds_z* out) {
  if (count > r.total - r.done) count = r.total - r.done;
  if (count > 0 && std::fread(out, sizeof(nds_z), (size_t)count, r.file.f) != (size_t)count)
    throw Error(NDS_ERR_FILE, "unexpected end of file");
  r.done += count;
  if (r.done == r.total) {  // tensor_file.cpp:94-95: nothing may follow the payload
    if (std::fgetc(r.file.f) != EOF) throw Error(NDS_ERR_FILE, "'" + r.path + "': trailing bytes after payload");
  }
}

void ndt1_create(Ndt1Writer& w, const char* path, int n_modes, const int64_t* dims) {
  w.path = path ? path : "";
  if (n_modes < 1 || n_modes > 64) throw Error(NDS_ERR_INVALID, "tensor order must be 1..64");
  int64_t total = 1;
  for (int j = 0; j < n_modes; ++j) {
    if (dims[j] < 1) throw Error(NDS_ERR_INVALID, "tensor dimensions must be at least 1");
    if (__builtin_mul_overflow(total, dims[j], &total)) throw Error(NDS_ERR_OVERFLOW, "tensor size overflows int64");
  }
  w.file.f = std::fopen(w.path.c_str(), "wb");
  if (!w.file.f) throw Error(NDS_ERR_FILE, "cannot open '" + w.path + "' for writing");
  unsigned char h[12] = {'N', 'D', 'T', '1', 1, 0, 0, 0};
  for (int i = 0; i < 4; ++i) h[8 + i] = (unsigned char)(((uint32_t)n_modes >> (8 * i)) & 0xff);
  bool ok = std::fwrite(h, 1, 12, w.file.f) == 12;
  for (int j = 0; j < n_modes && ok; ++j) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(((uint64_t)dims[j] >> (8 * i)) & 0xff);
    ok = std::fwrite(b, 1, 8, w.file.f) == 8;
  }
  if (!ok) throw Error(NDS_ERR_FILE, "write to '" + w.path + "' failed");
}

void ndt1_write(Ndt1Writer& w, int64_t count, const nds_z* data) {
  if (count > 0 && std::fwrite(data, sizeof(nds_z), (size_t)count, w.file.f) != (size_t)count)
    throw Error(NDS_ERR_FILE, "write to '" + w.path + "' failed");
}

void ndt1_close(Ndt1Writer& w) {
  if (w.file.f && std::fclose(w.file.f) != 0) {
    w.file.f = nullptr;
    throw Error(NDS_ERR_FILE, "write to '" + w.path + "' failed");
  }
  w.file.f = nullptr;
}

// ---- xoshiro256++ (rng.hpp:12-49) ------------------------------------------------------------
struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) {
      sm += 0x9e3779b97f4a7c15ULL;
      uint64_t z = sm;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      w = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  nds_z uniform_complex() {
    const double re = uniform();
    return nds_z{re, uniform()};
  }
};

// Draw order of rng.cpp:18-33: the N matrices (column-major), then each listed tensor in turn.
void random_draw(uint64_t seed, int n_modes, const int64_t* dims, nds_z* const* mats, int n_tensors,
                 nds_z* const* tensors) {
  Xoshiro rng(seed);
  int64_t total = 1;
  for (int j = 0; j < n_modes; ++j) {
    const int64_t n = dims[j];
    for (int64_t e = 0; e < n * n; ++e) mats[j][e] = rng.uniform_complex();
    total *= n;
  }
  for (int k = 0; k < n_tensors; ++k)
    for (int64_t e = 0; e < total; ++e) tensors[k][e] = rng.uniform_complex();
}

}  // namespace nds
