// NDT1 container streaming and the reference's seeded generator (ndt1.cpp).
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include "error.h"
#include "ndsylv_b200.h"

namespace nds {

struct Ndt1File {
  std::FILE* f = nullptr;
  ~Ndt1File() {
    if (f) std::fclose(f);
  }
};

struct Ndt1Reader {
  Ndt1File file;
  std::string path;
  int n_modes = 0;
  int64_t dims[NDS_MAX_MODES] = {};
  int64_t total = 0, done = 0;
};

struct Ndt1Writer {
  Ndt1File file;
  std::string path;
};

void ndt1_open(Ndt1Reader& r, const char* path);              // parse + validate the header
void ndt1_read(Ndt1Reader& r, int64_t count, nds_z* out);     // next entries; trailing bytes -> error
void ndt1_create(Ndt1Writer& w, const char* path, int n_modes, const int64_t* dims);
void ndt1_write(Ndt1Writer& w, int64_t count, const nds_z* data);
void ndt1_close(Ndt1Writer& w);

// rng.cpp:18-33 draw order: the N matrices (column-major), then n_tensors tensors.
void random_draw(uint64_t seed, int n_modes, const int64_t* dims, nds_z* const* mats, int n_tensors,
                 nds_z* const* tensors);

}  // namespace nds
