#pragma once

#include "error.h"

namespace nds {

// Host complex Schur: a (n x n, column-major) = u t u^H. Throws nds::Error.
void schur_host(int n, const nds_z* a, nds_z* u, nds_z* t);

// Seeded standard normals (see nds_randn).
void randn_host(uint64_t seed, uint64_t stream, int64_t count, double* out);

}  // namespace nds
