#pragma once

#include "error.h"

namespace nds {

// Host complex Schur: a (n x n, column-major) = u t u^H. Throws nds::Error.
void schur_host(int n, const nds_z* a, nds_z* u, nds_z* t);

// exp(t T) of an upper triangular T (n x n, column-major): Parlett recurrence when the diagonal
// is well separated, else Taylor scaling and squaring (matfun.cpp). Throws nds::Error.
void triangular_exp_host(int n, const nds_z* t_mat, double t, nds_z* f);
// The Parlett route's separation test on T's diagonal (host and device route choice).
bool exp_diagonal_separated(int n, const nds_z* t_mat);

// Seeded standard normals (see nds_randn).
void randn_host(uint64_t seed, uint64_t stream, int64_t count, double* out);

}  // namespace nds
