// meshgen.cpp -- seeded synthetic inputs for the BASELINE configurations.
//
// Host-side input generation (not on the timed path).  The meshes restate the
// reference generators bit-exactly -- unit_square_mesh (mesh.hpp:96-143) and
// unit_cube_mesh (mesh.hpp:148-214) -- and add what the reference lacks
// (SURVEY 8d): interior-vertex jitter, Fisher-Yates cell permutation and
// coefficient fields, all driven by one self-contained splitmix64 stream so
// that inputs never depend on <random> implementation details.  The P2
// cell->node map restates fem/space.hpp:48-72 (sort-based instead of
// std::set/std::map; identical numbering) and extends it to tetrahedra.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "loam_gpu.h"

namespace {

struct SplitMix64 {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// Local edges of the P2 cell row, in node order after the vertices.
constexpr int kTriEdges[3][2] = {{1, 2}, {0, 2}, {0, 1}};                         // space.hpp:66-71
constexpr int kTetEdges[6][2] = {{2, 3}, {1, 3}, {1, 2}, {0, 3}, {0, 2}, {0, 1}}; // extension

} // namespace

extern "C" {

int loam_gpu_unit_square_mesh(int n, double* coords, int32_t* cv) {
  if (n < 1) return LOAM_ERR(InvalidSubdivision);
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      int64_t v = static_cast<int64_t>(j) * (n + 1) + i;
      coords[2 * v] = static_cast<double>(i) / n;
      coords[2 * v + 1] = static_cast<double>(j) / n;
    }
  int64_t k = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      int a = j * (n + 1) + i, b = a + 1, c = a + n + 2, d = a + n + 1;
      cv[k++] = a; cv[k++] = b; cv[k++] = c; // SW-NE split, positively oriented
      cv[k++] = a; cv[k++] = c; cv[k++] = d;
    }
  return 0;
}

int loam_gpu_unit_cube_mesh(int n, double* coords, int32_t* cv) {
  if (n < 1) return LOAM_ERR(InvalidSubdivision);
  const int s = n + 1;
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) {
        int64_t v = (static_cast<int64_t>(k) * s + j) * s + i;
        coords[3 * v] = static_cast<double>(i) / n;
        coords[3 * v + 1] = static_cast<double>(j) / n;
        coords[3 * v + 2] = static_cast<double>(k) / n;
      }
  // Kuhn subdivision: one tet per axis permutation, odd ones re-oriented.
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const bool odd[6] = {false, true, true, false, false, true};
  int64_t w = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (int p = 0; p < 6; ++p) {
          int ijk[3] = {i, j, k};
          int tet[4];
          tet[0] = (ijk[2] * s + ijk[1]) * s + ijk[0];
          for (int step = 0; step < 3; ++step) {
            ijk[perms[p][step]] += 1;
            tet[step + 1] = (ijk[2] * s + ijk[1]) * s + ijk[0];
          }
          if (odd[p]) std::swap(tet[2], tet[3]);
          for (int t = 0; t < 4; ++t) cv[w++] = tet[t];
        }
  return 0;
}

// x += (2u - 1) * amp * h for every coordinate of every interior vertex, in
// vertex order then coordinate order.  h = 1/n.
int loam_gpu_jitter(int gdim, int n, double amp, uint64_t seed, double* coords) {
  if ((gdim != 2 && gdim != 3) || n < 1) return LOAM_ERR(InvalidArgument);
  SplitMix64 rng{seed};
  const int s = n + 1;
  const int64_t nv = gdim == 2 ? static_cast<int64_t>(s) * s : static_cast<int64_t>(s) * s * s;
  const double h = 1.0 / n;
  for (int64_t v = 0; v < nv; ++v) {
    int64_t i = v % s, j = (v / s) % s, k = gdim == 3 ? v / (static_cast<int64_t>(s) * s) : 1;
    bool interior = i > 0 && i < n && j > 0 && j < n && (gdim == 2 || (k > 0 && k < n));
    if (!interior) continue;
    for (int d = 0; d < gdim; ++d) coords[v * gdim + d] += (2.0 * rng.uniform() - 1.0) * amp * h;
  }
  return 0;
}

// Fisher-Yates over cell rows, from the last cell down, j = next() % (i+1).
int loam_gpu_permute_cells(int ncells, int arity, uint64_t seed, int32_t* cv) {
  if (ncells < 0 || arity < 1) return LOAM_ERR(InvalidArgument);
  SplitMix64 rng{seed};
  for (int64_t i = static_cast<int64_t>(ncells) - 1; i >= 1; --i) {
    int64_t j = static_cast<int64_t>(rng.next() % static_cast<uint64_t>(i + 1));
    if (j != i)
      for (int a = 0; a < arity; ++a) std::swap(cv[i * arity + a], cv[j * arity + a]);
  }
  return 0;
}

int loam_gpu_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out) {
  SplitMix64 rng{seed};
  for (int64_t k = 0; k < count; ++k) out[k] = lo + (hi - lo) * rng.uniform();
  return 0;
}

// P2 cell->node map (space.hpp:48-72): vertex nodes keep their ids, unique
// sorted-pair edges are numbered lexicographically from nv.  Returns the node
// count (>0) or a negative error code.
int loam_gpu_p2_cell_node_map(int ncells, int nv, int gdim, const int32_t* cv, int32_t* cn) {
  if (gdim != 2 && gdim != 3) return -LOAM_ERR(InvalidArgument);
  const int nvc = gdim + 1, ne = gdim == 2 ? 3 : 6, row = nvc + ne;
  const int (*edges)[2] = gdim == 2 ? kTriEdges : kTetEdges;
  std::vector<uint64_t> keys(static_cast<size_t>(ncells) * ne);
  auto key_of = [&](int64_t c, int k) {
    uint32_t a = static_cast<uint32_t>(cv[c * nvc + edges[k][0]]);
    uint32_t b = static_cast<uint32_t>(cv[c * nvc + edges[k][1]]);
    if (a > b) std::swap(a, b);
    return (static_cast<uint64_t>(a) << 32) | b;
  };
  for (int64_t c = 0; c < ncells; ++c)
    for (int k = 0; k < ne; ++k) keys[c * ne + k] = key_of(c, k);
  std::vector<uint64_t> uniq(keys);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  for (int64_t c = 0; c < ncells; ++c) {
    for (int v = 0; v < nvc; ++v) cn[c * row + v] = cv[c * nvc + v];
    for (int k = 0; k < ne; ++k) {
      auto it = std::lower_bound(uniq.begin(), uniq.end(), keys[c * ne + k]);
      cn[c * row + nvc + k] = nv + static_cast<int32_t>(it - uniq.begin());
    }
  }
  return nv + static_cast<int>(uniq.size());
}

// Dof expansion of a node map: out[e][a*dim+d] = map[e][a]*dim + d, the Map a
// vector-valued Mat needs to pass validate (parloop.hpp:119-121).
int loam_gpu_expand_map(int nsrc, int arity, const int32_t* map, int dim, int32_t* out) {
  if (dim < 1) return LOAM_ERR(InvalidArgument);
  for (int64_t e = 0; e < nsrc; ++e)
    for (int a = 0; a < arity; ++a)
      for (int d = 0; d < dim; ++d)
        out[(e * arity + a) * dim + d] = map[e * arity + a] * dim + d;
  return 0;
}

} // extern "C"
