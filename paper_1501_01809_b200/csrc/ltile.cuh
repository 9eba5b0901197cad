// ltile.cuh -- edge-link tiles for vector P1 matrices on tetrahedra (linear
// elasticity, sm_100a).
//
// Same par_loop as ntile.cuh (assemble_matrix(elasticity) on a dof-expanded
// vertex map, fem/assemble.hpp:85-104 -> parloop.hpp:191-384, 12x12 element
// matrices added by Mat::addto, data.hpp:205-222, into the 3x3-blocked pattern
// of build_sparsity, data.hpp:149-179), owner-computes per 3x3 node block
// (v, w), but WITHOUT a per-tile cell table: the cells around the mesh edge
// (v, w) are (v, w, p_i, p_{i+1}) for the vertices p_0, p_1, ... of the edge's
// LINK (a closed ring inside the mesh, an open fan on its boundary).  The
// block's thread walks the link once, reading one vertex position per cell
// from the tile's coordinate window, and forms each cell's contribution
//   V g_v g_w^T = m n^T / (6 |D|),   n = (p - v) x (q - v),  D = (w - v) . n,
//   m = (q - w) x (p - w) = (p - v) x e - (q - v) x e - n,   e = w - v
// in registers (the cross products with e are carried from cell to cell).
// The node tiles were bound by shared-memory wavefronts (a 96-byte cell record
// written per tile cell, two random 24-byte gradient reads per block and
// cell, ncu l1tex data pipe 93 % busy); here a block reads 24 bytes per cell
// and nothing is written to shared memory but the result.  The diagonal block
// is minus the sum of its row's off-diagonal blocks (the barycentric
// gradients of a cell sum to zero), summed in column order.
//
// The plan declines -- the node tiles run instead -- unless every edge's link
// is a single ring or fan (manifold mesh) and the pattern is the (map, map)
// pattern.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct LtilePlan {
  int ntiles = 0, max_seg = 0, max_slots = 0, max_blob = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile (ltile.cu)
  DevBuf<uint8_t> blob;  // per tile: block records, link vertex slots, diagonal records
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
};

struct LtileSpec {
  int tile_nodes = 64, tile_slots = 1024, tile_runs = 32, max_link = 24;
};

// Arguments as build_ntile (ntile.cuh).  False when a link is not a ring or
// fan, the pattern is not the (map, map) pattern's node structure, or a tile
// limit cannot be met.
bool build_ltile(LtilePlan& out, const LtileSpec& sp, int ncells, int nnodes, const int32_t* sorted_rows,
                 const int32_t* sorted_x, int nverts, const PairPlan& pp, const int64_t* row_ptr, int64_t nnz,
                 cudaStream_t s);

void launch_ltile(const LtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s);

} // namespace loam_gpu
