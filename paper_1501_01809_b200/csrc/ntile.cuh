// ntile.cuh -- node-block tiles for vector P1 matrices (linear elasticity, sm_100a).
//
// The par_loop of assemble_matrix(elasticity) on a dof-expanded vertex map
// (fem/assemble.hpp:85-104 -> parloop.hpp:191-384, 12x12 element matrices,
// 3x3-blocked CSR) adds, per cell, 16 node blocks of 3x3 values.  Summed
// through shared-memory read-modify-writes that is 764 M element entries for
// config 4 -- more shared-memory traffic than the SM can move in 1 ms.  Here
// every 3x3 node block (v, w) of the matrix is one ITEM owned by one thread:
// it walks the cells containing both v and w (4-6 for an edge, the 24 cells of
// v for the diagonal, split over 4 threads), reads the cell's barycentric
// gradients g_v, g_w and measure from a per-tile cell table in shared memory,
// accumulates the 9 values in registers and writes each once into the tile's
// contiguous row segment, which one TMA bulk store writes to HBM.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct NtilePlan {
  int ntiles = 0, max_seg = 0, max_cells = 0, max_slots = 0, max_blob = 0, max_diag = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile (ntile.cu)
  DevBuf<uint8_t> blob;  // per tile: item records, pair records, cell vertex slots
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
};

struct NtileSpec {
  int tile_nodes = 12, tile_items = 512, tile_pairs = 4096, tile_cells = 1023, tile_slots = 1024, tile_runs = 32;
};

// From the locality-sorted node map (ncells x 4), the sorted coordinate map,
// the pair plan (node-level ranks) and the Mat's dof-level row offsets (3x3
// blocked).  False when the pattern is not the (map, map) pattern's node
// structure or a tile limit cannot be met.
bool build_ntile(NtilePlan& out, const NtileSpec& sp, int ncells, int nnodes, const int32_t* sorted_rows,
                 const int32_t* sorted_x, int nverts, const PairPlan& pp, const int64_t* row_ptr, int64_t nnz,
                 cudaStream_t s);

void launch_ntile(const NtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s);

} // namespace loam_gpu
