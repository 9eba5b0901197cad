// wtile.cuh -- link-walk tiles for scalar P2 matrices on tetrahedra (sm_100a).
//
// Same par_loop as etile.cuh: assemble_matrix(mass / stiffness / helmholtz) on
// a P2 tetrahedral space (fem/assemble.hpp:85-104 -> parloop.hpp:191-384, 10x10
// element matrices added by Mat::addto, data.hpp:205-222, into the pattern of
// build_sparsity(map, map), data.hpp:149-179), with the same division of the
// matrix -- every EDGE row is owner-computed and carries the vertex rows by
// symmetry (A[u][e] = A[e][u] stored at a planned position; A[v][w] summed by
// the edge row (v, w); vertex diagonals RED-added by the edge that owns each
// (cell, vertex) share) -- but WITHOUT the edge tiles' per-tile cell tables:
// the cells of edge node e = (v, w) are (v, w, p_i, p_{i+1}) for the vertices
// p_0, p_1, ... of the edge's LINK (ring or fan, as ltile.cuh), so the row's
// thread walks the link once, reads one vertex position per cell from the
// tile's TMA-staged coordinate window, forms the cell's geometry and its
// element row (the catalogue functor FormT<FORM, 3, 2>::row for the canonical
// cell (v, w, p_i, p_{i+1}), local edge (0, 1)) in registers and carries the
// partial sums of the columns two consecutive cells share (p, (v,p), (w,p)).
// Every entry of the row is written once into the tile's segment: no Gram
// table, no pair records, no read-modify-write, no lane-interleaved segment
// to rebuild.
//
// The plan declines -- the edge tiles run instead -- unless the structure of
// etile.cuh holds and every edge's link is one ring or fan.  In deterministic
// mode the diagonal shares go to per-(edge, endpoint) slots that a second
// kernel sums per vertex in edge order instead of by RED.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct WtilePlan {
  int ntiles = 0, max_seg = 0, max_slots = 0, max_blob = 0, nverts = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile (wtile.cu)
  DevBuf<uint8_t> blob;  // per tile: row headers, link slots, in-row ranks, transposed positions
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
  DevBuf<int32_t> dpos;  // position of every vertex diagonal (zeroed before a fresh assembly)
  // deterministic mode: the edge rows store their diagonal shares in slots
  // 2 (e - nverts) + endpoint and k_wt_dsum sums vertex v over dslots[dptr[v] .. dptr[v + 1])
  bool det = false;
  int nedges = 0;
  DevBuf<int32_t> dptr, dslots;
};

struct WtileSpec {
  int tile_rows = 128, tile_slots = 1024, tile_runs = 32, max_link = 12;
  bool det = false; // deterministic diagonals (WtilePlan::det)
};

// rows / xmap: the (locality-sorted) P2 cell->node map (ncells x 10) and
// cell->vertex map (ncells x 4), pp: build_pairs(rows), row_ptr / col_idx: the
// Mat's pattern (device).
bool build_wtile(WtilePlan& out, const WtileSpec& sp, int ncells, int nnodes, int nverts, const int32_t* rows,
                 const int32_t* xmap, const PairPlan& pp, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                 cudaStream_t s);

void launch_wtile(const WtilePlan& p, int form, const double* coords, double* out, const FormParams& prm,
                  bool accumulate, int* next_tile, int* reset_tile, cudaStream_t s);

} // namespace loam_gpu
