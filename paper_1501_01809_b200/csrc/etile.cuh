// etile.cuh -- edge-tile assembly of scalar P2 matrices (sm_100a).
//
// The par_loop of assemble_matrix(mass|stiffness|helmholtz, P2)
// (fem/assemble.hpp:85-104 -> parloop.hpp:191-384) scatters, per cell, a
// 10x10 (tets) / 6x6 (triangles) element matrix into the CSR values.  The
// catalogue forms are symmetric and a P2 map has two node roles -- vertex
// nodes (local 0..d) and edge nodes (local d+1..) -- and every vertex-node pair
// sharing a cell is the endpoint pair of exactly one edge node whose cells
// are exactly the cells containing both vertices.  So every entry of the
// matrix can be produced by the EDGE rows alone:
//   * edge row e: owner-computes over e's cells (4-6 in 3D), in a shared
//     segment, written once;
//   * vertex row v, edge column e: A[v][e] = A[e][v] -- written (transposed)
//     by edge row e;
//   * vertex row v, vertex column w != v: the (v,w) element entries of the
//     cells of the edge node (v,w) -- summed and written by that edge row;
//   * vertex diagonal A[v][v]: each (cell, vertex) contribution is assigned
//     to one edge of the cell and RED-added by that edge row (the diagonal
//     is zeroed first).
// Edge tiles share cell geometry: the tile's distinct cells (0.4 per pair on
// the Kuhn meshes) get their barycentric-gradient Gram matrix V g_p.g_q once,
// in shared memory; a pair's element row is then ~40 FMAs of those values.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct EtilePlan {
  int gd = 3, cd = 1, ntiles = 0, e0 = 0, nedge = 0, rec_bytes = 0, tile_threads = 128;
  bool compact = false; // 5-bit ranks, per-row constant ranks (rows <= 32 entries)
  int max_rows = 0, max_seg = 0, max_segT = 0, max_cells = 0, max_slots = 0, max_blob = 0;
  int64_t ndiag = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile (etile.cu)
  // per tile, 16-byte aligned sections (one TMA copy): segment offsets u16,
  // transposed-entry offsets u16, pair counts u8 + per-warp (segment base,
  // record base) u16, per row pos(A,B) / pos(B,A) / diag(A) / diag(B) (int4),
  // the value positions (in vertex rows) of the rows' vertex columns (int32),
  // lane-interleaved pair records, cell vertex slots (u16)
  DevBuf<uint8_t> blob;
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
  DevBuf<int32_t> diag;  // diagonal positions of the vertex rows (+ dof row length when cd = 2)
  uint32_t ktab[12] = {};
  // deterministic mode: the edge rows store their diagonal partial sums in
  // slots (2 e + endpoint) instead of RED-adding them; diagonal d (in `diag`
  // order) sums slots dslots[dptr[d] .. dptr[d + 1]) in that (edge-ascending)
  // order
  bool det = false;
  DevBuf<int32_t> dptr, dslots;
};

struct EtileSpec {
  int tile_rows = 128; // 64 or 128: consumer threads per CTA, one edge row each
  int tile_seg = 4096, tile_pairs = 1024, tile_cells = 512, tile_slots = 768, tile_runs = 32;
  bool det = false; // deterministic diagonals (EtilePlan::det)
};

// Builds the plan from the locality-sorted row map (ncells x nrn, P2), the
// sorted coordinate map (ncells x (gd+1)), the pair plan with its slot ranks
// and the Mat's row offsets.  Returns false when the structure does not hold
// (node roles, edge <-> vertex-pair bijection, vertex nodes numbered first,
// nnz < 2^31) or a tile limit cannot be met; the caller then uses another plan.
bool build_etile(EtilePlan& out, const EtileSpec& sp, int gd, int ncells, int nrows_node,
                 const int32_t* sorted_rows, const int32_t* sorted_x, int nverts, const PairPlan& pp,
                 const int64_t* row_ptr, int64_t nnz, int cd, cudaStream_t s);

// cd = 2: the Mat is the component-diagonal 2-vector expansion of the scalar
// form (Taylor-Hood velocity block nu grad u : grad v, elements.cuh F_STOKES_A):
// dof entry (2i+d, 2j+c) = delta_dc K_ij on a 2x2-blocked pattern.
//
// One assembly through the plan (form: F_MASS / F_STIFFNESS / F_HELMHOLTZ /
// F_STOKES_A).
void launch_etile(int form, const EtilePlan& p, const double* coords, double* out, const FormParams& prm,
                  bool accumulate, int* next_tile, int* reset_tile, cudaStream_t s);

} // namespace loam_gpu
