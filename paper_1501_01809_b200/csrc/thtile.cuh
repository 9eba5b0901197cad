// thtile.cuh -- the three Taylor-Hood Stokes blocks in ONE launch (sm_100a).
//
// Reference path replaced: fem::assemble_blocks (fem/assemble.hpp:439-448)
// over the nested 2x2 BlockMat of solver.hpp:21-28 -- three par_loops
// (parloop.hpp:191-384) with the element kernels restated in elements.cuh
// (FormT<F_STOKES_A / _B / _BT>), each adding its element matrices with
// Mat::addto (data.hpp:205-222) into its own pattern from build_sparsity
// (data.hpp:149-179):
//   A   (velocity dofs x velocity dofs, 2x2 component blocks)
//   B   (pressure vertices x velocity dofs)
//   B^T (velocity dofs x pressure vertices)
// Run one after the other they read the maps and coordinates three times and
// recompute every cell's geometry per block.  Here every ROW of all three
// matrices is owner-computed from vertex positions alone, by items that are
// mesh edges with their (at most two) cells:
//   * an EDGE item (v, w | p, q) owns velocity edge node e = (v, w): its two A
//     rows (9 column nodes: v, w, p, q, e, (v,p), (w,p), (v,q), (w,q)) and its
//     two B^T rows (pressure columns v, w, p, q);
//   * a SPOKE item (v -> w | p, q) of vertex v owns the columns of v's rows
//     that carry w: A[v][w], A[v][(v,w)], A[v][(w,p)], the same three node
//     columns of pressure row B[v] and B^T[(v,.)][w]; the spokes of a vertex
//     follow its star (ring or fan), each owning the cell on its p side, whose
//     share of the (v, v) entries goes through a per-item scratch slot and is
//     summed per vertex in spoke order (fixed: the path is deterministic).
// A cell's geometry is formed in registers from three positions of the tile's
// TMA-staged coordinate window and serves the A, B and B^T entries at once;
// every value is written exactly once into the tile's three contiguous row
// segments in shared memory, which three TMA bulk stores write out.
//
// The plan declines -- the three loops then run one by one -- unless the
// velocity map is a P2 map over the coordinate map (vertex nodes first and
// equal to the vertex ids, edge node <-> vertex pair a bijection), pressure
// nodes are the vertices, every vertex star is one ring or fan, every edge has
// one or two cells, and the three patterns are exactly the (map, map) patterns.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct ThtilePlan {
  int ntiles = 0, max_seg = 0, max_slots = 0, max_blob = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile: 8 meta + the first 4 window runs (thtile.cu)
  DevBuf<uint8_t> blob;  // per tile: item window slots, item records, vertex records
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
};

struct ThtileSpec {
  int spoke_items = 128, edge_items = 64, tile_slots = 1024, tile_runs = 32;
};

// vnm: the velocity cell->node map (ncells x 6, device), xmap: the cell->vertex
// coordinate map (ncells x 3, device), pp: build_pairs(vnm) (node -> (cell, local)),
// rpA / rpB / rpT: the row offsets of the three patterns (device).
bool build_thtile(ThtilePlan& out, const ThtileSpec& sp, int ncells, int nnodes, int nverts, const int32_t* vnm,
                  const int32_t* xmap, const PairPlan& pp, const int64_t* rpA, int64_t nnzA, const int64_t* rpB,
                  int64_t nnzB, const int64_t* rpT, int64_t nnzT, cudaStream_t s);

// acc: bit 0 / 1 / 2 = add to the existing values of A / B / B^T instead of overwriting
void launch_thtile(const ThtilePlan& p, const double* coords, double* A, double* B, double* BT, double nu, int acc,
                   cudaStream_t s);

} // namespace loam_gpu
