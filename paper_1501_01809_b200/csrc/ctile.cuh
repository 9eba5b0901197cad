// ctile.cuh -- cell tiles for P2 actions (the config-3 residual, sm_100a).
//
// The par_loop of assemble_vector(helmholtz action, P2) (fem/assemble.hpp:
// 108-135 -> parloop.hpp:191-384) computes, per cell, a 10-entry element
// vector from the cell's 4 vertex coordinates and 10 coefficient values and
// INC-scatters it (parloop.hpp:301-308).  The cell-centric kernel gathers
// those 14 values per cell with dependent scattered loads and issues one fp64
// RED per entry: latency-bound on the gathers and on the L2 atomic units
// (15.7 M REDs for config 3).  Here consecutive (locality-sorted) cells form
// a tile whose unique nodes and vertices arrive as TMA bulk copies of id runs
// (no consumer-side gathers); every cell's element vector goes to shared
// memory, and each distinct node of the tile sums its entries there (fixed
// order) and issues ONE RED -- about a third of the REDs.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"

namespace loam_gpu {

struct CtilePlan {
  int ntiles = 0, nrn = 0, nv = 0, max_blob = 0, max_xslots = 0, max_cslots = 0, tile_cells = 256;
  DevBuf<int32_t> tiles; // 16 ints per tile (ctile.cu)
  DevBuf<uint8_t> blob;  // per tile: vertex slots, node slots, per-slot entry lists, node runs
  DevBuf<int32_t> xruns; // coordinate-window runs [lo, hi)
  DevBuf<int32_t> cruns; // coefficient-window runs [lo, hi)
};

// From the locality-sorted node map (ncells x nrn, the first gd+1 entries of a
// row are the cell's vertices = coordinate ids).  False when a tile limit
// cannot be met (the caller keeps the cell-centric kernel).
bool build_ctile(CtilePlan& out, int gd, int nrn, int ncells, const int32_t* sorted_rows, int nnodes, int nverts,
                 cudaStream_t s);

// One action assembly: out (nnodes, zeroed here unless accumulate) += the
// element vectors of form F (F_MASS_ACTION / F_STIFFNESS_ACTION /
// F_HELMHOLTZ_ACTION, P2).
void launch_ctile(int form, const CtilePlan& p, const double* coords, const double* coeff, double* out,
                  int64_t nout, const FormParams& prm, bool accumulate, int* next_tile, int* reset_tile,
                  cudaStream_t s);

} // namespace loam_gpu
