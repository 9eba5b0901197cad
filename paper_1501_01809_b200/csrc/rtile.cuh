// rtile.cuh -- row tiles with shared cell geometry for mixed-space blocks (sm_100a).
//
// The Taylor-Hood coupling blocks B (pressure rows x velocity columns) and
// B^T (config 5) are not symmetric squares, so the edge-tile transposition of
// etile.cuh does not apply: every row is owner-computed.  A tile is up to NT
// consecutive row nodes, one thread each (lanes sorted by pair count); the
// tile's distinct cells get their barycentric gradients and measure once in
// shared memory; a pair's element row comes from the canonical (permuted)
// geometry through the catalogue row functor (elements.cuh), and is added
// into a lane-interleaved row segment (conflict-free), rebuilt contiguous and
// written with one TMA bulk store.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "elements.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct RtilePlan {
  int form = -1, ntiles = 0, tile_threads = 64;
  int max_seg = 0, max_segT = 0, max_cells = 0, max_slots = 0, max_blob = 0;
  DevBuf<int32_t> tiles; // 16 ints per tile (rtile.cu)
  DevBuf<uint8_t> blob;  // per tile: row offsets, pair counts, lane order, records, cell slots
  DevBuf<int32_t> runs;  // coordinate-window runs [lo, hi)
};

struct RtileSpec {
  int tile_rows = 64, tile_seg = 8192, tile_pairs = 2048, tile_cells = 1023, tile_slots = 1024, tile_runs = 32;
};

// True when `form` has a row-tile kernel (F_STOKES_B, F_STOKES_BT).
bool rtile_form(int form);

// From the locality-sorted row map (ncells x nrn node level), the sorted
// coordinate map, the pair plan with its node-level ranks and the Mat's
// dof-level row offsets (rd x cd blocked).  False when a limit is not met.
bool build_rtile(RtilePlan& out, const RtileSpec& sp, int form, int gd, int nrn, int ncn, int rd, int cd,
                 int ncells, int nrows_node, const int32_t* sorted_rows, const int32_t* sorted_x, int nverts,
                 const PairPlan& pp, const int64_t* row_ptr, int64_t nnz, cudaStream_t s);

void launch_rtile(const RtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s);

} // namespace loam_gpu
