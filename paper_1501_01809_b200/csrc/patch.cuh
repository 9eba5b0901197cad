// patch.cuh -- cell-patch plan for the row-owner kernels k_patch_mat / k_patch_vec.
//
// The reference scatters every staged element tensor into its targets cell by
// cell (parloop.hpp:301-313; Mat::addto data.hpp:205-222).  The patch plan
// re-groups that work so that a CTA computes each cell's geometry ONCE and
// every output row is finished inside one CTA:
//   * cells are ordered along a Morton curve of their centroids (spatially
//     compact runs), and cut into PATCHES of consecutive cells;
//   * each row node is OWNED by the patch of the first cell (in that order)
//     that contains it; a patch's TILE CELLS are all cells incident to its
//     owned rows (its own cells plus a halo of neighbouring cells);
//   * the patch WINDOW is the sorted, de-duplicated list of the tile cells'
//     nodes; a tile cell is stored as NRN u16 window slots.  Because the
//     window is sorted by node id, the in-row rank of a column node -- its
//     position in the CSR row, the reference's Sparsity::find
//     (data.hpp:129-136) -- is a prefix popcount over a per-row bitmap of
//     window slots, computed in shared memory; no col_idx or rank table is
//     read at assembly time.
// Row values are accumulated in shared memory by one thread per owned row in
// a fixed pair order and written once (no zero-fill, no atomics).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "plan.cuh"

namespace loam_gpu {

struct PatchPlan {
  int npatches = 0;
  int nrn = 0;                 // slots per tile cell
  int max_win = 0, max_cells = 0, max_own = 0, max_pairs = 0;
  int64_t max_seg = 0;         // values of a patch's owned rows (matrices)
  int64_t tile_cells = 0, own_rows = 0;
  int64_t untouched = 0;       // nodes in no cell (never written by the kernel)
  bool halo = true;            // false: cell-owned patches (Dats), window ids flag shared nodes
  int64_t boundary = 0;        // (cell-owned) window entries shared with other patches
  DevBuf<int4> hdr;            // 2 per patch: {win_off, nwin, rec_off, ncells}, {own_off, nown, npairs, seg}
  DevBuf<int32_t> win;         // window node ids (each patch's run 16-byte aligned)
  DevBuf<uint16_t> recs;       // per patch [ncells x nrn] window slots (16-byte aligned runs)
  DevBuf<uint16_t> own;        // owned rows as window slots, ascending (cell-owned: per-node incidence offsets)
  DevBuf<int64_t> orp;         // (Mats) CSR offset of each owned row node's first dof row
  DevBuf<int32_t> oseg;        // (Mats) per patch nown+1 value-segment offsets (index own_off + patch)
};

struct PatchSpec {
  int gd = 2, nrn = 3;         // geometry dim, row-map arity
  int rd = 1, cd = 1;          // dof blocking of the Mat (1 for Dats)
  bool bilinear = false;
  int64_t budget = 8192;       // owned values per patch (matrices) / owned rows (Dats)
  int max_cells = 1024;        // tile cells per patch (cell-owned: cells per patch)
  bool halo = true;            // row-owner patches with halo cells (Mats); false: cell-owned (Dats)
};

// Build from the node-level row map (user cell order, device), the coordinate
// map (device) whose rows must equal the first gd+1 entries of the row map,
// and the coordinates (device).  For matrices `row_ptr` is the Mat's dof-row
// CSR offsets (device) whose pattern the caller has checked equals the
// (map, map) pattern.  Returns false when a patch limit cannot be met.
bool build_patch(PatchPlan& out, const PatchSpec& sp, int ncells, int nnodes, const int32_t* rows,
                 const int32_t* xmap, int xstride, const double* coords, const int64_t* row_ptr,
                 cudaStream_t s);

// True when the CSR (row_ptr, col_idx) equals build_sparsity(m, m, rd, cd).
bool pattern_is_map_pattern(const int32_t* m, int n, int arity, int target, int rd, int cd,
                            const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz, cudaStream_t s);
// The same test for a rectangular pattern: build_sparsity(rows, cols, rd, cd).
bool pattern_is_maps_pattern(const MapView& rows, const MapView& cols, int rd, int cd, const int64_t* row_ptr,
                             const int32_t* col_idx, int64_t nnz, cudaStream_t s);

} // namespace loam_gpu
