// plan.cuh -- execution plans for the par_loop engine (built on the device, cached).
//
// The reference caches one thing per (iteration set, conflict maps): the greedy
// colouring (parloop.hpp:153-168).  The B200 engine caches, per loop shape,
//   * a cell LOCALITY order (cells sorted by their smallest row node) and the
//     maps re-laid in that order, so every gather is coalesced/L2-resident;
//   * the owner-computes PAIR list: for each row node, the (cell, local index)
//     pairs incident to it (the node->cell inverse of the row map);
//   * for Mats, the per-pair SLOT RANKS: the in-row position of each column
//     node -- the "precomputed per-cell slot offsets into col_idx" of the
//     north star, compressed to one byte per entry -- and the warp chunking
//     of rows into shared-memory segments;
//   * the bit-exact greedy COLOURING (topology.hpp:86-125), when a loop or a
//     strategy needs it.
#pragma once
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace loam_gpu {

struct MapView {         // device map, row-major [n x arity]
  const int32_t* v = nullptr;
  int n = 0, arity = 0, target = 0;
};

struct CsrView {         // device CSR (data.hpp:116-142) with its dof expansion
  const int64_t* row_ptr = nullptr;
  const int32_t* col_idx = nullptr;
  int nrows = 0, ncols = 0;
  int64_t nnz = 0;
  int rd = 1, cd = 1;
};

struct LocalityPlan {
  DevBuf<int32_t> perm; // sorted position -> user cell
  int n = 0;
};

struct SortedMap {
  DevBuf<int32_t> v;    // rows of a map in locality order
  int arity = 0, target = 0;
};

struct PairPlan {
  int nrows_node = 0, nrn = 0, ncn = 0;
  int64_t npairs = 0;
  DevBuf<int32_t> ptr;   // [nrows_node + 1]
  DevBuf<int32_t> pairs; // sorted_cell * nrn + i, grouped by row node
  DevBuf<uint8_t> ranks; // [npairs * ncn] in-row node rank of each column node
  // warp chunks of consecutive row nodes whose value segment fits in smem
  DevBuf<int32_t> chunk_row; // [nchunks + 1]
  int nchunks = 0, seg_max = 0;
};

struct ColorPlan {
  DevBuf<int32_t> colors; // per user entity (bit-exact with the reference)
  DevBuf<int32_t> order;  // entities sorted by (colour, index)
  std::vector<int> offsets; // host: colour c is order[offsets[c] .. offsets[c+1])
  int ncolors = 0;
};

// Locality order: cells sorted (stably) by the smallest node of `key`.
void build_locality(const MapView& key, LocalityPlan& out, cudaStream_t s);
// out[p] = m[perm[p]] row by row.
void gather_rows(const MapView& m, const int32_t* perm, SortedMap& out, cudaStream_t s);
// Pair list of a (sorted) node-level row map.
void build_pairs(const int32_t* sorted_rows, int ncells, int nrn, int nrows_node, PairPlan& out,
                 cudaStream_t s);
// Slot ranks of the column nodes of each pair in its row (throws OutsideSparsity);
// verifies the pattern is blocked by (rd, cd) first.
// Scatter the pair plan's ranks (pair order) to cell-major order:
// out[(cell * nrn + i) * ncn + j] = pp.ranks[p * ncn + j] for pair p = (cell, i).
void cell_major_ranks(const PairPlan& pp, DevBuf<uint8_t>& out, cudaStream_t s);
void build_ranks(PairPlan& pp, const int32_t* sorted_rows, const int32_t* sorted_cols, int ncn,
                 const CsrView& csr, cudaStream_t s);
// Warp chunking of row nodes (<= max_rows nodes, segment <= smax doubles).
void build_chunks(PairPlan& pp, const CsrView& csr, int smax, int max_rows, cudaStream_t s);

// Neighbour-list plan (P1 forms whose row, column and coordinate maps are the
// same node map): the node-level pattern N(r) of every row is the list of
// cell-neighbour nodes, so a pair needs only (local index | in-row ranks of the
// cell's nodes) -- a 16/32-bit record -- and the kernel gathers each chunk's
// neighbour coordinates once instead of per pair.
constexpr int kRingInlineRuns = 4; // window runs stored inside a ring tile record

struct NbrPlan {
  int nrows_node = 0, nrn = 0, bits = 0, rec_bytes = 4, rd = 1, cd = 1;
  // plan-owned, 16-byte padded arrays; the tile kernel TMA-loads tile ranges of them
  DevBuf<int32_t> nptr;  // node-level pattern offsets [nrows_node + 1]
  DevBuf<int32_t> pptr;  // pair offsets per row [nrows_node + 1]
  DevBuf<uint8_t> recs;  // npairs records: in-row ranks of the cell's other vertices
  DevBuf<uint16_t> widx; // per pattern entry: slot of its node in the tile's vertex window
  DevBuf<uint8_t> selfr; // per row: rank of the row node in its own pattern row
  DevBuf<int32_t> runs;  // per tile: contiguous vertex runs [lo, hi) (lo, hi even or hi = nv)
  // CTA tiles of consecutive rows: {R0, R1, A0, A1, P0, P1, run_off, run_cnt}
  DevBuf<int32_t> tiles;
  int ntiles = 0;
  int max_rows = 0, max_adj = 0, max_pairs = 0, max_seg = 0, max_slots = 0, max_runs = 0; // per tile
  int max_len = 0; // longest node row
  // RING mode (P1 triangles on a manifold mesh): the cells around each row
  // vertex ordered along their ring / fan, one 16-bit record per chain vertex
  // (window slot << 3 | in-row rank), P+1 records per row (head first)
  bool ring = false;
  DevBuf<int32_t> rptr;      // [nrows_node + 1] record offsets (pptr[r] + r)
  DevBuf<uint16_t> rrecs;    // chain records
  DevBuf<uint32_t> rowinfo;  // self window slot | self rank << 16
  DevBuf<int32_t> rtiles;    // 16-int ring tiles: P0/P1 in ring-record units + inline runs
};
// Build from a (sorted) node-level map and a node-level pattern.  For Mats the
// pattern is the Mat's sparsity (csr, possibly blocked by rd/cd); for Dats
// csr.row_ptr == nullptr and the pattern of (map, map) is built here.
// Returns false when a row is too long for the packed record.
// Tiles hold <= tile_rows row nodes, <= tile_seg matrix values and a vertex
// window of <= tile_slots vertices in <= tile_runs contiguous runs.
bool build_nbr(NbrPlan& np, const int32_t* sorted_rows, int ncells, int nrn, int nrows_node,
               const CsrView& csr, int tile_rows, int tile_seg, int tile_slots, int tile_runs,
               cudaStream_t s);

// The ring mode of the neighbour plan built on the device (scalar P1 triangle
// Mats, tiles of exactly tile_rows rows): false when a tile or a row needs the
// host builder (build_nbr), which the caller then runs.
bool build_ring_dev(NbrPlan& np, const int32_t* sorted_rows, int ncells, int nrows_node, const CsrView& csr,
                    int tile_rows, int tile_seg, int tile_slots, cudaStream_t s);

// Canonical pair-tile plan (any catalogue form on simplices).  Each pair
// (row node r, cell e) is stored with the cell's local numbering PERMUTED so
// that r is a canonical local node (vertex rows: local vertex 0; P2 edge rows:
// the first local edge), making the element row a compile-time index.  Record
// (rec_bytes each): u16 window slots of the permuted vertices [GD+1], then
// u16 coefficient window slots [NCOEFF] (actions), then u8 in-row ranks of the
// permuted column nodes [NCN] (matrices), then u8 canonical index.
struct PTilePlan {
  int nrows_node = 0, rec_bytes = 0, ntiles = 0;
  int max_rows = 0, max_pairs = 0, max_seg = 0, max_slots = 0, max_cslots = 0;
  DevBuf<int32_t> pptr;   // pair offsets per row [nrows_node + 1] (+pad)
  DevBuf<int32_t> nptr;   // node-level pattern offsets [nrows_node + 1] (+pad)
  DevBuf<uint8_t> recs;   // npairs * rec_bytes (+pad)
  DevBuf<int32_t> runs;   // coordinate-window runs
  DevBuf<int32_t> cruns;  // coefficient-window runs
  DevBuf<int32_t> tiles;  // 12 ints per tile: R0,R1,A0,A1,P0,P1,run_off,run_cnt,crun_off,crun_cnt,0,0
};
struct PTileSpec {
  int gd = 2, nrn = 3, ncn = 0, ncoeff = 0, rd = 1, cd = 1;
  int tile_rows = 128, tile_seg = 4096, tile_pairs = 2048, tile_slots = 1024, tile_runs = 48;
};
// sorted_* are node-level maps in the locality order; pp holds the pairs and
// (for matrices) the ranks of the column nodes; csr the Mat pattern (matrices).
// Returns false when a tile limit cannot be met (caller falls back).
// Canonical local numbering of a pair (plan.cu): sigma[old vertex] = new vertex
// making row-space local node i canonical (vertex rows: local vertex 0; P2
// edge rows: the first local edge); returns the canonical local index (0 or
// gd+1).  induced() maps old local nodes (nloc of them, P1 or P2) to new.
int canonical_sigma(int gd, int nrn, int i, int* sigma);
void induced(int gd, int nloc, const int* sigma, int* newpos);

bool build_ptile(PTilePlan& out, const PTileSpec& sp, int ncells, int nrows_node, const int32_t* sorted_rows,
                 const int32_t* sorted_cols, const int32_t* sorted_x, int nverts, const int32_t* sorted_coeff,
                 int ncoeff_nodes, const PairPlan& pp, const CsrView& csr, cudaStream_t s);

// build_sparsity (data.hpp:149-179) on the device, bit-exact.
void build_sparsity_dev(const MapView& rows, const MapView& cols, int rd, int cd,
                        int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, cudaStream_t s);
// color_iteration (topology.hpp:86-125) on the device, bit-exact.
void color_dev(int n, const std::vector<MapView>& maps, ColorPlan& out, cudaStream_t s);

} // namespace loam_gpu
