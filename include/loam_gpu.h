/*
 * loam_gpu.h -- C ABI of the B200-native par_loop engine (drop-in boundary).
 *
 * The reference (`loam`, C++20 header-only, /root/reference/proj/include/loam)
 * has no FFI; its operator surface is the C++ API
 *     void loam::execute(const Parloop&, int threads)          parloop.hpp:191
 *     SparsityPtr loam::build_sparsity(row, col, rdim, cdim)   data.hpp:149
 *     Coloring loam::color_iteration(iter, conflict_maps)      topology.hpp:86
 *     void loam::validate(const Parloop&)                      parloop.hpp:89
 * over Set/Map/Dat/Mat/Global/Arg objects (topology.hpp:15-74,
 * data.hpp:15-234, parloop.hpp:17-59).  This header is exactly what an FFI
 * binding of those entry points needs: plain descriptors (POD, device
 * pointers, sizes, identities) and int error codes.  The C++ facade
 * paper_1501_01809_b200/csrc/loam_gpu.hpp restores the reference's class API
 * on top of it; INTEGRATION.md shows the ctypes and C++ bindings.
 *
 * Conventions
 *   - Every function returns 0 on success or LOAM_ERR(kind) = 1 + the
 *     loam::ErrorKind value (common.hpp:10-33); LOAM_GPU_ERR_CUDA reports a
 *     CUDA runtime failure.  loam_gpu_last_error() returns a thread-local
 *     message (the reference's Error::what()).
 *   - Pointers in descriptors are DEVICE pointers borrowed for the call
 *     ("execute borrows everything for its duration"); the
 *     library never frees caller memory.  The *_host variants take host
 *     pointers and stage the copies themselves.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered; loam_gpu_execute returns after enqueueing unless the
 *     kernel reports a device-side error (OutsideSparsity), which needs a
 *     sync: see LOAM_OPT_CHECK_SPARSITY.
 *   - No CPU fallback: without a usable sm_100 device every compute entry
 *     point fails with LOAM_GPU_ERR_NO_DEVICE.
 */
#ifndef LOAM_GPU_H
#define LOAM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* loam::ErrorKind (common.hpp:10-33), same order. */
enum loam_error_kind {
  LOAM_KIND_IndexOutOfRange = 0,
  LOAM_KIND_ArityMismatch,
  LOAM_KIND_SourceMismatch,
  LOAM_KIND_AsymmetricAdjacency,
  LOAM_KIND_IllegalAccess,
  LOAM_KIND_MapSourceMismatch,
  LOAM_KIND_ShapeMismatch,
  LOAM_KIND_UnboundIdentifier,
  LOAM_KIND_NonDividingFactor,
  LOAM_KIND_OutsideSparsity,
  LOAM_KIND_EmptyPartials,
  LOAM_KIND_DimensionMismatch,
  LOAM_KIND_InvalidSubdivision,
  LOAM_KIND_ParseError,
  LOAM_KIND_NonManifold,
  LOAM_KIND_CellMismatch,
  LOAM_KIND_UnsupportedForm,
  LOAM_KIND_MissingDiagonal,
  LOAM_KIND_SpaceMismatch,
  LOAM_KIND_IndefiniteBreakdown,
  LOAM_KIND_InstabilityDetected,
  LOAM_KIND_InvalidArgument
};
#define LOAM_ERR(kind) (1 + LOAM_KIND_##kind)
#define LOAM_GPU_ERR_CUDA 100      /* CUDA runtime error (message has details) */
#define LOAM_GPU_ERR_NO_DEVICE 101 /* no usable sm_100 device: no CPU fallback */

/* loam::Access (data.hpp:17), same order. */
enum loam_access { LOAM_READ = 0, LOAM_WRITE, LOAM_RW, LOAM_INC, LOAM_SUM, LOAM_MIN, LOAM_MAX };

enum loam_arg_kind { LOAM_ARG_DAT = 0, LOAM_ARG_MAT = 1, LOAM_ARG_GLOBAL = 2 };

/* loam::Map (topology.hpp:36-66): int32 row-major [source_size x arity].
 * `id` identifies the map object (the reference compares MapPtr identity);
 * plans (colourings, inverse maps, slot ranks) are cached per id exactly like
 * the reference's colouring cache (parloop.hpp:153-168).  id 0 = uncached.
 * A dof-expanded map (entries dim*n+d, what a vector Mat needs)
 * may declare its node map in `node_values`/`node_arity`/`node_target_size`
 * with `expand_dim` = dim so the device reads the 1/dim-size node map. */
typedef struct loam_map_desc {
  const int32_t* values;
  int32_t source_size, target_size, arity;
  uint64_t source_id, target_id, id;
  int32_t expand_dim; /* 0 or 1: plain map */
  const int32_t* node_values;
  int32_t node_arity, node_target_size;
  uint64_t node_id;   /* identity of the declared node map (0 = unknown) */
} loam_map_desc;

/* loam::Sparsity (data.hpp:116-142): CSR, int64 row offsets, int32 columns. */
typedef struct loam_sparsity_desc {
  const int64_t* row_ptr; /* [nrows+1] */
  const int32_t* col_idx; /* [nnz]     */
  int32_t nrows, ncols;
  int64_t nnz;
  int32_t row_dim, col_dim; /* dof expansion the pattern was built with (>=1) */
  uint64_t id;
  /* Provenance: the NODE-level maps the pattern was built from (the ids of
   * build_sparsity's row / column maps, or of the node maps a dof-expanded map
   * declares) and the dof dims at that level; 0 = unknown.  A loop whose
   * (row, column) maps are exactly these has exactly this pattern, so an
   * owner-computes kernel may write a fresh Mat's rows without zero-filling
   * them first.  Any other loop -- a sub-mesh loop into a whole-mesh pattern
   * (legal: parloop.hpp:119-121 compares shapes only) -- may touch only part
   * of the pattern: the library then zero-fills a fresh Mat before the loop
   * (data.hpp:185-187: untouched entries stay zero). */
  uint64_t pattern_row_map, pattern_col_map;
  int32_t pattern_row_dim, pattern_col_dim;
} loam_sparsity_desc;

/* loam::Arg (parloop.hpp:17-52) over a Dat, Mat or Global. */
typedef struct loam_arg_desc {
  int32_t kind;   /* loam_arg_kind */
  int32_t access; /* loam_access   */
  double* data;   /* Dat [set_size*dim] | Global [dim] | Mat values [nnz] */
  int32_t dim;    /* Dat / Global dim (Mat: ignored) */
  int32_t set_size;
  uint64_t set_id;  /* Dat's Set identity (direct args must match the iteration set) */
  uint64_t obj_id;  /* object identity for the written-alias check (parloop.hpp:131-137) */
  const loam_map_desc* map;     /* Dat: indirection or NULL (direct); Mat: row map */
  const loam_map_desc* col_map; /* Mat column map */
  const loam_sparsity_desc* sparsity; /* Mat pattern */
  int32_t flags;  /* LOAM_ARG_ZERO: treat the target as freshly zero-initialised
                     (make_dat/make_mat zero-fill, data.hpp:37-39,185-187, or
                     zero()); its current contents are ignored.  The library
                     zero-fills it only when the chosen path needs zeros (atomic /
                     colour scatter); owner-computes writes every entry once. */
} loam_arg_desc;
#define LOAM_ARG_ZERO 1

/* loam::ir::Kernel (kernel.hpp:504-511) as a registry key.  The reference
 * bakes literals (helmholtz kappa, ...) into the kernel AST; here they are
 * `params`.  An unregistered name is an error: there is no CPU fallback. */
typedef struct loam_kernel_desc {
  const char* name;
  const double* params;
  int32_t nparams;
} loam_kernel_desc;

/* ---- library ------------------------------------------------------------- */
const char* loam_gpu_last_error(void);
const char* loam_gpu_version(void);
int loam_gpu_device_ok(void); /* 1 when an sm_100 device is usable */

/* Tunables.  LOAM_OPT_INC_STRATEGY selects the indirect INC scatter:
 *   0 auto (owner-computes; cell-centric atomics for P2-tet actions),
 *   1 fp64 atomics (catalogue forms: one thread per cell, one RED per entry
 *     at a precomputed slot; other kernels: the staging engine),
 *   2 owner-computes row gather (pair lists),
 *   3 colouring (colour-major launches, plain read-modify-write),
 *   4 owner-computes neighbour-list tiles (P1 forms),
 *   5 warp-aggregated fp64 atomics (as 1, lanes hitting one address combine
 *     in the warp first).
 * LOAM_OPT_CHECK_SPARSITY: 1 (default) = a Mat INC/WRITE synchronises once to
 *   report OutsideSparsity like Mat::addto (data.hpp:214-216); 0 = the check
 *   is done only when the slot plan is built (plans prove the pattern).
 * LOAM_OPT_LOCALITY: 1 (default) = renumber cells internally for locality.
 * LOAM_OPT_TEST_KERNELS: 1 = also register the kernels the reference's own
 *   test suite builds (add_one, ones_block, double_direct, ...: test_parloop.cpp,
 *   test_data.cpp); 0 (default) = the product registry only.
 * LOAM_OPT_DETERMINISTIC: 1 = every scatter path is bitwise reproducible run
 *   to run (no fp64 atomics whose order varies: the reference's guarantee,
 *   parloop.hpp:182-190); 0 (default) = the fastest path per form, which may
 *   sum some entries with fp64 REDs (results differ in the last bits between
 *   runs, within 1e-12 of the reference).  Changing it clears the plan cache. */
enum loam_option { LOAM_OPT_INC_STRATEGY = 0, LOAM_OPT_CHECK_SPARSITY = 1, LOAM_OPT_LOCALITY = 2,
                   LOAM_OPT_TEST_KERNELS = 3, LOAM_OPT_DETERMINISTIC = 4 };
int loam_gpu_set_option(int option, int value);
int loam_gpu_get_option(int option);
int loam_gpu_plan_cache_clear(void);
/* Object identities.  Plans (colourings, pair lists, tiles) and the resident
 * host-call copies are cached by the ids in the descriptors, so ids must be
 * unique per process across every client (C++ facade, Python mirror, FFI
 * bindings): take them from loam_gpu_new_id().  loam_gpu_release_id(id)
 * evicts every cached plan and resident copy keyed by `id` (call it when a
 * Map or Sparsity is destroyed). */
uint64_t loam_gpu_new_id(void);
int loam_gpu_release_id(uint64_t id);
/* Number of kernels this library launched since load (bench gpu_launches). */
int64_t loam_gpu_launch_count(void);

/* ---- kernel registry ----------------------------------------------------- */
/* Staged parameter extents of a registered kernel (kernel.hpp:176-186 Param),
 * flattened: for each param, rank then extents.  Returns the param count or
 * -error.  `buf` holds at most `cap` ints. */
int loam_gpu_kernel_signature(const char* name, int32_t* buf, int cap);
/* Newline-separated registered kernel names (static storage). */
const char* loam_gpu_kernel_names(void);

/* ---- the operator -------------------------------------------------------- */
/* loam::validate (parloop.hpp:89-146): checks descriptors only. */
int loam_gpu_validate(const loam_kernel_desc* kernel, int32_t iterset_size, uint64_t iterset_id,
                      const loam_arg_desc* args, int nargs);
/* loam::execute (parloop.hpp:191-384) on device data. */
int loam_gpu_execute(const loam_kernel_desc* kernel, int32_t iterset_size, uint64_t iterset_id,
                     const loam_arg_desc* args, int nargs, void* stream);
/* loam::execute on HOST data (every pointer in args/maps/sparsity is host
 * memory, ideally pinned): uploads what the loop reads, runs, downloads what
 * it writes, synchronously -- the reference's host-memory calling convention.
 * Maps and Sparsities are immutable in the reference (shared_ptr<const Map>,
 * a Sparsity is never modified after build_sparsity): those with a nonzero
 * id are uploaded once per (id, host pointer, size) and kept resident;
 * Dats are copied on every call.  loam_gpu_plan_cache_clear() drops the
 * resident copies. */
int loam_gpu_execute_host(const loam_kernel_desc* kernel, int32_t iterset_size,
                          uint64_t iterset_id, const loam_arg_desc* args, int nargs,
                          void* stream);

/* nsteps independent executions of one loop (same kernel, iteration set,
 * maps and sparsity; args[k] is step k's argument array over its own host
 * Dat / Mat buffers).  Same per-step semantics and transfers as
 * loam_gpu_execute_host -- every step uploads what it reads and downloads
 * what it writes -- but the steps are pipelined: step k+1's host->device
 * copies run on one copy engine while step k's device->host copies run on
 * the other (two device buffer sets), kernels in order on `stream`.
 * Returns when every step's results are in host memory.  An extension (the
 * reference executes one loop per call); a time-stepping or multi-RHS caller
 * uses it to keep both PCIe directions busy. */
int loam_gpu_execute_host_batch(const loam_kernel_desc* kernel, int32_t iterset_size,
                                uint64_t iterset_id, const loam_arg_desc* const* args, int nargs,
                                int nsteps, void* stream);

/* fem::assemble_blocks (fem/assemble.hpp:439-448) assembles the blocks of a
 * nested BlockMat (solver.hpp:21-28) with one par_loop per block.  This entry
 * takes those loops together (device data, as loam_gpu_execute): every loop is
 * validated before anything is written, then the loops run in order -- except
 * that the Taylor-Hood Stokes triple (stokes_a_p2_tri, stokes_b_p2_tri,
 * stokes_bt_p2_tri over one cell set, velocity map, pressure map and
 * coordinate Dat) is assembled by ONE launch that forms every cell's geometry
 * once for the three blocks.  Results are those of the separate loops (values
 * to rounding; the fused path is deterministic run to run). */
typedef struct loam_loop_desc {
  const loam_kernel_desc* kernel;
  int32_t iterset_size;
  uint64_t iterset_id;
  const loam_arg_desc* args;
  int32_t nargs;
} loam_loop_desc;
int loam_gpu_execute_blocks(const loam_loop_desc* loops, int nloops, void* stream);
/* The same over HOST data (the calling convention of loam_gpu_execute_host:
 * uploads what the loops read -- one copy per host array across the loops --
 * runs them, downloads what they wrote, synchronously). */
int loam_gpu_execute_blocks_host(const loam_loop_desc* loops, int nloops, void* stream);

/* ---- consumers of the assembled matrix --------------------- */
/* y = A x by CSR traversal (data.hpp:236-250 mat_spmv): rows ascending, each
 * row folded in column order with a separate multiply and add -- bitwise
 * equal to the reference.  x_len must equal the column count
 * (DimensionMismatch otherwise); y has nrows entries.  Device pointers. */
int loam_gpu_spmv(const loam_sparsity_desc* sparsity, const double* values, const double* x,
                  int64_t x_len, double* y, void* stream);

/* 2x2 nested operator (solver.hpp:21-28 BlockMat): a null sparsity is a zero
 * block; block (i, j) is row_sizes[i] x col_sizes[j]. */
typedef struct loam_block_mat {
  const loam_sparsity_desc* sparsity[2][2];
  const double* values[2][2];
  int32_t row_sizes[2];
  int32_t col_sizes[2];
} loam_block_mat;

/* y_i = sum_j A_ij x_j on the flattened numbering (solver.hpp:33-58
 * block_spmv): each row folds its block-0 entries, then block 1 -- bitwise
 * equal to the reference. */
int loam_gpu_block_spmv(const loam_block_mat* op, const double* x, int64_t x_len, double* y,
                        void* stream);

/* solver.hpp:13-18 SolveReport; reason 0 rtol, 1 atol, 2 maxit. */
typedef struct loam_solve_report {
  int32_t iterations;
  double final_residual_norm;
  int32_t converged;
  int32_t reason;
} loam_solve_report;

/* Preconditioned CG (solver.hpp:80-207 cg_solve): x holds x0 on entry (zeros
 * are the reference default) and the iterate on return; stopping test
 * max(rtol ||b||, atol) on the recurrence, re-verified with the true
 * residual; IndefiniteBreakdown when p'Ap <= 0 or (jacobi != 0) a diagonal
 * entry is not positive; maxit returns the last iterate unconverged.  The
 * iteration runs on the device (flag-gated kernels, no per-iteration host
 * synchronisation); dot products are deterministic two-pass reductions. */
int loam_gpu_cg_solve(const loam_sparsity_desc* sparsity, const double* values, const double* b,
                      int64_t b_len, double* x, double rtol, double atol, int32_t maxit,
                      int32_t jacobi, loam_solve_report* report, void* stream);
int loam_gpu_cg_solve_block(const loam_block_mat* op, const double* b, int64_t b_len, double* x,
                            double rtol, double atol, int32_t maxit, int32_t jacobi,
                            loam_solve_report* report, void* stream);

/* ---- around the assembly loop ------------------------ */
/* Strong Dirichlet rows on a device CSR (fem/assemble.hpp:54-66
 * apply_dirichlet): for every bc node r, zero row r inside its sparsity, set
 * the diagonal to 1 and (rhs != NULL) rhs[r] = value; value = node_values[r]
 * when node_values != NULL (a bc Function), else `constant`
 * (DirichletBC::value_at, fem/bc.hpp:17-19).  rhs == NULL is
 * apply_dirichlet_rows (:69-79).  ShapeMismatch when the matrix is not
 * square; MissingDiagonal "diagonal (r, r) outside sparsity" -- reported
 * before any row is modified.  All arrays on the device. */
int loam_gpu_apply_dirichlet(const loam_sparsity_desc* sparsity, double* values, double* rhs,
                             const int32_t* nodes, int32_t nnodes, const double* node_values,
                             double constant, void* stream);
/* DirichletBC::apply (fem/bc.hpp:21-26): dat[r] = value for every bc node. */
int loam_gpu_bc_apply(double* dat, int32_t set_size, const int32_t* nodes, int32_t nnodes,
                      const double* node_values, double constant, void* stream);

/* pointwise (fem/assemble.hpp:150-319): out (=|+=|-=) expr over n values
 * (set size x dim), expr given as a postfix program over constants and
 * fields (field -1 = the output itself: the reference's RW staging).  One
 * rounding per operation, the reference's evaluation order: bitwise equal. */
enum loam_pw_opcode { LOAM_PW_CONST = 0, LOAM_PW_FIELD, LOAM_PW_ADD, LOAM_PW_SUB, LOAM_PW_MUL,
                      LOAM_PW_DIV, LOAM_PW_NEG };
enum loam_pw_assign { LOAM_PW_ASSIGN = 0, LOAM_PW_ADD_TO = 1, LOAM_PW_SUB_FROM = 2 };
typedef struct loam_pw_instr {
  int32_t op;    /* loam_pw_opcode */
  int32_t field; /* LOAM_PW_FIELD: index into fields, -1 = out */
  double value;  /* LOAM_PW_CONST */
} loam_pw_instr;
int loam_gpu_pointwise(double* out, int64_t n, int32_t op, const loam_pw_instr* program,
                       int32_t nprogram, const double* const* fields, int32_t nfields, void* stream);

/* Reductions of a device vector into *result (host), fixed order. */
enum loam_reduce_kind { LOAM_REDUCE_SUM = 0, LOAM_REDUCE_MIN, LOAM_REDUCE_MAX, LOAM_REDUCE_MAX_ABS };
int loam_gpu_reduce(const double* x, int64_t n, int32_t kind, double* result, void* stream);

/* ---- device-resident variants for CUDA-graph capture (extension) ---------
 * No host synchronisation, scalars in device memory: a time-stepping loop
 * built from them can be captured once and replayed (bench::run_wave,
 * bench.hpp:222-300, in wave.py). */
/* *result_dev = reduction of x (same order as loam_gpu_reduce). */
int loam_gpu_reduce_dev(const double* x, int64_t n, int32_t kind, double* result_dev, void* stream);
/* DirichletBC::apply with the constant read from device memory. */
int loam_gpu_bc_apply_dev(double* dat, int32_t set_size, const int32_t* nodes, int32_t nnodes,
                          const double* value_dev, void* stream);
/* One bench::run_wave step (bench.hpp:267-289) fused into the vertex-star
 * stiffness action: `args` describe the action loop (b INC, X READ, phi READ
 * over the cell->vertex map, kernel stiffness_action_p1_tri); the kernel
 * reads p_in / phi_in (device [n_vertices]) and writes p_out / phi_out
 * (distinct buffers): phi_h = phi - half_dt p; b = K phi_h; p += b pc;
 * p[bc != 0] = state[1]; phi = phi_h - half_dt p; state[2] = max(state[2],
 * |p|_inf).  Bitwise equal to the unfused chain (execute + pointwise +
 * bc_apply + reduce).  UnsupportedForm when the loop has no vertex-star plan
 * (the caller then runs the unfused chain). */
int loam_gpu_wave_step(const loam_kernel_desc* kernel, int32_t n, uint64_t iter, const loam_arg_desc* args,
                       int nargs, const double* p_in, const double* phi_in, double* p_out, double* phi_out,
                       const double* p_constant, const uint8_t* bc_mask, double half_dt, double* state,
                       void* stream);
/* The run_wave clock on device state s[6] = {t, bc value, |p|, max |p| over
 * t <= first_period, blow-up step (0 = none), steps}.  phase 0: s[1] =
 * sin(10 pi t) (the marker-1 forcing, bench.hpp:237); phase 1 (after |p| is
 * in s[2]): t += dt, steps += 1, the first-period maximum and the blow-up
 * test |p| > 1e3 * max (bench.hpp:262-266) record the first failing step. */
int loam_gpu_wave_clock(double* state_dev, double dt, double first_period, int32_t phase, void* stream);

/* ---- topology / data services ------------------------------------------- */
/* Map construction check (topology.hpp:45-48): every entry in [0, target). */
int loam_gpu_map_check(const loam_map_desc* map, void* stream);
/* loam::build_sparsity (data.hpp:149-179), bit-exact.  Allocates device
 * arrays *row_ptr ([rows+1] int64) and *col_idx ([nnz] int32), released with
 * loam_gpu_free. */
int loam_gpu_build_sparsity(const loam_map_desc* row_map, const loam_map_desc* col_map,
                            int row_dim, int col_dim, int64_t** row_ptr, int32_t** col_idx,
                            int64_t* nnz, void* stream);
/* loam::color_iteration (topology.hpp:86-125), bit-exact greedy colouring
 * computed on the device (Jones-Plassmann with ascending-index priority).
 * colors: device [n]. */
int loam_gpu_color_iteration(int32_t n, uint64_t iterset_id, const loam_map_desc* maps,
                             int nmaps, int32_t* colors, int32_t* num_colors, void* stream);

/* ---- mesh-side builders on the device ---------------------- */
/* P2 node numbering (fem/space.hpp:48-72): vertices keep their ids, unique
 * edges are numbered lexicographically from nverts; cell row = vertices then
 * edges ((1,2),(0,2),(0,1) for triangles; (2,3),(1,3),(1,2),(0,3),(0,2),(0,1)
 * for tetrahedra).  cv: device [ncells x (gdim+1)], cn: device
 * [ncells x 6|10].  Returns the node count in *nnodes.  Bit-exact with the
 * reference (triangles) and with loam_gpu_p2_cell_node_map. */
int loam_gpu_p2_cell_node_map_dev(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv,
                                  int32_t* cn, int32_t* nnodes, void* stream);
/* derive_exterior_facets (mesh.hpp:48-89, no markers): facets incident to
 * exactly one cell, in (cell, local facet) discovery order, as sorted vertex
 * tuples (*facet_vertices [n x gdim]) and (cell, local facet) pairs
 * (*facet_cell [n x 2]); device arrays allocated here, released with
 * loam_gpu_free.  NonManifold when a facet has more than two cells. */
int loam_gpu_exterior_facets(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv,
                             int32_t** facet_vertices, int32_t** facet_cell, int32_t* nfacets,
                             void* stream);
/* rcm_order (topology.hpp:131-178): reverse Cuthill-McKee over adjacency
 * lists given as CSR (row_ptr device [n+1], col_idx device), bit-exact with
 * the reference: seeds of minimum degree (lowest index) per component,
 * neighbours in (degree, index) order, reversed.  degree = list length.
 * order: device [n], order[new] = old.  IndexOutOfRange / AsymmetricAdjacency
 * at the first offending entry in list order, as the reference scans. */
int loam_gpu_rcm_order(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, int32_t* order,
                       void* stream);
/* vertex_adjacency (mesh.hpp:350-362): per vertex the sorted other vertices
 * sharing a cell, as CSR (device arrays allocated here, loam_gpu_free). */
int loam_gpu_vertex_adjacency(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv,
                              int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, void* stream);
/* The renumbering half of reorder (mesh.hpp:369-386) for a given perm
 * (perm[new] = old, device [nverts]): coords_out[new] = coords[perm[new]]
 * (may be null), cv_out[k] = new_of[cv[k]].  InvalidArgument when perm is not
 * a permutation. */
int loam_gpu_renumber_vertices(int32_t nverts, int32_t gdim, const double* coords, int32_t ncells,
                               const int32_t* cv, const int32_t* perm, double* coords_out, int32_t* cv_out,
                               void* stream);

/* ---- device memory helpers (for FFI callers without a CUDA binding) ------ */
int loam_gpu_malloc(void** ptr, size_t bytes);
int loam_gpu_free(void* ptr);
int loam_gpu_host_alloc(void** ptr, size_t bytes); /* pinned */
int loam_gpu_host_free(void* ptr);
int loam_gpu_memcpy(void* dst, const void* src, size_t bytes, void* stream); /* any direction */
int loam_gpu_memset(void* dst, int value, size_t bytes, void* stream);
int loam_gpu_stream_sync(void* stream);

/* ---- seeded synthetic inputs (host; csrc/meshgen.cpp) --------- */
int loam_gpu_unit_square_mesh(int n, double* coords, int32_t* cv);  /* mesh.hpp:96-143 */
int loam_gpu_unit_cube_mesh(int n, double* coords, int32_t* cv);    /* mesh.hpp:148-214 */
int loam_gpu_jitter(int gdim, int n, double amp, uint64_t seed, double* coords);
int loam_gpu_permute_cells(int ncells, int arity, uint64_t seed, int32_t* cv);
int loam_gpu_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out);
int loam_gpu_p2_cell_node_map(int ncells, int nv, int gdim, const int32_t* cv, int32_t* cn);
int loam_gpu_expand_map(int nsrc, int arity, const int32_t* map, int dim, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* LOAM_GPU_H */
