/*
 * loam_oracle -- CPU restatement of the reference par_loop hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker.
 * The product path (paper_1501_01809_b200/) never links or calls it.
 *
 * Every function restates an algorithm of the reference `loam` library
 * (/root/reference/proj/include/loam, C++20 header-only) and cites the
 * file:line it follows.  Parity pinning: tests/test_oracle_cpu.py checks this
 * restatement against (a) the reference's own known-answer tests (KATs copied
 * as numbers into the test, e.g. test_parloop.cpp:61-68, test_data.cpp:22-40,
 * test_topology.cpp:55-84, test_fem.cpp:141-161) and (b) golden vectors that
 * oracle/_ref (the reference headers compiled by oracle/Makefile) produced
 * for the P1/P2-triangle and P1-tet configurations (tests/golden/).
 * The P2-tet basis, the 14-point tet rule, elasticity and the Stokes blocks
 * have no reference implementation: they are pinned only against exact
 * symbolic integration (tests/exact_fem.py), i.e. "parity unpinned" by
 * reference tests, as DESIGN.md states.
 */
#ifndef LOAM_ORACLE_H
#define LOAM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Form identifiers shared with the product registry (same numbering). */
enum orc_form {
  ORC_MASS = 0,             /* bilinear  M_ij = int phi_i phi_j          (form.hpp:266) */
  ORC_STIFFNESS = 1,        /* bilinear  K_ij = int grad phi_i . grad phi_j (form.hpp:268-272) */
  ORC_HELMHOLTZ = 2,        /* bilinear  K + kappa M                      (form.hpp:273-274) */
  ORC_MASS_ACTION = 3,      /* linear    b_i = int (sum_k C_k phi_k) phi_i (form.hpp:306-312) */
  ORC_STIFFNESS_ACTION = 4, /* linear    b_i = int grad phi_i . grad u     (form.hpp:288-303) */
  ORC_HELMHOLTZ_ACTION = 5, /* linear    stiffness_action + kappa mass_action, one loop (new) */
  ORC_ELASTICITY = 6,       /* vector-P1 tet 12x12, params lambda, mu (new; config 4) */
  ORC_STOKES_A = 7,         /* vector-P2 tri 12x12 viscous block, param nu (new; config 5) */
  ORC_STOKES_B = 8,         /* P1 pressure x vector-P2 velocity 3x12: -int q div u (new) */
  ORC_STOKES_BT = 9         /* transpose of B, 12x3 (new) */
};

/* Error codes: 0 = ok, otherwise 1 + loam::ErrorKind (common.hpp:10-33). */
#define ORC_OK 0
#define ORC_ERR_INDEX_OUT_OF_RANGE (1 + 0)
#define ORC_ERR_OUTSIDE_SPARSITY (1 + 9)
#define ORC_ERR_UNSUPPORTED_FORM (1 + 16)
#define ORC_ERR_INVALID_ARGUMENT (1 + 21)

/* ---- topology ---------------------------------------------------------- */

/* Greedy first-fit colouring, ascending entity, union of conflict maps.
 * topology.hpp:86-125.  Returns num_colors (>=0) or -error. */
int orc_color_iteration(int n, int nmaps, const int32_t* const* maps, const int32_t* arity,
                        const int32_t* target_size, int32_t* colors);

/* Reverse Cuthill-McKee (topology.hpp:131-178) over adjacency lists given as
 * CSR (row_ptr [n+1], col_idx): checks every entry in list order (out of
 * range -> ORC_ERR_INDEX_OUT_OF_RANGE, no back entry ->
 * ORC_ERR_ASYMMETRIC_ADJACENCY, *fail = entry position), then BFS from the
 * minimum-(degree, index) unvisited vertex, unvisited neighbours appended in
 * (degree, index) order, reversed.  order[new] = old. */
#define ORC_ERR_ASYMMETRIC_ADJACENCY (1 + 3)
int orc_rcm_order(int n, const int64_t* row_ptr, const int32_t* col_idx, int32_t* order, int64_t* fail);

/* ---- sparsity (data.hpp:149-179) -------------------------------------- */

/* Builds the CSR union pattern.  Returns nnz (>=0) or -error.  The arrays are
 * allocated with malloc and must be released with orc_free. */
int64_t orc_build_sparsity(int nsrc, const int32_t* row_map, int ar_r, int nrt,
                           const int32_t* col_map, int ar_c, int nct, int row_dim, int col_dim,
                           int64_t** row_ptr_out, int32_t** col_idx_out);
void orc_free(void* p);

/* Position of (row, col) in the values array or -1 (data.hpp:129-136). */
int64_t orc_sparsity_find(const int64_t* row_ptr, const int32_t* col_idx, int nrows, int row,
                          int col);

/* ---- function spaces (space.hpp:48-72) --------------------------------- */

/* P2 cell->node map.  Vertex nodes keep their ids; unique edges keyed by the
 * sorted vertex pair are numbered lexicographically from nv.  Triangle rows:
 * v0,v1,v2,e(v1v2),e(v0v2),e(v0v1) (space.hpp:66-71).  Tet rows (extension,
 * not in the reference): v0..v3 then edges (2,3),(1,3),(1,2),(0,3),(0,2),(0,1).
 * cn must hold ncells*(gdim==2?6:10) ints.  Returns the node count. */
int orc_p2_cell_node_map(int ncells, int nv, int gdim, const int32_t* cv, int32_t* cn);

/* ---- element kernels (form.hpp:139-320, element.hpp) ------------------- */

/* Local element tensor for `form` on one cell.
 *   degree: Lagrange degree of the (test) space; gdim: 2 (triangle) / 3 (tet)
 *   X: (gdim+1) x gdim vertex coordinates;  C: coefficient nodal values
 *   params: kappa (helmholtz), lambda,mu (elasticity), nu (stokes)
 *   out: zero-initialised by the caller is NOT required; the kernel zeroes it.
 * Returns 0 or an error code. */
int orc_element(int form, int degree, int gdim, const double* params, const double* X,
                const double* C, double* out);

/* Local tensor shape of `form`: rows/cols (cols = 1 for linear forms). */
int orc_element_shape(int form, int degree, int gdim, int* rows, int* cols);

/* ---- assembly through the par_loop semantics (parloop.hpp:191-384) ----- */

/* Linear form INC into a node Dat (out is overwritten with the assembled
 * vector; zero-initialised first as assemble_vector's make_dat does,
 * assemble.hpp:111).  Entities are processed in ascending order. */
int orc_assemble_vector(int form, int degree, int gdim, const double* params, int ncells,
                        const int32_t* test_map, int ar_t, const int32_t* coord_map,
                        const double* coords, const int32_t* coeff_map, int ar_coeff,
                        const double* coeff, int nout, double* out);

/* Bilinear form INC into CSR values via Mat::addto (data.hpp:205-222).
 * values is zeroed first (data.hpp:187).  Returns ORC_ERR_OUTSIDE_SPARSITY
 * when a local entry is not in the pattern. */
int orc_assemble_matrix(int form, int degree, int gdim, const double* params, int ncells,
                        const int32_t* row_map, int ar_r, const int32_t* col_map, int ar_c,
                        const int32_t* coord_map, const double* coords, int nrows,
                        const int64_t* row_ptr, const int32_t* col_idx, double* values);

/* Same as orc_assemble_matrix but iterating cells in the reference's threaded
 * order (colour-major, entity-ascending inside a colour; parloop.hpp:234-235,
 * 322-352), which makes the result bitwise comparable with the reference. */
int orc_assemble_matrix_colored(int form, int degree, int gdim, const double* params, int ncells,
                                const int32_t* row_map, int ar_r, const int32_t* col_map,
                                int ar_c, const int32_t* coord_map, const double* coords,
                                int nrows, const int64_t* row_ptr, const int32_t* col_idx,
                                const int32_t* colors, int ncolors, double* values);

/* ---- consumers of the assembled matrix ---------------------
 * A nested operator is 2x2 blocks given as arrays of 4 row-major (i, j)
 * pointers; a null row_ptr is a zero block (solver.hpp:21-28).  A plain Mat
 * is block (0, 0) with row_sizes = {nrows, 0}, col_sizes = {ncols, 0}. */

/* y = A x: rows ascending, entries folded in column order, acc += v * x with a
 * separate multiply and add (data.hpp:236-250; solver.hpp:33-58 for nested). */
void orc_block_spmv(const int32_t* row_sizes, const int32_t* col_sizes, const int64_t* const* row_ptr,
                    const int32_t* const* col_idx, const double* const* values, const double* x, double* y);

/* cg_iterate (solver.hpp:80-168) with cg_solve's Jacobi set-up
 * (solver.hpp:64-76, 180-201).  x: x0 in, iterate out.  Returns 0, or
 * ORC_ERR_INDEFINITE (non-positive Jacobi diagonal: *fail = row; p'Ap <= 0:
 * *fail = iteration).  report: iterations, converged, reason (0 rtol, 1 atol,
 * 2 maxit); *rnorm = final residual norm. */
#define ORC_ERR_INDEFINITE 20
int orc_cg(const int32_t* row_sizes, const int32_t* col_sizes, const int64_t* const* row_ptr,
           const int32_t* const* col_idx, const double* const* values, int nested, const double* b, double* x,
           double rtol, double atol, int maxit, int jacobi, int32_t* report, double* rnorm, int32_t* fail);

/* ---- around the assembly loop ------------------------ */

/* pointwise (fem/assemble.hpp:150-319): out (=|+=|-=) expr for every one of n
 * values; expr is a postfix program (op codes as include/loam_gpu.h
 * loam_pw_opcode: 0 const, 1 field, 2 add, 3 sub, 4 mul, 5 div, 6 neg; field
 * -1 = out).  assign: 0 =, 1 +=, 2 -=.  Evaluated like the reference's
 * lowered AST: one rounding per operation, left operand first. */
int orc_pointwise(double* out, int64_t n, int assign, const int32_t* ops, const int32_t* fidx,
                  const double* vals, int nprog, const double* const* fields);

/* apply_dirichlet (fem/assemble.hpp:54-66; rhs NULL: apply_dirichlet_rows
 * :69-79): for each node r in order, zero row r, find (r, r), set it to 1,
 * rhs[r] = node_values ? node_values[r] : constant.  Returns
 * ORC_ERR_MISSING_DIAGONAL (*fail = r) at the first row without a diagonal,
 * after modifying the earlier rows -- the reference's order. */
#define ORC_ERR_MISSING_DIAGONAL (1 + 17)
int orc_apply_dirichlet(int nrows, const int64_t* row_ptr, const int32_t* col_idx, double* values,
                        double* rhs, const int32_t* nodes, int nn, const double* node_values,
                        double constant, int32_t* fail);

/* ---- seeded synthetic inputs (SURVEY 8d generator; bench --impl reference) */
int orc_unit_square_mesh(int n, double* coords, int32_t* cv);  /* mesh.hpp:96-143 */
int orc_unit_cube_mesh(int n, double* coords, int32_t* cv);    /* mesh.hpp:148-214 */
int orc_jitter(int gdim, int n, double amp, uint64_t seed, double* coords);
int orc_permute_cells(int ncells, int arity, uint64_t seed, int32_t* cv);
int orc_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif
