// ref_harness.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against the headers
// where they lie (-I/root/reference/proj/include) into oracle/_ref/libloam_ref.so.
// Nothing from the reference is copied into this repository.  Used by
//   * tests/ to pin the C restatement (oracle/loam_oracle.c) and the CUDA path,
//   * tools/make_golden.py to write tests/golden/*.npz,
//   * bench.py --impl reference / cpu_baseline to time the reference par_loop.
//
// For configs 3-5 the reference has no element kernel (fem/element.hpp:179-180,
// fem/form.hpp:30-45); there the reference ENGINE (build_sparsity, execute,
// Mat::addto) runs a host kernel (kernel.hpp:523-529) whose body is the C
// restatement orc_element (oracle/loam_oracle.c), linked into this library.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "loam/loam.hpp"
#ifdef LOAM_REF_HAVE_BENCH
#include "loam/bench.hpp"
#endif
#include "loam_oracle.h"

using namespace loam;

namespace {

thread_local std::string g_error;

int fail_code(const Error& e) {
  g_error = e.what();
  return 1 + static_cast<int>(e.kind());
}

MeshPtr mesh_from_arrays(int gdim, int ncells, int nv, const int32_t* cv, const double* coords,
                         bool facets) {
  auto mesh = std::make_shared<Mesh>();
  mesh->dim = gdim;
  mesh->cells = make_set(ncells, "cells");
  mesh->vertices = make_set(nv, "vertices");
  std::vector<int> table(cv, cv + static_cast<size_t>(ncells) * (gdim + 1));
  mesh->cell_vertex_map = make_map(mesh->cells, mesh->vertices, gdim + 1, std::move(table),
                                   "cell_vertex");
  mesh->coordinates = make_dat(mesh->vertices, gdim, "coordinates");
  auto x = mesh->coordinates->mutable_view();
  std::memcpy(x.data(), coords, sizeof(double) * static_cast<size_t>(nv) * gdim);
  if (facets) loam::detail::derive_exterior_facets(*mesh, nullptr);
  return mesh;
}

template <class T>
T* copy_out(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Catalogue form for (kind, degree) on V.  kind uses the orc_form numbering.
fem::Form catalogue_form(int kind, const fem::FunctionSpacePtr& V, const fem::FunctionPtr& u,
                         double kappa) {
  switch (kind) {
  case ORC_MASS: return fem::mass(V, V);
  case ORC_STIFFNESS: return fem::stiffness(V, V);
  case ORC_HELMHOLTZ: return fem::helmholtz(V, V, kappa);
  case ORC_MASS_ACTION: return fem::mass_action(V, u);
  case ORC_STIFFNESS_ACTION: return fem::stiffness_action(V, u);
  default: fail(ErrorKind::UnsupportedForm, "not a reference catalogue form");
  }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }
void ref_free(void* p) { std::free(p); }

// mesh.hpp:96-143
int ref_unit_square_mesh(int n, double* coords, int32_t* cv) {
  try {
    auto m = unit_square_mesh(n);
    auto x = m->coordinates->view();
    std::memcpy(coords, x.data(), sizeof(double) * x.size());
    const auto& v = m->cell_vertex_map->values();
    std::memcpy(cv, v.data(), sizeof(int32_t) * v.size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// mesh.hpp:148-214
int ref_unit_cube_mesh(int n, double* coords, int32_t* cv) {
  try {
    auto m = unit_cube_mesh(n);
    auto x = m->coordinates->view();
    std::memcpy(coords, x.data(), sizeof(double) * x.size());
    const auto& v = m->cell_vertex_map->values();
    std::memcpy(cv, v.data(), sizeof(int32_t) * v.size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// topology.hpp:86-125 (through the cached conflict_coloring entry point is not
// needed: the cache returns the same colouring).  Returns num_colors or -err.
int ref_color_iteration(int n, int nmaps, const int32_t* const* maps, const int32_t* arity,
                        const int32_t* target, int32_t* colors) {
  try {
    auto iter = make_set(n, "iter");
    std::vector<MapPtr> ms;
    for (int m = 0; m < nmaps; ++m) {
      auto t = make_set(target[m], "target");
      std::vector<int> vals(maps[m], maps[m] + static_cast<size_t>(n) * arity[m]);
      ms.push_back(make_map(iter, t, arity[m], std::move(vals)));
    }
    auto c = color_iteration(iter, ms);
    std::memcpy(colors, c.colors.data(), sizeof(int32_t) * c.colors.size());
    return c.num_colors;
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// data.hpp:149-179.  Returns nnz or -err; arrays via ref_free.
int64_t ref_build_sparsity(int nsrc, const int32_t* row_map, int ar_r, int nrt,
                           const int32_t* col_map, int ar_c, int nct, int row_dim, int col_dim,
                           int64_t** rp, int32_t** ci) {
  try {
    auto src = make_set(nsrc);
    auto rt = make_set(nrt);
    auto ct = make_set(nct);
    auto rm = make_map(src, rt, ar_r,
                       std::vector<int>(row_map, row_map + static_cast<size_t>(nsrc) * ar_r));
    auto cm = make_map(src, ct, ar_c,
                       std::vector<int>(col_map, col_map + static_cast<size_t>(nsrc) * ar_c));
    auto sp = build_sparsity(rm, cm, row_dim, col_dim);
    std::vector<int64_t> offs(sp->row_offsets().begin(), sp->row_offsets().end());
    *rp = copy_out(offs);
    *ci = copy_out(sp->col_indices());
    return sp->nnz();
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// space.hpp:30-82 for triangles (degree 2).  Returns node count or -err.
int ref_p2_tri_map(int ncells, int nv, const int32_t* cv, const double* coords, int32_t* cn) {
  try {
    auto mesh = mesh_from_arrays(2, ncells, nv, cv, coords, true);
    auto V = fem::make_function_space(mesh, 2);
    const auto& v = V->cell_node_map->values();
    std::memcpy(cn, v.data(), sizeof(int32_t) * v.size());
    return V->node_set->size();
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// Local element tensor of a catalogue form through the reference kernel
// pipeline: compile_local_kernel -> hoist_invariants -> fold_constants ->
// interpret (assemble.hpp:16-19, kernel.hpp:482-495).
int ref_local_kernel(int kind, int degree, int gdim, double kappa, const double* X,
                     const double* C, double* out) {
  try {
    auto mesh = gdim == 2 ? unit_square_mesh(1) : unit_cube_mesh(1);
    auto V = fem::make_function_space(mesh, degree);
    auto u = fem::make_function(V);
    auto form = catalogue_form(kind, V, u, kappa);
    auto kernel = fem::detail::optimized_kernel(form);
    const auto& params = kernel->params();
    std::vector<std::vector<Real>> bufs;
    for (const auto& p : params) bufs.emplace_back(p.size(), 0.0);
    std::memcpy(bufs[1].data(), X, sizeof(double) * bufs[1].size());
    if (bufs.size() > 2) std::memcpy(bufs[2].data(), C, sizeof(double) * bufs[2].size());
    std::vector<Real*> ptrs;
    for (auto& b : bufs) ptrs.push_back(b.data());
    ir::invoke(*kernel, {ptrs.data(), ptrs.size()});
    std::memcpy(out, bufs[0].data(), sizeof(double) * bufs[0].size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// fem::assemble_vector (assemble.hpp:108-135) of a catalogue linear form on
// the given mesh; kind ORC_HELMHOLTZ_ACTION = stiffness_action + kappa *
// mass_action as two reference loops (no single catalogue form).
// coeff lives on the degree-`degree` node set the reference builds.
int ref_assemble_vector(int kind, int degree, int gdim, double kappa, int ncells, int nv,
                        const int32_t* cv, const double* coords, const double* coeff,
                        int threads, double* out, int* nout) {
  try {
    auto mesh = mesh_from_arrays(gdim, ncells, nv, cv, coords, degree == 2);
    auto V = fem::make_function_space(mesh, degree);
    auto u = fem::make_function(V);
    auto w = u->dat->mutable_view();
    std::memcpy(w.data(), coeff, sizeof(double) * w.size());
    *nout = V->node_set->size();
    if (kind == ORC_HELMHOLTZ_ACTION) {
      auto a = fem::assemble_vector(fem::stiffness_action(V, u), {}, threads);
      auto b = fem::assemble_vector(fem::mass_action(V, u), {}, threads);
      auto av = a->view();
      auto bv = b->view();
      for (size_t i = 0; i < av.size(); ++i) out[i] = av[i] + kappa * bv[i];
    } else {
      auto a = fem::assemble_vector(catalogue_form(kind, V, u, kappa), {}, threads);
      auto av = a->view();
      std::memcpy(out, av.data(), sizeof(double) * av.size());
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// fem::assemble_matrix (assemble.hpp:85-104) of a catalogue bilinear form.
// Returns nnz or -err; rp/ci/vals via ref_free.
int64_t ref_assemble_matrix(int kind, int degree, int gdim, double kappa, int ncells, int nv,
                            const int32_t* cv, const double* coords, int threads, int* nrows,
                            int64_t** rp, int32_t** ci, double** vals) {
  try {
    auto mesh = mesh_from_arrays(gdim, ncells, nv, cv, coords, degree == 2);
    auto V = fem::make_function_space(mesh, degree);
    auto mat = fem::assemble_matrix(catalogue_form(kind, V, nullptr, kappa), {}, threads);
    const auto& sp = *mat->sparsity();
    *nrows = sp.nrows();
    std::vector<int64_t> offs(sp.row_offsets().begin(), sp.row_offsets().end());
    *rp = copy_out(offs);
    *ci = copy_out(sp.col_indices());
    *vals = copy_out(mat->values());
    return sp.nnz();
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// The reference ENGINE with a restated host kernel: build_sparsity +
// Mat + execute (parloop.hpp:191-384) for forms the reference catalogue
// lacks (P2 tet, elasticity, Stokes blocks).  Maps are dof-expanded where the
// Mat is vector valued.  Returns nnz or -err.
int64_t ref_engine_matrix(int form, int degree, int gdim, const double* params, int ncells,
                          const int32_t* row_map, int ar_r, int nrt, const int32_t* col_map,
                          int ar_c, int nct, const int32_t* coord_map, int nv,
                          const double* coords, int threads, int64_t** rp, int32_t** ci,
                          double** vals) {
  try {
    auto cells = make_set(ncells, "cells");
    auto rt = make_set(nrt, "rows");
    auto ct = nct == nrt && col_map == row_map ? rt : make_set(nct, "cols");
    auto verts = make_set(nv, "vertices");
    auto rm = make_map(cells, rt, ar_r,
                       std::vector<int>(row_map, row_map + static_cast<size_t>(ncells) * ar_r));
    auto cm = col_map == row_map
                  ? rm
                  : make_map(cells, ct, ar_c,
                             std::vector<int>(col_map, col_map + static_cast<size_t>(ncells) * ar_c));
    auto xm = make_map(cells, verts, gdim + 1,
                       std::vector<int>(coord_map, coord_map + static_cast<size_t>(ncells) * (gdim + 1)));
    auto X = make_dat(verts, gdim, "coordinates");
    std::memcpy(X->mutable_view().data(), coords, sizeof(double) * static_cast<size_t>(nv) * gdim);
    auto mat = make_mat(build_sparsity(rm, cm), "assembled");
    std::vector<double> p(params, params + 4);
    auto kernel = ir::make_host_kernel(
        "host_form_" + std::to_string(form), {{"A", {ar_r, ar_c}}, {"X", {gdim + 1, gdim}}},
        [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], nullptr, a[0]); });
    Parloop loop{kernel, cells, {arg(mat, Access::INC, rm, cm), arg(X, Access::READ, xm)}};
    execute(loop, threads);
    const auto& sp = *mat->sparsity();
    std::vector<int64_t> offs(sp.row_offsets().begin(), sp.row_offsets().end());
    *rp = copy_out(offs);
    *ci = copy_out(sp.col_indices());
    *vals = copy_out(mat->values());
    return sp.nnz();
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// Same engine for a residual with a restated host kernel (P2 tet action).
int ref_engine_vector(int form, int degree, int gdim, const double* params, int ncells,
                      const int32_t* test_map, int ar_t, int nt, const int32_t* coord_map,
                      int nv, const double* coords, const double* coeff, int threads,
                      double* out) {
  try {
    auto cells = make_set(ncells, "cells");
    auto nodes = make_set(nt, "nodes");
    auto verts = make_set(nv, "vertices");
    auto tm = make_map(cells, nodes, ar_t,
                       std::vector<int>(test_map, test_map + static_cast<size_t>(ncells) * ar_t));
    auto xm = make_map(cells, verts, gdim + 1,
                       std::vector<int>(coord_map, coord_map + static_cast<size_t>(ncells) * (gdim + 1)));
    auto X = make_dat(verts, gdim, "coordinates");
    std::memcpy(X->mutable_view().data(), coords, sizeof(double) * static_cast<size_t>(nv) * gdim);
    auto u = make_dat(nodes, 1, "u");
    std::memcpy(u->mutable_view().data(), coeff, sizeof(double) * static_cast<size_t>(nt));
    auto b = make_dat(nodes, 1, "assembled");
    std::vector<double> p(params, params + 4);
    auto kernel = ir::make_host_kernel(
        "host_form_" + std::to_string(form),
        {{"A", {ar_t}}, {"X", {gdim + 1, gdim}}, {"C", {ar_t}}},
        [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], a[2], a[0]); });
    Parloop loop{kernel, cells, {arg(b, Access::INC, tm), arg(X, Access::READ, xm), arg(u, Access::READ, tm)}};
    execute(loop, threads);
    auto bv = b->view();
    std::memcpy(out, bv.data(), sizeof(double) * bv.size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// Timed reference ENGINE on arbitrary maps (bench per-config CPU figures):
// the reference's build_sparsity (timed once into *sparsity_s), then `steps`
// timed rounds of Mat::zero / Dat reset + loam::execute with `threads`
// workers and the restated host kernel (kernel.hpp:523-529).  col_map NULL =
// a residual: Dat INC through row_map, coefficient `coeff` READ through it.
int ref_time_engine(int form, int degree, int gdim, const double* params, int ncells, const int32_t* row_map,
                    int ar_r, int nrt, const int32_t* col_map, int ar_c, int nct, const int32_t* coord_map,
                    int nv, const double* coords, const double* coeff, int threads, int warmup, int steps,
                    double* times, double* sparsity_s) {
  try {
    auto cells = make_set(ncells, "cells");
    auto rt = make_set(nrt, "rows");
    auto verts = make_set(nv, "vertices");
    auto rm = make_map(cells, rt, ar_r, std::vector<int>(row_map, row_map + static_cast<size_t>(ncells) * ar_r));
    auto xm = make_map(cells, verts, gdim + 1,
                       std::vector<int>(coord_map, coord_map + static_cast<size_t>(ncells) * (gdim + 1)));
    auto X = make_dat(verts, gdim, "coordinates");
    std::memcpy(X->mutable_view().data(), coords, sizeof(double) * static_cast<size_t>(nv) * gdim);
    std::vector<double> p(params, params + 4);
    MatPtr mat;
    DatPtr vec, u;
    Parloop loop;
    *sparsity_s = 0.0;
    if (col_map) {
      auto ct = nct == nrt && col_map == row_map ? rt : make_set(nct, "cols");
      auto cm = col_map == row_map
                    ? rm
                    : make_map(cells, ct, ar_c, std::vector<int>(col_map, col_map + static_cast<size_t>(ncells) * ar_c));
      const double t0 = now();
      auto sp = build_sparsity(rm, cm);
      *sparsity_s = now() - t0;
      mat = make_mat(sp, "assembled");
      auto kernel = ir::make_host_kernel(
          "host_form_" + std::to_string(form), {{"A", {ar_r, ar_c}}, {"X", {gdim + 1, gdim}}},
          [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], nullptr, a[0]); });
      loop = Parloop{kernel, cells, {arg(mat, Access::INC, rm, cm), arg(X, Access::READ, xm)}};
    } else {
      vec = make_dat(rt, 1, "assembled");
      u = make_dat(rt, 1, "u");
      std::memcpy(u->mutable_view().data(), coeff, sizeof(double) * static_cast<size_t>(nrt));
      auto kernel = ir::make_host_kernel(
          "host_form_" + std::to_string(form), {{"A", {ar_r}}, {"X", {gdim + 1, gdim}}, {"C", {ar_r}}},
          [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], a[2], a[0]); });
      loop = Parloop{kernel, cells, {arg(vec, Access::INC, rm), arg(X, Access::READ, xm), arg(u, Access::READ, rm)}};
    }
    auto run = [&]() {
      if (mat) mat->zero();
      if (vec) {
        auto w = vec->mutable_view();
        std::fill(w.begin(), w.end(), 0.0);
      }
      execute(loop, threads);
    };
    for (int i = 0; i < warmup; ++i) run();
    for (int i = 0; i < steps; ++i) {
      const double t0 = now();
      run();
      times[i] = now() - t0;
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// ---------------------------------------------------------------------------
// Timing entry for bench.py (--impl reference and the cpu_baseline leg).
// Builds the reference objects once, runs `warmup` untimed executes, then
// times `steps` calls of loam::execute (the reference par_loop, parloop.hpp:191)
// with `threads` workers, each preceded by Mat::zero()/Dat reset as
// assemble_matrix/assemble_vector's fresh allocation would do.  The element
// kernel is the reference's own optimised AST kernel (assemble.hpp:16-19)
// when `as_shipped` is nonzero, else a compiled host kernel (orc_element).
// Writes per-step seconds into times[steps].  Returns 0 or err.
int ref_time_execute(int form, int degree, int gdim, const double* params, int ncells, int nv,
                     const int32_t* cv, const double* coords, const double* coeff,
                     int as_shipped, int threads, int warmup, int steps, double* times) {
  try {
    auto mesh = mesh_from_arrays(gdim, ncells, nv, cv, coords, degree == 2);
    auto V = fem::make_function_space(mesh, degree);
    auto u = fem::make_function(V);
    if (coeff) std::memcpy(u->dat->mutable_view().data(), coeff,
                           sizeof(double) * static_cast<size_t>(V->node_set->size()));
    const bool bilinear = form == ORC_MASS || form == ORC_STIFFNESS || form == ORC_HELMHOLTZ;
    std::vector<Parloop> loops;
    MatPtr mat;
    DatPtr vec;
    const double kappa = params[0];
    std::vector<double> p(params, params + 4);
    if (bilinear) {
      mat = make_mat(build_sparsity(V->cell_node_map, V->cell_node_map), "assembled");
      ir::KernelPtr kernel;
      if (as_shipped) {
        kernel = fem::detail::optimized_kernel(catalogue_form(form, V, u, kappa));
      } else {
        const int m = V->element.node_count;
        kernel = ir::make_host_kernel(
            "host_form", {{"A", {m, m}}, {"X", {gdim + 1, gdim}}},
            [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], nullptr, a[0]); });
      }
      loops.push_back({kernel, mesh->cells,
                       {arg(mat, Access::INC, V->cell_node_map, V->cell_node_map),
                        arg(mesh->coordinates, Access::READ, mesh->cell_vertex_map)}});
    } else {
      vec = make_dat(V->node_set, 1, "assembled");
      std::vector<ir::KernelPtr> kernels;
      if (as_shipped) {
        if (form == ORC_HELMHOLTZ_ACTION) { // two catalogue loops
          kernels.push_back(fem::detail::optimized_kernel(fem::stiffness_action(V, u)));
          kernels.push_back(fem::detail::optimized_kernel(fem::mass_action(V, u)));
        } else {
          kernels.push_back(fem::detail::optimized_kernel(catalogue_form(form, V, u, kappa)));
        }
      } else {
        const int m = V->element.node_count;
        kernels.push_back(ir::make_host_kernel(
            "host_form", {{"A", {m}}, {"X", {gdim + 1, gdim}}, {"C", {m}}},
            [=](Real* const* a) { orc_element(form, degree, gdim, p.data(), a[1], a[2], a[0]); }));
      }
      for (auto& k : kernels)
        loops.push_back({k, mesh->cells,
                         {arg(vec, Access::INC, V->cell_node_map),
                          arg(mesh->coordinates, Access::READ, mesh->cell_vertex_map),
                          arg(u->dat, Access::READ, V->cell_node_map)}});
    }
    auto run = [&]() {
      if (mat) mat->zero();
      if (vec) {
        auto w = vec->mutable_view();
        std::fill(w.begin(), w.end(), 0.0);
      }
      for (auto& l : loops) execute(l, threads);
    };
    for (int i = 0; i < warmup; ++i) run();
    for (int i = 0; i < steps; ++i) {
      double t0 = now();
      run();
      times[i] = now() - t0;
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// ---- consumers of the assembled matrix (data.hpp:236-250, solver.hpp) ----
// A block is given as (nrows, ncols, row_offsets, col_indices, values); a null
// row_offsets pointer is a zero block.

}  // extern "C" (helpers below are C++)

namespace {
MatPtr mat_from_csr(int nrows, int ncols, const int64_t* rp, const int32_t* ci, const double* v) {
  std::vector<long> offs(rp, rp + nrows + 1);
  std::vector<int> cols(ci, ci + rp[nrows]);
  auto sp = std::make_shared<const Sparsity>(nrows, ncols, std::move(offs), std::move(cols));
  auto m = make_mat(sp);
  std::memcpy(m->values().data(), v, sizeof(double) * static_cast<size_t>(rp[nrows]));
  return m;
}

BlockMat block_from_csr(const int32_t* rs, const int32_t* cs, const int64_t* const* rp, const int32_t* const* ci,
                        const double* const* v) {
  BlockMat op;
  for (int i = 0; i < 2; ++i) {
    op.row_sizes[i] = rs[i];
    op.col_sizes[i] = cs[i];
    for (int j = 0; j < 2; ++j)
      if (rp[2 * i + j]) op.blocks[i][j] = mat_from_csr(rs[i], cs[j], rp[2 * i + j], ci[2 * i + j], v[2 * i + j]);
  }
  return op;
}

void report_out(const SolveReport& r, int32_t* out_i, double* out_d) {
  out_i[0] = r.iterations;
  out_i[1] = r.converged ? 1 : 0;
  out_i[2] = r.reason == SolveReport::Reason::rtol ? 0 : (r.reason == SolveReport::Reason::atol ? 1 : 2);
  out_d[0] = r.final_residual_norm;
}
} // namespace

extern "C" {

// data.hpp:236-250
int ref_spmv(int nrows, int ncols, const int64_t* rp, const int32_t* ci, const double* v, const double* x,
             int64_t xlen, double* y) {
  try {
    auto m = mat_from_csr(nrows, ncols, rp, ci, v);
    auto out = mat_spmv(*m, std::span<const Real>(x, static_cast<size_t>(xlen)));
    std::memcpy(y, out.data(), sizeof(double) * out.size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// solver.hpp:33-58; rp/ci/v: 4 block pointers in row-major (i, j) order
int ref_block_spmv(const int32_t* rs, const int32_t* cs, const int64_t* const* rp, const int32_t* const* ci,
                   const double* const* v, const double* x, int64_t xlen, double* y) {
  try {
    auto op = block_from_csr(rs, cs, rp, ci, v);
    auto out = block_spmv(op, std::span<const Real>(x, static_cast<size_t>(xlen)));
    std::memcpy(y, out.data(), sizeof(double) * out.size());
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// solver.hpp:170-207 (nested = 0: block (0, 0) as a plain Mat); x: x0 in, iterate out
int ref_cg_solve(int nested, const int32_t* rs, const int32_t* cs, const int64_t* const* rp,
                 const int32_t* const* ci, const double* const* v, const double* b, int64_t blen, double* x,
                 int64_t xlen, double rtol, double atol, int maxit, int jacobi, int32_t* out_i, double* out_d) {
  try {
    std::vector<Real> x0(x, x + xlen);
    const auto pc = jacobi ? Preconditioner::Jacobi : Preconditioner::None;
    std::span<const Real> bs(b, static_cast<size_t>(blen));
    std::pair<std::vector<Real>, SolveReport> res;
    if (nested) res = cg_solve(block_from_csr(rs, cs, rp, ci, v), bs, x0, rtol, atol, maxit, pc);
    else res = cg_solve(*mat_from_csr(rs[0], cs[0], rp[0], ci[0], v[0]), bs, x0, rtol, atol, maxit, pc);
    std::memcpy(x, res.first.data(), sizeof(double) * res.first.size());
    report_out(res.second, out_i, out_d);
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

} // extern "C"

// ---- around the assembly loop (fem/assemble.hpp, fem/bc.hpp) --------------
namespace {
fem::Pw pw_from_program(const int32_t* ops, const int32_t* fidx, const double* vals, int nprog,
                        const std::vector<DatPtr>& fields, const DatPtr& out) {
  std::vector<fem::Pw> st;
  for (int q = 0; q < nprog; ++q) {
    switch (ops[q]) {
    case 0: st.push_back(fem::pw(vals[q])); break;
    case 1: st.push_back(fem::pw(fidx[q] < 0 ? out : fields[fidx[q]])); break;
    case 6: st.back() = -st.back(); break;
    default: {
      fem::Pw b = st.back();
      st.pop_back();
      fem::Pw a = st.back();
      st.back() = ops[q] == 2 ? a + b : ops[q] == 3 ? a - b : ops[q] == 4 ? a * b : a / b;
    }
    }
  }
  return st.back();
}
} // namespace

extern "C" {

// fem::pointwise (fem/assemble.hpp:252-314) on a Set of `size` nodes of `dim`
// components; out in/out.
int ref_pointwise(int size, int dim, int assign, const int32_t* ops, const int32_t* fidx, const double* vals,
                  int nprog, int nfields, const double* const* fields, double* out) {
  try {
    auto set = make_set(size, "nodes");
    auto o = make_dat(set, dim, "out");
    std::memcpy(o->mutable_view().data(), out, sizeof(double) * static_cast<size_t>(size) * dim);
    std::vector<DatPtr> fs;
    for (int k = 0; k < nfields; ++k) {
      fs.push_back(make_dat(set, dim, "field"));
      std::memcpy(fs.back()->mutable_view().data(), fields[k], sizeof(double) * static_cast<size_t>(size) * dim);
    }
    const auto op = assign == 0 ? fem::PwOp::Assign : assign == 1 ? fem::PwOp::Add : fem::PwOp::Sub;
    fem::pointwise(o, op, pw_from_program(ops, fidx, vals, nprog, fs, o));
    std::memcpy(out, o->view().data(), sizeof(double) * static_cast<size_t>(size) * dim);
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

// fem::apply_dirichlet / apply_dirichlet_rows (fem/assemble.hpp:54-79) with a
// DirichletBC (fem/bc.hpp) on a node set of nrows nodes; values / rhs in-out.
int ref_apply_dirichlet(int nrows, const int64_t* rp, const int32_t* ci, double* values, double* rhs,
                        const int32_t* nodes, int nn, const double* node_values, double constant) {
  try {
    auto A = mat_from_csr(nrows, nrows, rp, ci, values);
    auto space = std::make_shared<fem::FunctionSpace>();
    space->node_set = make_set(nrows, "nodes");
    fem::DirichletBC bc;
    bc.space = space;
    bc.constant = constant;
    if (node_values) {
      bc.function = std::make_shared<fem::Function>();
      bc.function->space = space;
      bc.function->dat = make_dat(space->node_set, 1, "bc");
      std::memcpy(bc.function->dat->mutable_view().data(), node_values, sizeof(double) * nrows);
    }
    bc.nodes.assign(nodes, nodes + nn);
    int code = 0;
    try {
      if (rhs) {
        auto b = make_dat(space->node_set, 1, "rhs");
        std::memcpy(b->mutable_view().data(), rhs, sizeof(double) * nrows);
        try {
          fem::apply_dirichlet(*A, *b, bc);
        } catch (const Error& e) {
          code = fail_code(e);
        }
        std::memcpy(rhs, b->view().data(), sizeof(double) * nrows);
      } else {
        fem::apply_dirichlet_rows(*A, bc);
      }
    } catch (const Error& e) {
      code = fail_code(e);
    }
    std::memcpy(values, A->values().data(), sizeof(double) * static_cast<size_t>(rp[nrows]));
    return code;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

} // extern "C"

#ifdef LOAM_REF_HAVE_BENCH
extern "C" {
// bench::run_wave (bench.hpp:222-300): the reference's explicit wave loop.
// samples: [cap x 4] rows (t, |p|_inf, |phi|_inf, energy) every 100 steps.
int ref_run_wave(int n, double dt, double T, int cap, double* samples, int32_t* nsamples) {
  try {
    auto r = bench::run_wave(n, dt, T, 1);
    const int m = std::min<int>(cap, static_cast<int>(r.sample_times.size()));
    for (int k = 0; k < m; ++k) {
      samples[4 * k] = r.sample_times[k];
      samples[4 * k + 1] = r.norm_p[k];
      samples[4 * k + 2] = r.norm_phi[k];
      samples[4 * k + 3] = r.energy[k];
    }
    *nsamples = m;
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}
} // extern "C"
#endif

extern "C" {
// mesh.hpp:48-89 derive_exterior_facets (markers none): returns the facet
// count; facet_vertices [n x gdim] and facet_cell [n x 2] malloc'ed (ref_free).
int ref_exterior_facets(int gdim, int ncells, int nv, const int32_t* cv, int32_t** fverts, int32_t** fcell) {
  try {
    std::vector<double> coords(static_cast<size_t>(nv) * gdim, 0.0);
    auto mesh = mesh_from_arrays(gdim, ncells, nv, cv, coords.data(), true);
    std::vector<int32_t> fc;
    for (auto& pr : mesh->facet_cell) {
      fc.push_back(pr.first);
      fc.push_back(pr.second);
    }
    *fverts = copy_out(std::vector<int32_t>(mesh->facet_vertex_map->values().begin(),
                                            mesh->facet_vertex_map->values().end()));
    *fcell = copy_out(fc);
    return static_cast<int>(mesh->facet_cell.size());
  } catch (const Error& e) {
    return -fail_code(e);
  }
}
} // extern "C"

extern "C" {
// topology.hpp:131-178 rcm_order over CSR adjacency lists; 0 or -err.
int ref_rcm_order(int n, const int64_t* rp, const int32_t* ci, int32_t* order) {
  try {
    std::vector<std::vector<int>> adj(n);
    for (int u = 0; u < n; ++u) adj[u].assign(ci + rp[u], ci + rp[u + 1]);
    const auto r = rcm_order(n, adj);
    std::copy(r.begin(), r.end(), order);
    return 0;
  } catch (const Error& e) {
    return -fail_code(e);
  }
}

// mesh.hpp:350-362 vertex_adjacency + 364-396 reorder on a mesh built from
// arrays: writes perm [nv], the renumbered coords [nv x gdim] and cv.
int ref_reorder(int gdim, int ncells, int nv, const int32_t* cv, const double* coords, int32_t* perm,
                double* coords_out, int32_t* cv_out) {
  try {
    auto mesh = mesh_from_arrays(gdim, ncells, nv, cv, coords, true);
    auto [out, p] = reorder(*mesh);
    std::copy(p.begin(), p.end(), perm);
    auto x = out->coordinates->view();
    std::copy(x.begin(), x.end(), coords_out);
    const auto& m = out->cell_vertex_map->values();
    std::copy(m.begin(), m.end(), cv_out);
    return 0;
  } catch (const Error& e) {
    return -fail_code(e);
  }
}
} // extern "C"
