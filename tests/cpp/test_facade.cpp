// test_facade.cpp -- the reference's own par_loop tests, restated through the
// C++ drop-in facade (paper_1501_01809_b200/csrc/loam_gpu.hpp).  Each case cites
// the reference test it mirrors (/root/reference/proj/tests/...).  Catch2 is not
// in the image, so a minimal CHECK harness stands in.  Run by
// tests/test_cpp_facade_gpu.py on a B200.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "loam_gpu.hpp"

using namespace loam_gpu;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);            \
    }                                                                         \
  } while (0)

template <class F>
static void expect_error(ErrorKind kind, F&& f, const char* needle = nullptr) {
  try {
    f();
    CHECK(false && "expected an error");
  } catch (const Error& e) {
    CHECK(e.kind() == kind);
    if (needle) CHECK(std::string(e.what()).find(needle) != std::string::npos);
  }
}

struct TwoTriangles { // test_parloop.cpp:13-17
  SetPtr cells = make_set(2, "cells");
  SetPtr vertices = make_set(4, "vertices");
  MapPtr map = make_map(cells, vertices, 3, {0, 1, 2, 1, 3, 2}, "cell_vertex");
};

static void test_direct_loop() { // test_parloop.cpp:46-59
  auto set = make_set(3);
  auto a = make_dat(set, 1, "a"), b = make_dat(set, 1, "b");
  auto bw = b->mutable_view();
  bw[0] = 1; bw[1] = 2; bw[2] = 3;
  execute({kernel("double_direct"), set, {arg(a, Access::WRITE), arg(b, Access::READ)}});
  auto av = a->view();
  CHECK(std::vector<Real>(av.begin(), av.end()) == (std::vector<Real>{2, 4, 6}));
}

static void test_indirect_inc() { // test_parloop.cpp:61-68
  TwoTriangles m;
  auto v = make_dat(m.vertices, 1, "v");
  execute({kernel("add_one"), m.cells, {arg(v, Access::INC, m.map)}});
  auto vv = v->view();
  CHECK(std::vector<Real>(vv.begin(), vv.end()) == (std::vector<Real>{1, 2, 2, 1}));
}

static void test_mat_inc() { // test_parloop.cpp:70-87
  TwoTriangles m;
  auto mat = make_mat(build_sparsity(m.map, m.map));
  execute({kernel("ones_block"), m.cells, {arg(mat, Access::INC, m.map, m.map)}});
  CHECK(mat->at(1, 1) == 2.0 && mat->at(2, 2) == 2.0 && mat->at(0, 0) == 1.0 && mat->at(3, 3) == 1.0);
  double dense[4][4] = {};
  for (int e = 0; e < 2; ++e)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dense[m.map->row(e)[i]][m.map->row(e)[j]] += 1.0;
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) CHECK(mat->at(r, c) == dense[r][c]);
}

static void test_validate() { // test_parloop.cpp:89-149
  TwoTriangles m;
  auto mat = make_mat(build_sparsity(m.map, m.map));
  expect_error(ErrorKind::IllegalAccess,
               [&] { validate({kernel("ones_block"), m.cells, {arg(mat, Access::READ, m.map, m.map)}}); },
               "write-only");
  auto g = make_global(1);
  auto cf = make_dat(m.cells, 1);
  expect_error(ErrorKind::IllegalAccess,
               [&] { validate({kernel("sum"), m.cells, {arg(g, Access::INC), arg(cf, Access::READ)}}); });
  auto v = make_dat(m.vertices, 1, "v");
  auto version = v->version();
  validate({kernel("add_one"), m.cells, {arg(v, Access::INC, m.map)}});
  CHECK(v->version() == version);
  auto other = make_set(5);
  expect_error(ErrorKind::MapSourceMismatch,
               [&] { validate({kernel("add_one"), other, {arg(v, Access::INC, m.map)}}); });
  auto edge_map = make_map(m.cells, m.vertices, 2, {0, 1, 1, 3});
  expect_error(ErrorKind::ShapeMismatch,
               [&] { validate({kernel("add_one"), m.cells, {arg(v, Access::INC, edge_map)}}); });
  expect_error(ErrorKind::IllegalAccess, [&] {
    validate({kernel("double_direct"), m.vertices, {arg(v, Access::WRITE), arg(v, Access::READ)}});
  });
}

static void test_versions_and_write_independence() { // test_parloop.cpp:151-180
  auto set = make_set(3);
  auto a = make_dat(set, 1), b = make_dat(set, 1);
  auto version = b->version();
  execute({kernel("double_direct"), set, {arg(a, Access::WRITE), arg(b, Access::READ)}});
  CHECK(b->version() == version);
  CHECK(a->version() > 0);
  auto s4 = make_set(4);
  auto bb = make_dat(s4, 1);
  {
    auto w = bb->mutable_view();
    for (int i = 0; i < 4; ++i) w[i] = i + 1.0;
  }
  auto run_from = [&](Real fill) {
    auto x = make_dat(s4, 1);
    auto w = x->mutable_view();
    std::fill(w.begin(), w.end(), fill);
    execute({kernel("double_direct"), s4, {arg(x, Access::WRITE), arg(bb, Access::READ)}});
    auto xv = x->view();
    return std::vector<Real>(xv.begin(), xv.end());
  };
  CHECK(run_from(0.0) == run_from(123.456));
}

static void test_canary() { // test_parloop.cpp:182-200
  auto cells = make_set(2), vertices = make_set(5);
  auto map = make_map(cells, vertices, 2, {0, 1, 2, 3});
  auto v = make_dat(vertices, 1);
  v->mutable_view()[4] = -777.0;
  execute({kernel("fill"), cells, {arg(v, Access::WRITE, map)}});
  CHECK(v->view()[4] == -777.0);
  CHECK(v->view()[0] == 1.0);
}

static void test_globals() { // test_parloop.cpp:202-237
  auto set = make_set(100);
  auto field = make_dat(set, 1);
  {
    auto w = field->mutable_view();
    for (int i = 0; i < 100; ++i) w[i] = std::sin(0.37 * i) * 10.0;
  }
  auto g = make_global(1);
  execute({kernel("sum"), set, {arg(g, Access::SUM), arg(field, Access::READ)}});
  Real expect = 0.0, mx = -1e300, mn = 1e300, mag = 0.0;
  for (Real x : field->view()) {
    expect += x;
    mag += std::abs(x);
    mx = std::max(mx, x);
    mn = std::min(mn, x);
  }
  CHECK(std::abs(g->view()[0] - expect) <= 1e-12 * mag);
  auto gmax = make_global(1), gmin = make_global(1);
  execute({kernel("maxval"), set, {arg(gmax, Access::MAX), arg(field, Access::READ)}});
  execute({kernel("maxval"), set, {arg(gmin, Access::MIN), arg(field, Access::READ)}});
  CHECK(gmax->view()[0] == mx && gmin->view()[0] == mn);
}

static void test_rw() { // test_parloop.cpp:357-373
  TwoTriangles m;
  auto v = make_dat(m.vertices, 1);
  {
    auto w = v->mutable_view();
    for (int i = 0; i < 4; ++i) w[i] = 1.0;
  }
  execute({kernel("bump"), m.cells, {arg(v, Access::RW, m.map)}}, 4);
  auto vv = v->view();
  CHECK(std::vector<Real>(vv.begin(), vv.end()) == (std::vector<Real>{2, 3, 3, 2}));
}

static void test_sparsity_and_colouring() { // test_data.cpp:22-62, test_topology.cpp:55-84
  TwoTriangles m;
  auto sp = build_sparsity(m.map, m.map);
  CHECK(sp->nrows() == 4 && sp->ncols() == 4 && sp->nnz() == 14);
  auto s5 = make_set(5);
  auto ident = make_map(s5, s5, 1, {0, 1, 2, 3, 4});
  auto si = build_sparsity(ident, ident);
  CHECK(si->nnz() == 5);
  for (int i = 0; i < 5; ++i) CHECK(si->find(i, i) == i);
  auto c = color_iteration(m.cells, {m.map});
  CHECK(c.colors == (std::vector<int>{0, 1}) && c.num_colors == 2);
  auto fc = make_set(4), fv = make_set(9);
  auto fan = make_map(fc, fv, 3, {0, 1, 2, 0, 3, 4, 0, 5, 6, 0, 7, 8});
  CHECK(color_iteration(fc, {fan}).colors == (std::vector<int>{0, 1, 2, 3}));
  expect_error(ErrorKind::SourceMismatch, [&] { color_iteration(fc, {m.map}); });
}

static void test_outside_sparsity_and_map_range() { // test_data.cpp:93-124, topology.hpp:45-48
  auto cells = make_set(1), verts = make_set(4);
  auto map = make_map(cells, verts, 3, {0, 1, 2});
  auto mat = make_mat(build_sparsity(map, map));
  auto other = make_map(cells, verts, 3, {0, 1, 3});
  expect_error(ErrorKind::OutsideSparsity,
               [&] { execute({kernel("ones_block"), cells, {arg(mat, Access::INC, map, other)}}); }, "3)");
  expect_error(ErrorKind::IndexOutOfRange, [&] { make_map(cells, verts, 3, {0, 1, 4}); });
}

static void test_stiffness_reference_triangle() { // test_fem.cpp:141-161 through an assembled one-cell mesh
  auto cells = make_set(1), verts = make_set(3);
  auto map = make_map(cells, verts, 3, {0, 1, 2});
  auto X = make_dat(verts, 2, "coordinates");
  {
    auto w = X->mutable_view();
    const Real c[6] = {0, 0, 1, 0, 0, 1};
    for (int i = 0; i < 6; ++i) w[i] = c[i];
  }
  auto K = make_mat(build_sparsity(map, map));
  execute({kernel("stiffness_p1_tri"), cells, {arg(K, Access::INC, map, map), arg(X, Access::READ, map)}});
  const Real expected[3][3] = {{1.0, -0.5, -0.5}, {-0.5, 0.5, 0.0}, {-0.5, 0.0, 0.5}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) CHECK(std::abs(K->at(i, j) - expected[i][j]) <= 1e-14);
  auto M = make_mat(build_sparsity(map, map));
  execute({kernel("mass_p1_tri"), cells, {arg(M, Access::INC, map, map), arg(X, Access::READ, map)}});
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) CHECK(std::abs(M->at(i, j) - (i == j ? 2.0 : 1.0) / 24.0) <= 1e-15);
  expect_error(ErrorKind::InvalidArgument, [&] {
    execute({kernel("no_such_kernel"), cells, {arg(K, Access::INC, map, map), arg(X, Access::READ, map)}});
  }, "no CPU fallback");
}

// ---- matrix consumers ----------------------------------------
static MatPtr dense_mat(const std::vector<Real>& entries, int n) { // test_solver.cpp:10-20
  auto nodes = make_set(n);
  auto one = make_set(1);
  std::vector<int> all(n);
  for (int i = 0; i < n; ++i) all[i] = i;
  auto map = make_map(one, nodes, n, all);
  auto mat = make_mat(build_sparsity(map, map));
  mat->addto(all, all, entries, Access::WRITE);
  return mat;
}

static void test_spmv() { // test_data.cpp:175-205
  auto diag = dense_mat({2, 0, 0, 3}, 2);
  std::vector<Real> x{1.0, 1.0};
  CHECK(mat_spmv(*diag, x) == (std::vector<Real>{2.0, 3.0}));
  auto full = dense_mat({4, 1, 1, 3}, 2);
  std::vector<Real> x2{1.0, 2.0};
  CHECK(mat_spmv(*full, x2) == (std::vector<Real>{6.0, 7.0}));
  std::vector<Real> bad{1.0, 2.0, 3.0};
  expect_error(ErrorKind::DimensionMismatch, [&] { mat_spmv(*full, bad); });
}

static void test_block_spmv() { // test_solver.cpp:171-206
  auto A = dense_mat({2, 1, 1, 2}, 2), B = dense_mat({0, 1, 2, 0}, 2), C = dense_mat({1, 1, 0, 1}, 2);
  BlockMat diag;
  diag.blocks[0][0] = A;
  diag.blocks[1][1] = A;
  diag.row_sizes = {2, 2};
  diag.col_sizes = {2, 2};
  std::vector<Real> x{1, 2, 3, 4};
  auto y = block_spmv(diag, x);
  auto Au = mat_spmv(*A, {x.data(), 2}), Av = mat_spmv(*A, {x.data() + 2, 2});
  CHECK(std::vector<Real>(y.begin(), y.begin() + 2) == Au);
  CHECK(std::vector<Real>(y.begin() + 2, y.end()) == Av);
  BlockMat anti;
  anti.blocks[0][1] = B;
  anti.blocks[1][0] = C;
  anti.row_sizes = {2, 2};
  anti.col_sizes = {2, 2};
  auto z = block_spmv(anti, x);
  CHECK(std::vector<Real>(z.begin(), z.begin() + 2) == mat_spmv(*B, {x.data() + 2, 2}));
  CHECK(std::vector<Real>(z.begin() + 2, z.end()) == mat_spmv(*C, {x.data(), 2}));
  std::vector<Real> bad{1, 2, 3};
  expect_error(ErrorKind::DimensionMismatch, [&] { block_spmv(diag, bad); });
}

static void test_cg() { // test_solver.cpp:24-123
  std::vector<Real> e(25, 0.0);
  for (int i = 0; i < 5; ++i) e[i * 5 + i] = 1.0;
  std::vector<Real> b{0.3, 0.1, 0.7, 0.2, 0.9};
  auto [x, rep] = cg_solve(*dense_mat(e, 5), b);
  CHECK(rep.converged && rep.iterations == 1);
  for (int i = 0; i < 5; ++i) CHECK(std::abs(x[i] - b[i]) <= 1e-14);
  auto [x2, rep2] = cg_solve(*dense_mat({4, 1, 1, 3}, 2), std::vector<Real>{1, 2}, {}, 1e-12, 1e-16, 10);
  CHECK(rep2.converged && std::abs(x2[0] - 1.0 / 11) <= 1e-12 && std::abs(x2[1] - 7.0 / 11) <= 1e-12);
  expect_error(ErrorKind::IndefiniteBreakdown, [&] {
    cg_solve(*dense_mat({0, 1, 1, 3}, 2), std::vector<Real>{1, 2}, {}, 1e-10, 1e-15, 10, Preconditioner::Jacobi);
  });
  expect_error(ErrorKind::IndefiniteBreakdown, [&] {
    cg_solve(*dense_mat({1, 0, 0, -1}, 2), std::vector<Real>{1, 1}, {}, 1e-10, 1e-15, 10);
  }, "after 1 iterations");
  // maxit returns the iterate unconverged: B^T B + I, n = 30
  const int n = 30;
  std::vector<Real> Bm(n * n), A(n * n, 0.0), rhs(n);
  unsigned s = 47;
  auto u = [&] { s = s * 1103515245u + 12345u; return (s >> 8) / 16777216.0; };
  for (auto& v : Bm) v = u();
  for (auto& v : rhs) v = u();
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      for (int k = 0; k < n; ++k) A[i * n + j] += Bm[k * n + i] * Bm[k * n + j];
      if (i == j) A[i * n + j] += 1.0;
    }
  auto [x3, rep3] = cg_solve(*dense_mat(A, n), rhs, {}, 1e-14, 0.0, 2);
  CHECK(!rep3.converged && rep3.reason == SolveReport::Reason::maxit && rep3.iterations == 2);
  // block operator [[A, 0], [0, A]] equals two independent solves
  BlockMat op;
  auto Am = dense_mat(A, n);
  op.blocks[0][0] = op.blocks[1][1] = Am;
  op.row_sizes = op.col_sizes = {n, n};
  std::vector<Real> bb(rhs);
  bb.insert(bb.end(), rhs.begin(), rhs.end());
  auto [xb, repb] = cg_solve(op, bb, {}, 1e-10, 1e-16, 200, Preconditioner::Jacobi);
  CHECK(repb.converged);
  auto r = block_spmv(op, xb);
  Real rn = 0.0, bn = 0.0;
  for (size_t i = 0; i < bb.size(); ++i) {
    rn += (bb[i] - r[i]) * (bb[i] - r[i]);
    bn += bb[i] * bb[i];
  }
  CHECK(std::sqrt(rn) <= 1e-10 * std::sqrt(bn) + 1e-12);
}

static void test_rcm() { // test_topology.cpp rcm_order cases
  CHECK(rcm_order(3, {{1}, {0, 2}, {1}}) == (std::vector<int>{2, 1, 0}));
  CHECK(rcm_order(1, {{}}) == (std::vector<int>{0}));
  CHECK(rcm_order(4, {{1, 2, 3}, {0}, {0}, {0}}) == (std::vector<int>{3, 2, 0, 1}));
  expect_error(ErrorKind::AsymmetricAdjacency, [] { rcm_order(2, {{1}, {}}); });
  expect_error(ErrorKind::IndexOutOfRange, [] { rcm_order(2, {{3}, {0}}); });
}

// fem::assemble_blocks (fem/assemble.hpp:439-448): the Taylor-Hood triple through
// execute_blocks (one launch) equals the three loops run one by one.
static void test_execute_blocks_taylor_hood() {
  const int n = 9, nv = (n + 1) * (n + 1), nc = 2 * n * n;
  std::vector<Real> xy(2 * (size_t)nv);
  std::vector<int> cv(3 * (size_t)nc), cn(6 * (size_t)nc);
  CHECK(loam_gpu_unit_square_mesh(n, xy.data(), cv.data()) == 0);
  CHECK(loam_gpu_jitter(2, n, 0.2, 7, xy.data()) == 0);
  CHECK(loam_gpu_p2_cell_node_map(nc, nv, 2, cv.data(), cn.data()) > 0); // (returns the node count)
  int nn = 0;
  for (int x : cn) nn = std::max(nn, x + 1);
  auto cells = make_set(nc), verts = make_set(nv), nodes = make_set(nn);
  auto pm = make_map(cells, verts, 3, cv), vnm = make_map(cells, nodes, 6, cn);
  auto vdm = make_expanded_map(vnm, 2);
  auto X = make_dat(verts, 2, "coordinates");
  {
    auto w = X->mutable_view();
    for (size_t i = 0; i < xy.size(); ++i) w[i] = xy[i];
  }
  auto spA = build_sparsity(vnm, vnm, 2, 2), spB = build_sparsity(pm, vnm, 1, 2), spT = build_sparsity(vnm, pm, 2, 1);
  auto loops = [&](const MatPtr& A, const MatPtr& B, const MatPtr& T) {
    return std::vector<Parloop>{
        {kernel("stokes_a_p2_tri", {1.0}), cells, {arg(A, Access::INC, vdm, vdm), arg(X, Access::READ, pm)}},
        {kernel("stokes_b_p2_tri"), cells, {arg(B, Access::INC, pm, vdm), arg(X, Access::READ, pm)}},
        {kernel("stokes_bt_p2_tri"), cells, {arg(T, Access::INC, vdm, pm), arg(X, Access::READ, pm)}}};
  };
  auto A1 = make_mat(spA), B1 = make_mat(spB), T1 = make_mat(spT);
  for (const Parloop& lp : loops(A1, B1, T1)) execute(lp);
  auto A2 = make_mat(spA), B2 = make_mat(spB), T2 = make_mat(spT);
  execute_blocks(loops(A2, B2, T2)); // plan
  A2->zero();
  B2->zero();
  T2->zero();
  const int64_t before = loam_gpu_launch_count();
  execute_blocks(loops(A2, B2, T2));
  CHECK(loam_gpu_launch_count() - before == 1);
  auto close = [](const std::vector<Real>& a, const std::vector<Real>& b) {
    Real num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      num = std::max(num, std::abs(a[i] - b[i]));
      den = std::max(den, std::abs(b[i]));
    }
    return a.size() == b.size() && num <= 1e-12 * den;
  };
  CHECK(close(A2->values(), A1->values()));
  CHECK(close(B2->values(), B1->values()));
  CHECK(close(T2->values(), T1->values()));
  // B^T really is the transpose of B (to rounding: rows of B and of B^T are owned by different items)
  for (int v = 0; v < nv; v += 7)
    for (int d = 0; d < 2 * nn; d += 11) CHECK(std::abs(B2->at(v, d) - T2->at(d, v)) <= 1e-15);
  // an illegal loop in the list: nothing is written
  auto A3 = make_mat(spA), B3 = make_mat(spB), T3 = make_mat(spT);
  auto bad = loops(A3, B3, T3);
  bad[2].args[0] = arg(T3, Access::INC, vdm, vdm);
  expect_error(ErrorKind::ShapeMismatch, [&] { execute_blocks(bad); });
  for (Real x : A3->values()) CHECK(x == 0.0);
}

int main() {
  loam_gpu_set_option(LOAM_OPT_TEST_KERNELS, 1); // the reference test-suite kernels
  const std::vector<std::pair<const char*, void (*)()>> cases = {
      {"direct loop doubles a field", test_direct_loop},
      {"indirect INC accumulates cell incidence", test_indirect_inc},
      {"mat INC assembles both triangles", test_mat_inc},
      {"validate rejects illegal descriptors", test_validate},
      {"versions / WRITE independence", test_versions_and_write_independence},
      {"kernels observe only staged slots", test_canary},
      {"global reductions", test_globals},
      {"RW indirect updates", test_rw},
      {"sparsity and colouring KATs", test_sparsity_and_colouring},
      {"OutsideSparsity / map range", test_outside_sparsity_and_map_range},
      {"stiffness on the reference triangle", test_stiffness_reference_triangle},
      {"spmv by CSR traversal", test_spmv},
      {"block spmv skips zero blocks and swaps components", test_block_spmv},
      {"cg known answers, breakdown, maxit, block operator", test_cg},
      {"rcm_order known answers and errors", test_rcm},
      {"execute_blocks: Taylor-Hood triple in one launch", test_execute_blocks_taylor_hood},
  };
  for (auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION %s\n", e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
