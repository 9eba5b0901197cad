// test_ref_adapter.cpp -- the REFERENCE's own objects and fem:: callers routed
// to the B200 through include/loam_gpu_ref.hpp, compared with the reference's
// own CPU execution of the same calls.
//
// Built in the container (it needs the reference headers, -I<ref>/proj/include)
// by __graft_entry__.build() / tests/cpp/Makefile into tests/cpp/bin (shipped
// to the GPU box with the snapshot like the .so files); run by
// tests/test_ref_adapter_gpu.py on a B200.  The reference code here is used as
// the checker (loam::execute, fem::assemble_*): test infrastructure only.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "loam/fem/assemble.hpp"
#include "loam/mesh.hpp"
#include "loam_gpu_ref.hpp"

using namespace loam;
using namespace loam::ir;

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
    if (needle && std::string(e.what()).find(needle) == std::string::npos) {
      std::printf("  message was: %s\n", e.what());
      CHECK(false && "message");
    }
  }
}

static double rel_max(const std::vector<Real>& a, const std::vector<Real>& b) {
  if (a.size() != b.size()) return 1e300;
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return den > 0 ? num / den : num;
}

template <class S>
static std::vector<Real> vec(S s) {
  return std::vector<Real>(s.begin(), s.end());
}

// deterministic interior jitter (splitmix64) so the cells are not all congruent
static void jitter(Mesh& mesh, int n, double amp, uint64_t seed) {
  auto x = mesh.coordinates->mutable_view();
  const int d = mesh.dim, nv = mesh.vertices->size();
  const double h = 1.0 / n;
  for (int v = 0; v < nv; ++v) {
    bool interior = true;
    for (int c = 0; c < d; ++c) interior = interior && x[v * d + c] > 1e-12 && x[v * d + c] < 1 - 1e-12;
    if (!interior) continue;
    for (int c = 0; c < d; ++c) {
      seed += 0x9e3779b97f4a7c15ULL;
      uint64_t z = seed;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      z ^= z >> 31;
      x[v * d + c] += (2.0 * ((z >> 11) * 0x1.0p-53) - 1.0) * amp * h;
    }
  }
}

// ---- the reference's par_loop KATs with the reference's own AST kernels ------
struct TwoTriangles { // test_parloop.cpp:13-17
  SetPtr cells = make_set(2, "cells");
  SetPtr vertices = make_set(4, "vertices");
  MapPtr map = make_map(cells, vertices, 3, {0, 1, 2, 1, 3, 2}, "cell_vertex");
};

static KernelPtr add_one_indirect() { // test_parloop.cpp:27-33
  KernelAst ast;
  ast.name = "add_one";
  ast.params = {{"V", {3}}};
  ast.body = {loop("i", 3, {accum("V", {ref("i")}, lit(1.0))})};
  return make_kernel(ast);
}

static KernelPtr ones_block() { // test_parloop.cpp:35-42
  KernelAst ast;
  ast.name = "ones_block";
  ast.params = {{"A", {3, 3}}};
  ast.body = {loop("i", 3, {loop("j", 3, {accum("A", {ref("i"), ref("j")}, lit(1.0))})})};
  return make_kernel(ast);
}

static KernelPtr doubling_direct() { // test_parloop.cpp:19-25
  KernelAst ast;
  ast.name = "double_direct";
  ast.params = {{"A", {1}}, {"B", {1}}};
  ast.body = {assign("A", {lit(0.0)}, lit(2.0) * idx("B", {lit(0.0)}))};
  return make_kernel(ast);
}

static void test_parloop_kats() {
  std::printf("parloop KATs through loam_gpu_ref::execute\n");
  { // test_parloop.cpp:61-68: [1, 2, 2, 1]
    TwoTriangles m;
    auto v = make_dat(m.vertices, 1, "v");
    const auto v0 = v->version();
    loam_gpu_ref::execute({add_one_indirect(), m.cells, {arg(v, Access::INC, m.map)}});
    CHECK(vec(v->view()) == (std::vector<Real>{1, 2, 2, 1}));
    CHECK(v->version() == v0 + 1); // one mutable_view per execute, like loam::execute
    loam_gpu_ref::execute({add_one_indirect(), m.cells, {arg(v, Access::INC, m.map)}});
    CHECK(vec(v->view()) == (std::vector<Real>{2, 4, 4, 2}));
  }
  { // test_parloop.cpp:357-373 style: Mat INC of ones into the map pattern
    TwoTriangles m;
    auto sp = loam_gpu_ref::build_sparsity(m.map, m.map);
    auto ref_sp = build_sparsity(m.map, m.map);
    CHECK(sp->row_offsets() == ref_sp->row_offsets());
    CHECK(sp->col_indices() == ref_sp->col_indices());
    auto A = make_mat(sp, "A"), B = make_mat(ref_sp, "B");
    loam_gpu_ref::execute({ones_block(), m.cells, {arg(A, Access::INC, m.map, m.map)}});
    execute(Parloop{ones_block(), m.cells, {arg(B, Access::INC, m.map, m.map)}});
    CHECK(A->values() == B->values());
    CHECK(A->at(1, 2) == 2.0 && A->at(0, 3) == 0.0);
  }
  { // test_parloop.cpp:46-59 direct loop
    auto set = make_set(3);
    auto a = make_dat(set, 1, "a"), b = make_dat(set, 1, "b");
    auto bw = b->mutable_view();
    bw[0] = 1, bw[1] = 2, bw[2] = 3;
    loam_gpu_ref::execute({doubling_direct(), set, {arg(a, Access::WRITE), arg(b, Access::READ)}});
    CHECK(vec(a->view()) == (std::vector<Real>{2, 4, 6}));
  }
  { // validate runs first, before any mutation, with the reference's messages
    TwoTriangles m;
    auto v = make_dat(m.vertices, 1, "v");
    auto other = make_set(2, "other");
    auto bad = make_map(other, m.vertices, 3, {0, 1, 2, 1, 3, 2}, "bad");
    expect_error(ErrorKind::MapSourceMismatch,
                 [&] { loam_gpu_ref::execute({add_one_indirect(), m.cells, {arg(v, Access::INC, bad)}}); },
                 "source differs from iteration set");
    expect_error(ErrorKind::IllegalAccess, [&] {
      loam_gpu_ref::execute({add_one_indirect(), m.cells, {arg(v, Access::INC, m.map), arg(v, Access::READ, m.map)}});
    });
    CHECK(vec(v->view()) == (std::vector<Real>{0, 0, 0, 0}));
  }
  { // a kernel without a device implementation is an error, not a CPU fallback
    TwoTriangles m;
    auto v = make_dat(m.vertices, 1, "v");
    KernelAst ast;
    ast.name = "not_on_the_device";
    ast.params = {{"V", {3}}};
    ast.body = {loop("i", 3, {accum("V", {ref("i")}, lit(1.0))})};
    expect_error(ErrorKind::InvalidArgument,
                 [&] { loam_gpu_ref::execute({make_kernel(ast), m.cells, {arg(v, Access::INC, m.map)}}); },
                 "no device implementation");
    CHECK(vec(v->view()) == (std::vector<Real>{0, 0, 0, 0}));
  }
  { // OutsideSparsity names the entry (test_data.cpp:110-116 through execute)
    TwoTriangles m;
    auto diag = make_map(m.cells, m.vertices, 1, {0, 1}, "diag");
    auto sp = build_sparsity(diag, diag);
    auto A = make_mat(sp, "A");
    expect_error(ErrorKind::OutsideSparsity, [&] {
      loam_gpu_ref::execute({ones_block(), m.cells, {arg(A, Access::INC, m.map, m.map)}});
    }, "outside sparsity");
  }
}

// ---- fem:: callers: the reference's own assemble_* vs the adapter -----------
static void compare_mat(const char* what, const MatPtr& gpu, const MatPtr& ref, double tol = 1e-12) {
  const bool pattern = gpu->sparsity()->row_offsets() == ref->sparsity()->row_offsets() &&
                       gpu->sparsity()->col_indices() == ref->sparsity()->col_indices();
  const double err = rel_max(gpu->values(), ref->values());
  std::printf("  %-44s nnz %9ld  pattern %s  rel err %.2e\n", what, ref->sparsity()->nnz(),
              pattern ? "bit-exact" : "DIFFERS", err);
  CHECK(pattern);
  CHECK(err <= tol);
}

static void compare_dat(const char* what, const DatPtr& gpu, const DatPtr& ref, double tol = 1e-12) {
  const double err = rel_max(vec(gpu->view()), vec(ref->view()));
  std::printf("  %-44s n %9zu  rel err %.2e\n", what, ref->view().size(), err);
  CHECK(err <= tol);
}

static fem::FunctionPtr random_function(const fem::FunctionSpacePtr& V, uint64_t seed, double lo, double hi) {
  auto f = fem::make_function(V, "u");
  auto x = f->dat->mutable_view();
  for (auto& v : x) {
    seed += 0x9e3779b97f4a7c15ULL;
    uint64_t z = seed;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    v = lo + (hi - lo) * ((z >> 11) * 0x1.0p-53);
  }
  return f;
}

static void test_fem_callers(int n2, int n3) {
  using namespace loam::fem;
  std::printf("fem::assemble_* through the adapter (square %d^2, cube %d^3)\n", n2, n3);
  const int T = 8;
  auto sq = unit_square_mesh(n2);
  jitter(*sq, n2, 0.2, 2);
  auto cube = unit_cube_mesh(n3);
  jitter(*cube, n3, 0.15, 4);
  for (int p : {1, 2}) {
    auto V = make_function_space(sq, p);
    const std::string tag = "P" + std::to_string(p) + " tri ";
    compare_mat((tag + "stiffness (C2 shape)").c_str(), loam_gpu_ref::fem::assemble_matrix(stiffness(V, V)),
                assemble_matrix(stiffness(V, V), {}, T));
    compare_mat((tag + "mass").c_str(), loam_gpu_ref::fem::assemble_matrix(mass(V, V)),
                assemble_matrix(mass(V, V), {}, T));
    compare_mat((tag + "helmholtz kappa=2.5").c_str(), loam_gpu_ref::fem::assemble_matrix(helmholtz(V, V, 2.5)),
                assemble_matrix(helmholtz(V, V, 2.5), {}, T));
    auto u = random_function(V, 1000 + p, 0.0, 1.0);
    compare_dat((tag + "stiffness action").c_str(), loam_gpu_ref::fem::assemble_vector(stiffness_action(V, u)),
                assemble_vector(stiffness_action(V, u), {}, T));
    compare_dat((tag + "mass action").c_str(), loam_gpu_ref::fem::assemble_vector(mass_action(V, u)),
                assemble_vector(mass_action(V, u), {}, T));
    compare_dat((tag + "source (Function density)").c_str(), loam_gpu_ref::fem::assemble_vector(source(V, u)),
                assemble_vector(source(V, u), {}, T));
    compare_dat((tag + "source (constant density 3)").c_str(), loam_gpu_ref::fem::assemble_vector(source(V, 3.0)),
                assemble_vector(source(V, 3.0), {}, T));
  }
  {
    auto V = make_function_space(cube, 1);
    compare_mat("P1 tet stiffness", loam_gpu_ref::fem::assemble_matrix(stiffness(V, V)),
                assemble_matrix(stiffness(V, V), {}, T));
    compare_mat("P1 tet helmholtz kappa=1", loam_gpu_ref::fem::assemble_matrix(helmholtz(V, V, 1.0)),
                assemble_matrix(helmholtz(V, V, 1.0), {}, T));
    auto u = random_function(V, 77, -1.0, 1.0);
    compare_dat("P1 tet stiffness action", loam_gpu_ref::fem::assemble_vector(stiffness_action(V, u)),
                assemble_vector(stiffness_action(V, u), {}, T));
  }
  { // C1 shape: the Helmholtz residual as the reference states it -- two cell
    // loops (stiffness action + kappa * mass action, form.hpp:55-73)
    auto V = make_function_space(sq, 1);
    auto u = random_function(V, 1001, 0.0, 1.0);
    auto g1 = loam_gpu_ref::fem::assemble_vector(stiffness_action(V, u));
    auto g2 = loam_gpu_ref::fem::assemble_vector(mass_action(V, u));
    auto r1 = assemble_vector(stiffness_action(V, u), {}, T);
    auto r2 = assemble_vector(mass_action(V, u), {}, T);
    auto gv = g1->mutable_view();
    auto rv = r1->mutable_view();
    for (size_t i = 0; i < gv.size(); ++i) gv[i] += g2->view()[i], rv[i] += r2->view()[i];
    compare_dat("C1 shape: stiffness action + mass action", g1, r1);
  }
  { // Dirichlet rows through the caller (assemble.hpp:100-101)
    auto V = make_function_space(sq, 1);
    DirichletBC bc = dirichlet_bc(V, 0.0, {1, 2, 3, 4});
    compare_mat("P1 tri stiffness with Dirichlet rows", loam_gpu_ref::fem::assemble_matrix(stiffness(V, V), {bc}),
                assemble_matrix(stiffness(V, V), {bc}, T));
  }
  { // nested blocks (assemble.hpp:439-448, test_fem.cpp:524-566): P2/P1 mixed
    auto V2 = make_function_space(sq, 2);
    auto V1 = make_function_space(sq, 1);
    MixedForm mixed;
    mixed.test = {V2, V1};
    mixed.trial = {V2, V1};
    mixed.blocks[0][0] = std::make_shared<const Form>(stiffness(V2, V2));
    mixed.blocks[1][1] = std::make_shared<const Form>(mass(V1, V1));
    auto g = loam_gpu_ref::fem::assemble_blocks(mixed);
    auto r = assemble_blocks(mixed, T);
    CHECK(g.row_sizes == r.row_sizes && g.col_sizes == r.col_sizes);
    CHECK(!g.blocks[0][1] && !g.blocks[1][0]);
    compare_mat("blocks [0][0] P2 stiffness", g.blocks[0][0], r.blocks[0][0]);
    compare_mat("blocks [1][1] P1 mass", g.blocks[1][1], r.blocks[1][1]);
    std::vector<Real> x(g.ncols());
    for (size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.1 * i);
    const double e = rel_max(block_spmv(g, x), block_spmv(r, x));
    std::printf("  %-44s rel err %.2e\n", "block_spmv of the nested result", e);
    CHECK(e <= 1e-12);
  }
}

int main(int argc, char** argv) {
  const int n2 = argc > 1 ? std::atoi(argv[1]) : 96;
  const int n3 = argc > 2 ? std::atoi(argv[2]) : 10;
  if (!loam_gpu_device_ok()) {
    std::printf("no sm_100 device\n");
    return 2;
  }
  loam_gpu_set_option(LOAM_OPT_TEST_KERNELS, 1); // add_one, ones_block, double_direct
  try {
    test_parloop_kats();
    test_fem_callers(n2, n3);
  } catch (const std::exception& e) {
    std::printf("  UNCAUGHT %s\n", e.what());
    ++g_fail;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
