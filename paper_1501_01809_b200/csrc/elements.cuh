// elements.cuh -- element kernels of the form catalogue, B200 (sm_100a) device code.
//
// The reference generates one quadrature-loop AST per form and interprets it
// (fem/form.hpp:201-320 -> kernel.hpp:482-495).  For affine simplices every
// catalogue integrand is a polynomial in the barycentric coordinates lambda_k
// whose gradients g_k = grad(lambda_k) are constant per cell, so each local
// entry is an exact closed form in
//     V = |detJ| * |reference cell|      (form.hpp:157, quadrature weights sum to |ref|)
//     g_k (physical barycentric gradients; g_k[a] = K_{a,k-1}, K = J^{-T}, form.hpp:139-178)
// and a few rational integrals int(lambda^alpha) = V d! alpha! / (|alpha|+d)!.
// The results equal the reference's quadrature sums up to rounding (the rules
// are exact for these degrees, element.hpp:31-33); parity is checked at 1e-12.
//
// Every form exposes a ROW functor -- local row i of the element tensor,
// i possibly thread-dependent -- used by the owner-computes gather
// (engine.cu), and the full tensor is the row functor unrolled over i.
#pragma once
#include <type_traits>
#include <cstdint>

namespace loam_gpu {

// Catalogue forms; numbering shared with oracle/loam_oracle.h (orc_form).
// Forms whose RD x CD node blocks are structurally diagonal (component-wise
// operators such as nu grad u : grad v) declare DIAG_BLOCK: a scatter may skip
// the off-diagonal components (they are zero in every element row).
template <class F, class = void>
struct diag_block : std::false_type {};
template <class F>
struct diag_block<F, std::void_t<decltype(F::DIAG_BLOCK)>> : std::bool_constant<F::DIAG_BLOCK> {};

enum FormId : int {
  F_MASS = 0,
  F_STIFFNESS = 1,
  F_HELMHOLTZ = 2,
  F_MASS_ACTION = 3,
  F_STIFFNESS_ACTION = 4,
  F_HELMHOLTZ_ACTION = 5,
  F_ELASTICITY = 6,
  F_STOKES_A = 7,
  F_STOKES_B = 8,
  F_STOKES_BT = 9,
};

// Rational barycentric integrals divided by V (d = spatial dimension):
//   qint(x,y) = int l_x l_y / V          (1+delta)/((d+1)(d+2))
//   eint(a,x) = int (4 l_a - 1) l_x / V
// (int l^alpha = V d! alpha! / (|alpha|+d)!), plus the P2 mass constants below.
template <int D>
struct Simplex;

template <>
struct Simplex<2> {
  // q: 2/4! *2 = 1/6 ; 1/12 ; e_same = 4/6 - 1/3 ; e_diff = 4/12 - 1/3
  static constexpr double q_same = 1.0 / 6, q_diff = 1.0 / 12;
  static constexpr double l1 = 1.0 / 3;
  static constexpr double ref_measure = 0.5;
  static constexpr int NV = 3, NE = 3;
  // local edge k of the P2 row -> vertex pair (space.hpp:66-71): (1,2),(0,2),(0,1)
  __host__ __device__ static constexpr int edge_a(int k) { return k == 0 ? 1 : 0; }
  __host__ __device__ static constexpr int edge_b(int k) { return k == 2 ? 1 : 2; }
};

template <>
struct Simplex<3> {
  static constexpr double q_same = 1.0 / 10, q_diff = 1.0 / 20;
  static constexpr double l1 = 1.0 / 4;
  static constexpr double ref_measure = 1.0 / 6;
  static constexpr int NV = 4, NE = 6;
  // extension: (2,3),(1,3),(1,2),(0,3),(0,2),(0,1) -- UFC order; restricted to
  // the face opposite vertex 3 it reproduces the triangle order above.
  __host__ __device__ static constexpr int edge_a(int k) {
    return k == 0 ? 2 : (k == 1 || k == 2) ? 1 : 0;
  }
  __host__ __device__ static constexpr int edge_b(int k) {
    return (k == 0 || k == 1 || k == 3) ? 3 : (k == 2 || k == 4) ? 2 : 1;
  }
};

// int l_x l_y / V
template <int D>
__host__ __device__ __forceinline__ double qint(int x, int y) {
  return x == y ? Simplex<D>::q_same : Simplex<D>::q_diff;
}
// int (4 l_a - 1) l_x / V
template <int D>
__host__ __device__ __forceinline__ double eint(int a, int x) {
  return 4.0 * qint<D>(a, x) - Simplex<D>::l1;
}

// ---------------------------------------------------------------------------
// Geometry: J_ab = X[b+1][a] - X[0][a] (form.hpp:143-146), K = J^{-T}
// (form.hpp:160-177), V = |detJ| * |ref| (form.hpp:157).

// 0.5 / x (x > 0 a doubled triangle area): fast_rcp with the halving done on
// the seed's exponent by an integer add (exact for normal values), so it costs
// the integer pipe instead of an FP64 multiply.
__device__ __forceinline__ double fast_half_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  const double rh = __hiloint2double(__double2hiint(r) - 0x00100000, __double2loint(r));
  return fma(rh, fma(e, e, e), rh);
}

template <int D>
struct Geom {
  double g[D + 1][D]; // physical barycentric gradients
  double V;
};

// 1/x to within an ulp without the IEEE-division slow path (x is a nonzero,
// finite Jacobian determinant): hardware seed r0 = (1 - eps)/x, |eps| < 2^-20,
// and one third-order correction r0 (1 + e + e^2), e = 1 - x r0 = eps, whose
// residual is eps^3 < 2^-60 (three FMAs; two Newton steps take four).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

template <int D>
__device__ __forceinline__ void geometry(const double (&X)[D + 1][D], Geom<D>& G) {
  if constexpr (D == 2) {
    const double J00 = X[1][0] - X[0][0], J01 = X[2][0] - X[0][0];
    const double J10 = X[1][1] - X[0][1], J11 = X[2][1] - X[0][1];
    const double det = J00 * J11 - J01 * J10;
    const double r = fast_rcp(det);
    // K = [[J11, -J10], [-J01, J00]] / det ; g_k[a] = K[a][k-1]
    G.g[1][0] = J11 * r;
    G.g[1][1] = -J01 * r;
    G.g[2][0] = -J10 * r;
    G.g[2][1] = J00 * r;
    G.g[0][0] = -(G.g[1][0] + G.g[2][0]);
    G.g[0][1] = -(G.g[1][1] + G.g[2][1]);
    G.V = fabs(det) * 0.5;
  } else {
    double J[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) J[a][b] = X[b + 1][a] - X[0][a];
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = -(J[1][0] * J[2][2] - J[1][2] * J[2][0]);
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double c10 = -(J[0][1] * J[2][2] - J[0][2] * J[2][1]);
    const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    const double c12 = -(J[0][0] * J[2][1] - J[0][1] * J[2][0]);
    const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    const double c21 = -(J[0][0] * J[1][2] - J[0][2] * J[1][0]);
    const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double r = fast_rcp(det);
    // g_k[a] = K[a][k-1] = c[a][k-1] / det
    G.g[1][0] = c00 * r; G.g[1][1] = c10 * r; G.g[1][2] = c20 * r;
    G.g[2][0] = c01 * r; G.g[2][1] = c11 * r; G.g[2][2] = c21 * r;
    G.g[3][0] = c02 * r; G.g[3][1] = c12 * r; G.g[3][2] = c22 * r;
#pragma unroll
    for (int a = 0; a < 3; ++a) G.g[0][a] = -(G.g[1][a] + G.g[2][a] + G.g[3][a]);
    G.V = fabs(det) * (1.0 / 6.0);
  }
}

template <int D>
__device__ __forceinline__ double dot(const double* a, const double* b) {
  double s = a[0] * b[0];
#pragma unroll
  for (int k = 1; k < D; ++k) s = fma(a[k], b[k], s);
  return s;
}

// Select vector k of g with a runtime k without dynamic register indexing.
template <int D>
__device__ __forceinline__ void sel(const Geom<D>& G, int k, double (&out)[D]) {
#pragma unroll
  for (int a = 0; a < D; ++a) out[a] = G.g[0][a];
#pragma unroll
  for (int m = 1; m <= D; ++m)
    if (k == m)
#pragma unroll
      for (int a = 0; a < D; ++a) out[a] = G.g[m][a];
}

// ---------------------------------------------------------------------------
// Scalar Lagrange P1 / P2: entries of stiffness (grad.grad) and mass.

// P1: int grad l_i . grad l_j = V g_i.g_j ; int l_i l_j = V qint(i,j)

// P2 basis: node n < NV is vertex n with phi = l_n(2 l_n - 1), grad = (4 l_n - 1) g_n;
// node NV+k is edge (a,b) with phi = 4 l_a l_b, grad = 4 (l_b g_a + l_a g_b).
// int grad phi_i . grad phi_j / V is a combination of D_kl = g_k.g_l with
// rational weights.  Row state: the i-dependent vectors, selected once per row.
template <int D>
struct P2Row {
  int i, a, b;        // vertex row: a = i; edge row: (a, b)
  bool vertex;
  double ga[D], gb[D];
  __device__ __forceinline__ P2Row(const Geom<D>& G, int i_) : i(i_) {
    constexpr int NV = Simplex<D>::NV;
    vertex = i < NV;
    a = vertex ? i : Simplex<D>::edge_a(i - NV);
    b = vertex ? i : Simplex<D>::edge_b(i - NV);
    sel<D>(G, a, ga);
    sel<D>(G, b, gb);
  }
  // stiffness entry (i, j) for a compile-time j, times 1/V
  __device__ __forceinline__ double stiff(const Geom<D>& G, int j) const {
    constexpr int NV = Simplex<D>::NV;
    if (vertex) {
      if (j < NV) {
        const double c = i == j ? 16.0 * Simplex<D>::q_same - 8.0 * Simplex<D>::l1 + 1.0
                                : 16.0 * Simplex<D>::q_diff - 8.0 * Simplex<D>::l1 + 1.0;
        return c * dot<D>(ga, G.g[j]);
      }
      const int c = Simplex<D>::edge_a(j - NV), d = Simplex<D>::edge_b(j - NV);
      return 4.0 * (eint<D>(a, d) * dot<D>(ga, G.g[c]) + eint<D>(a, c) * dot<D>(ga, G.g[d]));
    }
    if (j < NV)
      return 4.0 * (eint<D>(j, b) * dot<D>(ga, G.g[j]) + eint<D>(j, a) * dot<D>(gb, G.g[j]));
    const int c = Simplex<D>::edge_a(j - NV), d = Simplex<D>::edge_b(j - NV);
    return 16.0 * (qint<D>(b, d) * dot<D>(ga, G.g[c]) + qint<D>(b, c) * dot<D>(ga, G.g[d]) +
                   qint<D>(a, d) * dot<D>(gb, G.g[c]) + qint<D>(a, c) * dot<D>(gb, G.g[d]));
  }
};


// int phi_i phi_j / V for P2 (exact rationals, classified by index coincidence).
template <int D>
__host__ __device__ constexpr double p2_mass_const(int kind);
// kinds: 0 vv diag, 1 vv off, 2 ve vertex-in-edge, 3 ve vertex-not-in-edge,
//        4 ee same, 5 ee sharing one vertex, 6 ee disjoint
template <>
__host__ __device__ constexpr double p2_mass_const<2>(int kind) {
  // triangle: diag 6/180, off -1/180, ve in 0, ve out -4/180, ee same 32/180, share 16/180
  return kind == 0 ? 6.0 / 180 : kind == 1 ? -1.0 / 180 : kind == 2 ? 0.0 : kind == 3 ? -4.0 / 180
       : kind == 4 ? 32.0 / 180 : kind == 5 ? 16.0 / 180 : 0.0;
}
template <>
__host__ __device__ constexpr double p2_mass_const<3>(int kind) {
  // tetrahedron (x 1/420): diag 6, off 1, ve in -4, ve out -6, ee same 32, share 16, disjoint 8
  return kind == 0 ? 6.0 / 420 : kind == 1 ? 1.0 / 420 : kind == 2 ? -4.0 / 420 : kind == 3 ? -6.0 / 420
       : kind == 4 ? 32.0 / 420 : kind == 5 ? 16.0 / 420 : 8.0 / 420;
}

template <int D>
__host__ __device__ __forceinline__ int p2_mass_kind(int i, int j) {
  constexpr int NV = Simplex<D>::NV;
  if (i < NV && j < NV) return i == j ? 0 : 1;
  if (i < NV || j < NV) {
    const int v = i < NV ? i : j, e = (i < NV ? j : i) - NV;
    return (Simplex<D>::edge_a(e) == v || Simplex<D>::edge_b(e) == v) ? 2 : 3;
  }
  const int a = Simplex<D>::edge_a(i - NV), b = Simplex<D>::edge_b(i - NV);
  const int c = Simplex<D>::edge_a(j - NV), d = Simplex<D>::edge_b(j - NV);
  const int shared = (a == c) + (a == d) + (b == c) + (b == d);
  return i == j ? 4 : shared == 1 ? 5 : 6;
}

// Row i (runtime) of the P2 stiffness K_ij = int grad phi_i . grad phi_j / V
// and mass M_ij = int phi_i phi_j / V tensors for every compile-time j: one
// vertex/edge branch per row, the dot products g_a . g_m shared by the whole
// row, and the rational constants selected by index coincidence (same
// integrals as P2Row::stiff / p2_mass_const, evaluated without per-entry
// branching).
template <int D, bool STIFF, bool MASS>
__device__ __forceinline__ void p2_rows(int i, const Geom<D>& G, double* K, double* M) {
  constexpr int NV = Simplex<D>::NV, NE = Simplex<D>::NE;
  constexpr double qs = Simplex<D>::q_same, qd = Simplex<D>::q_diff, l1 = Simplex<D>::l1;
  constexpr double cs = 16.0 * qs - 8.0 * l1 + 1.0, co = 16.0 * qd - 8.0 * l1 + 1.0;
  constexpr double es = 4.0 * qs - l1, ed = 4.0 * qd - l1;
  constexpr double m0 = p2_mass_const<D>(0), m1 = p2_mass_const<D>(1), m2 = p2_mass_const<D>(2),
                   m3 = p2_mass_const<D>(3), m4 = p2_mass_const<D>(4), m5 = p2_mass_const<D>(5),
                   m6 = p2_mass_const<D>(6);
  if (i < NV) {
    const int v = i;
    if constexpr (STIFF) {
      double gv[D], dv[NV];
      sel<D>(G, v, gv);
#pragma unroll
      for (int m = 0; m < NV; ++m) dv[m] = dot<D>(gv, G.g[m]);
#pragma unroll
      for (int j = 0; j < NV; ++j) K[j] = (v == j ? cs : co) * dv[j];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int a = Simplex<D>::edge_a(e), b = Simplex<D>::edge_b(e);
        K[NV + e] = 4.0 * ((v == b ? es : ed) * dv[a] + (v == a ? es : ed) * dv[b]);
      }
    }
    if constexpr (MASS) {
#pragma unroll
      for (int j = 0; j < NV; ++j) M[j] = v == j ? m0 : m1;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        M[NV + e] = (Simplex<D>::edge_a(e) == v || Simplex<D>::edge_b(e) == v) ? m2 : m3;
    }
  } else {
    const int e = i - NV;
    const int a = Simplex<D>::edge_a(e), b = Simplex<D>::edge_b(e);
    if constexpr (STIFF) {
      double ga[D], gb[D], da[NV], db[NV];
      sel<D>(G, a, ga);
      sel<D>(G, b, gb);
#pragma unroll
      for (int m = 0; m < NV; ++m) {
        da[m] = dot<D>(ga, G.g[m]);
        db[m] = dot<D>(gb, G.g[m]);
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) K[j] = 4.0 * ((j == b ? es : ed) * da[j] + (j == a ? es : ed) * db[j]);
#pragma unroll
      for (int f = 0; f < NE; ++f) {
        const int c = Simplex<D>::edge_a(f), d = Simplex<D>::edge_b(f);
        K[NV + f] = 16.0 * ((b == d ? qs : qd) * da[c] + (b == c ? qs : qd) * da[d] + (a == d ? qs : qd) * db[c] +
                            (a == c ? qs : qd) * db[d]);
      }
    }
    if constexpr (MASS) {
#pragma unroll
      for (int j = 0; j < NV; ++j) M[j] = (j == a || j == b) ? m2 : m3;
#pragma unroll
      for (int f = 0; f < NE; ++f) {
        const int c = Simplex<D>::edge_a(f), d = Simplex<D>::edge_b(f);
        const int shared = (a == c) + (a == d) + (b == c) + (b == d);
        M[NV + f] = e == f ? m4 : (shared == 1 ? m5 : m6);
      }
    }
  }
}

template <int D, int P>
struct Lagrange {
  static constexpr int N = P == 1 ? D + 1 : (D == 2 ? 6 : 10);
};

// ---------------------------------------------------------------------------
// Form traits.  For each form:
//   NR, NC       local row / column count of the staged tensor (A extents)
//   NRN, NCN     node arity of the row / column maps (NR = NRN*RD)
//   RD, CD       dof expansion of rows / columns (vector spaces)
//   HAS_COEFF    linear (action) forms read a coefficient through the test map
//   row(i, G, C, prm, out)   out[0..NC) = row i of the tensor (RD=CD=1 scalar case)
// Vector forms produce the node-row block: rows (i, 0..RD), cols NC.

struct FormParams {
  double p[4];
};

template <int FORM, int D, int P>
struct FormT;

// Bilinear scalar forms: mass / stiffness / helmholtz (form.hpp:263-283)
template <int FORM, int D, int P>
struct ScalarBilinear {
  static constexpr int N = Lagrange<D, P>::N;
  static constexpr int NR = N, NC = N, NRN = N, NCN = N, RD = 1, CD = 1, GD = D;
  static constexpr int ID = FORM, DEG = P;
  static constexpr bool HAS_COEFF = false, BILINEAR = true;
  static constexpr int NCOEFF = 0;
  __device__ __forceinline__ static void row(int i, const Geom<D>& G, const double*,
                                             const FormParams& prm, double* out) {
    if constexpr (P == 1) {
      double gi[D];
      sel<D>(G, i, gi);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double k = dot<D>(gi, G.g[j]), m = qint<D>(i, j);
        double v;
        if constexpr (FORM == F_MASS) v = m;
        else if constexpr (FORM == F_STIFFNESS) v = k;
        else v = fma(prm.p[0], m, k);
        out[j] = G.V * v;
      }
    } else {
      double K[N], M[N];
      p2_rows<D, FORM != F_MASS, FORM != F_STIFFNESS>(i, G, K, M);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double v;
        if constexpr (FORM == F_MASS) v = M[j];
        else if constexpr (FORM == F_STIFFNESS) v = K[j];
        else v = fma(prm.p[0], M[j], K[j]);
        out[j] = G.V * v;
      }
    }
  }
};
template <int D, int P> struct FormT<F_MASS, D, P> : ScalarBilinear<F_MASS, D, P> {};
template <int D, int P> struct FormT<F_STIFFNESS, D, P> : ScalarBilinear<F_STIFFNESS, D, P> {};
template <int D, int P> struct FormT<F_HELMHOLTZ, D, P> : ScalarBilinear<F_HELMHOLTZ, D, P> {};

// Linear action forms: b_i = sum_j A_ij C_j (form.hpp:288-312); helmholtz
// action = stiffness action + kappa * mass action in one loop.
template <int FORM, int D, int P>
struct ScalarAction {
  static constexpr int N = Lagrange<D, P>::N;
  static constexpr int NR = N, NC = 1, NRN = N, NCN = 0, RD = 1, CD = 1, GD = D;
  static constexpr int ID = FORM, DEG = P;
  static constexpr bool HAS_COEFF = true, BILINEAR = false;
  static constexpr int NCOEFF = N;
  __device__ __forceinline__ static void row(int i, const Geom<D>& G, const double* C,
                                             const FormParams& prm, double* out) {
    if constexpr (P == 1) {
      double gi[D], gu[D];
      sel<D>(G, i, gi);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s = C[0] * G.g[0][a];
#pragma unroll
        for (int k = 1; k < N; ++k) s = fma(C[k], G.g[k][a], s);
        gu[a] = s;
      }
      double b = 0.0;
      if constexpr (FORM != F_MASS_ACTION) b = G.V * dot<D>(gi, gu);
      if constexpr (FORM != F_STIFFNESS_ACTION) {
        double sum = C[0], ci = C[0];
#pragma unroll
        for (int k = 1; k < N; ++k) {
          sum += C[k];
          if (k == i) ci = C[k];
        }
        // int l_i sum_k C_k l_k = V (q_diff sum_k C_k + (q_same - q_diff) C_i)
        const double m = G.V * fma(Simplex<D>::q_same - Simplex<D>::q_diff, ci, Simplex<D>::q_diff * sum);
        b = FORM == F_MASS_ACTION ? m : fma(prm.p[0], m, b);
      }
      out[0] = b;
    } else {
      double K[N], M[N];
      p2_rows<D, FORM != F_MASS_ACTION, FORM != F_STIFFNESS_ACTION>(i, G, K, M);
      double b = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double a;
        if constexpr (FORM == F_MASS_ACTION) a = M[j];
        else if constexpr (FORM == F_STIFFNESS_ACTION) a = K[j];
        else a = fma(prm.p[0], M[j], K[j]);
        b = fma(a, C[j], b);
      }
      out[0] = G.V * b;
    }
  }
};
template <int D, int P> struct FormT<F_MASS_ACTION, D, P> : ScalarAction<F_MASS_ACTION, D, P> {};
template <int D, int P> struct FormT<F_STIFFNESS_ACTION, D, P> : ScalarAction<F_STIFFNESS_ACTION, D, P> {};
template <int D, int P> struct FormT<F_HELMHOLTZ_ACTION, D, P> : ScalarAction<F_HELMHOLTZ_ACTION, D, P> {};

// Linear elasticity, vector P1 tet (config 4): a(u,v) = int 2 mu eps(u):eps(v)
// + lambda div u div v.  Local dof (a,d) = a*3+d.  Entry
//   V [ mu d_de (g_a.g_b) + mu g_a[e] g_b[d] + lambda g_a[d] g_b[e] ].
template <>
struct FormT<F_ELASTICITY, 3, 1> {
  static constexpr int ID = F_ELASTICITY;
  static constexpr int NR = 12, NC = 12, NRN = 4, NCN = 4, RD = 3, CD = 3, GD = 3;
  static constexpr bool HAS_COEFF = false, BILINEAR = true;
  static constexpr int NCOEFF = 0;
  // out: RD x NC block for node row a
  __device__ __forceinline__ static void row(int a, const Geom<3>& G, const double*,
                                             const FormParams& prm, double* out) {
    const double lam = prm.p[0], mu = prm.p[1];
    double ga[3];
    sel<3>(G, a, ga);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double gg = mu * dot<3>(ga, G.g[b]);
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          double v = fma(mu * ga[e], G.g[b][d], lam * ga[d] * G.g[b][e]);
          if (d == e) v += gg;
          out[d * 12 + b * 3 + e] = G.V * v;
        }
    }
  }
  // tensor row (a, d) only: used when one lane owns one dof row
  __device__ __forceinline__ static void subrow(int a, int d, const Geom<3>& G, const double*,
                                                const FormParams& prm, double* out) {
    const double lam = prm.p[0], mu = prm.p[1];
    double ga[3];
    sel<3>(G, a, ga);
    const double gad = d == 0 ? ga[0] : (d == 1 ? ga[1] : ga[2]);
    double mga[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) mga[k] = mu * ga[k] * G.V;
    const double lgad = lam * gad * G.V;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double gbd = d == 0 ? G.g[b][0] : (d == 1 ? G.g[b][1] : G.g[b][2]);
      const double gg = dot<3>(mga, G.g[b]);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        double v = fma(mga[e], gbd, lgad * G.g[b][e]);
        if (d == e) v += gg;
        out[b * 3 + e] = v;
      }
    }
  }
};

// Taylor-Hood Stokes blocks (config 5), velocity vector P2 tri (dof (b,e) = b*2+e),
// pressure P1 tri.
//   A  = nu int grad u : grad v      (component-diagonal)           12 x 12
//   B  = - int q div u               pressure rows, velocity cols   3 x 12
//   BT = B^T                         velocity rows, pressure cols   12 x 3
template <>
struct FormT<F_STOKES_A, 2, 2> {
  static constexpr int ID = F_STOKES_A;
  static constexpr int NR = 12, NC = 12, NRN = 6, NCN = 6, RD = 2, CD = 2, GD = 2;
  static constexpr bool HAS_COEFF = false, BILINEAR = true;
  static constexpr bool DIAG_BLOCK = true; // (d, c) blocks vanish for d != c
  static constexpr int NCOEFF = 0;
  __device__ __forceinline__ static void row(int a, const Geom<2>& G, const double*,
                                             const FormParams& prm, double* out) {
    double K[6];
    p2_rows<2, true, false>(a, G, K, nullptr);
    const double scale = prm.p[0] * G.V;
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const double s = scale * K[b];
      out[0 * 12 + b * 2 + 0] = s;
      out[0 * 12 + b * 2 + 1] = 0.0;
      out[1 * 12 + b * 2 + 0] = 0.0;
      out[1 * 12 + b * 2 + 1] = s;
    }
  }
  __device__ __forceinline__ static void subrow(int a, int d, const Geom<2>& G, const double*,
                                                const FormParams& prm, double* out) {
    double K[6];
    p2_rows<2, true, false>(a, G, K, nullptr);
    const double scale = prm.p[0] * G.V;
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const double s = scale * K[b];
      out[b * 2 + 0] = d == 0 ? s : 0.0;
      out[b * 2 + 1] = d == 1 ? s : 0.0;
    }
  }
};

// int l_p d_e phi_b / V for pressure basis p (P1) and velocity node b (P2):
//   vertex b: (4 l_b - 1) g_b[e] -> eint(b,p) g_b[e]
//   edge (x,y): 4 (l_y g_x[e] + l_x g_y[e]) -> 4 (q(p,y) g_x[e] + q(p,x) g_y[e])
template <>
struct FormT<F_STOKES_B, 2, 2> {
  static constexpr int ID = F_STOKES_B;
  static constexpr int NR = 3, NC = 12, NRN = 3, NCN = 6, RD = 1, CD = 2, GD = 2;
  static constexpr bool HAS_COEFF = false, BILINEAR = true;
  static constexpr int NCOEFF = 0;
  __device__ __forceinline__ static void row(int p, const Geom<2>& G, const double*,
                                             const FormParams&, double* out) {
#pragma unroll
    for (int b = 0; b < 6; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v;
        if (b < 3) {
          v = eint<2>(b, p) * G.g[b][e];
        } else {
          const int x = Simplex<2>::edge_a(b - 3), y = Simplex<2>::edge_b(b - 3);
          v = 4.0 * (qint<2>(p, y) * G.g[x][e] + qint<2>(p, x) * G.g[y][e]);
        }
        out[b * 2 + e] = -G.V * v;
      }
  }
};

template <>
struct FormT<F_STOKES_BT, 2, 2> {
  static constexpr int ID = F_STOKES_BT;
  static constexpr int NR = 12, NC = 3, NRN = 6, NCN = 3, RD = 2, CD = 1, GD = 2;
  static constexpr bool HAS_COEFF = false, BILINEAR = true;
  static constexpr int NCOEFF = 0;
  __device__ __forceinline__ static void row(int b, const Geom<2>& G, const double*,
                                             const FormParams&, double* out) {
    const P2Row<2> R(G, b); // vertex: ga = g_b ; edge (x,y): ga = g_x, gb = g_y
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const double v = R.vertex ? eint<2>(b, p) * R.ga[e]
                                  : 4.0 * (qint<2>(p, R.b) * R.ga[e] + qint<2>(p, R.a) * R.gb[e]);
        out[e * 3 + p] = -G.V * v;
      }
  }
  __device__ __forceinline__ static void subrow(int b, int e, const Geom<2>& G, const double*,
                                                const FormParams&, double* out) {
    const P2Row<2> R(G, b);
    const double gae = e == 0 ? R.ga[0] : R.ga[1], gbe = e == 0 ? R.gb[0] : R.gb[1];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double v = R.vertex ? eint<2>(b, p) * gae
                                : 4.0 * (qint<2>(p, R.b) * gae + qint<2>(p, R.a) * gbe);
      out[p] = -G.V * v;
    }
  }
};

// Row d of node row i's RD x NC block (the whole row for scalar rows).
template <class F>
__device__ __forceinline__ void form_subrow(int i, int d, const Geom<F::GD>& G, const double* C,
                                            const FormParams& prm, double* out) {
  if constexpr (F::RD == 1) F::row(i, G, C, prm, out);
  else F::subrow(i, d, G, C, prm, out);
}

// Full local tensor (NR x NC, row-major, the staged layout of staged_extents,
// parloop.hpp:63-70): unrolled row functor.  For vector forms node row a
// covers tensor rows a*RD .. a*RD+RD-1.
template <class F>
__device__ __forceinline__ void element_tensor(const Geom<F::GD>& G, const double* C,
                                               const FormParams& prm, double* A) {
#pragma unroll
  for (int a = 0; a < F::NRN; ++a) F::row(a, G, C, prm, A + a * F::RD * F::NC);
}

} // namespace loam_gpu
