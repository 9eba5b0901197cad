// patch_kernels.cuh -- row-owner kernels over the cell-patch plan (patch.cuh).
//
// One CTA per patch (persistent over patches).  Per patch:
//   1. stage the window node ids, the tile cells' u16 window slots and the
//      owned-row list in shared memory;
//   2. per TILE CELL (one thread each): gather the vertex coordinates through
//      the window and compute the geometry ONCE (Mats: g_1..g_d and V kept in
//      shared memory; Dats: the whole element vector, computed from the
//      geometry and the coefficients);
//   3. Dats: add the owned entries of each element vector into a per-row
//      shared accumulator, then write every owned node once.
//      Mats: set the bits of each owned pair's column window slots in its
//      row's bitmap and prefix-count it (in-row rank of a column node =
//      popcount of the smaller slots, because the window is sorted by node id
//      like the CSR row, data.hpp:129-136); then one thread per OWNED PAIR
//      evaluates the element row from the shared geometry and adds it into the
//      row's value segment in shared memory; finally the owned rows' CSR
//      segments are written once, warp per row.
// Shared-memory fp64 adds are CAS loops on sm_100a (ATOMS.CAST.SPIN.64);
// contention is low because concurrent pairs rarely share a row, but the
// summation order is not fixed (results agree to rounding, like the fp64
// atomic strategy).
// This is the reference's stage-in / kernel / stage-out of parloop.hpp:253-313
// with the INC scatter turned into a row-owner gather: every output value is
// written exactly once and no global atomics or zero-fill are needed.
#pragma once
#include <cstdint>

#include "elements.cuh"

namespace loam_gpu {

struct PatchArgs {
  const int4* hdr;
  int npatches;
  const int32_t* win;
  const uint16_t* recs;
  const uint16_t* own;
  const int64_t* orp;   // Mats: CSR offset per owned row node
  const int32_t* oseg;  // Mats: value-segment offsets per patch (nown + 1 each)
  const double* coords;
  const double* coeff;
  FormParams prm;
  double* out;
  int accumulate;
  int max_win, max_cells, max_own, max_pairs, max_seg, bw;
  int64_t nverts; // coordinate rows (vertex nodes have ids < nverts)
};

// ---------------------------------------------------------------------------
// Whole element vector of an action form (b_i for every local row i).  The
// default evaluates the row functor for every i; P2 actions use the gradient
// of u_h instead of the 10 x 10 tensor (same integrals, ~6x fewer flops):
//   grad u_h = sum_m l_m w_m,  w_m = 4 u_m g_m - S + 4 sum_{edges (m,x) or (x,m)} u_e g_x,
//   S = sum_n u_n g_n;  t_k = q_diff W + (q_same - q_diff) w_k,  W = sum w_m,  T = sum t_k
//   vertex n: int grad phi_n . grad u_h = V g_n . (4 t_n - T)
//   edge (a,b):                        = 4 V (g_a . t_b + g_b . t_a)
// (int l_k l_m = V q(k,m), grad phi as in elements.cuh P2Row).  The mass part
// uses the exact P2 mass constants (p2_mass_const) with compile-time indices.
template <class F>
struct ElemVec {
  __device__ __forceinline__ static void all(const Geom<F::GD>& G, const double* C, const FormParams& prm,
                                             double* out) {
#pragma unroll
    for (int i = 0; i < F::NRN; ++i) F::row(i, G, C, prm, out + i);
  }
};

template <int FORM, int D>
struct ElemVec<FormT<FORM, D, 2>> {
  using F = FormT<FORM, D, 2>;
  static constexpr int NV = D + 1, NE = Simplex<D>::NE, N = NV + NE;
  __device__ __forceinline__ static void all(const Geom<D>& G, const double* C, const FormParams& prm,
                                             double* out) {
    double y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = 0.0;
    if constexpr (FORM != F_MASS_ACTION) {
      double S[D], w[NV][D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s = C[0] * G.g[0][a];
#pragma unroll
        for (int n = 1; n < NV; ++n) s = fma(C[n], G.g[n][a], s);
        S[a] = s;
      }
#pragma unroll
      for (int m = 0; m < NV; ++m)
#pragma unroll
        for (int a = 0; a < D; ++a) w[m][a] = fma(4.0 * C[m], G.g[m][a], -S[a]);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int ea = Simplex<D>::edge_a(e), eb = Simplex<D>::edge_b(e);
        const double ue = 4.0 * C[NV + e];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          w[eb][a] = fma(ue, G.g[ea][a], w[eb][a]);
          w[ea][a] = fma(ue, G.g[eb][a], w[ea][a]);
        }
      }
      constexpr double qs = Simplex<D>::q_same, qd = Simplex<D>::q_diff;
      double Wv[D], t[NV][D], T[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s = w[0][a];
#pragma unroll
        for (int m = 1; m < NV; ++m) s += w[m][a];
        Wv[a] = s;
      }
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int a = 0; a < D; ++a) t[k][a] = fma(qs - qd, w[k][a], qd * Wv[a]);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s = t[0][a];
#pragma unroll
        for (int k = 1; k < NV; ++k) s += t[k][a];
        T[a] = s;
      }
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) s = fma(G.g[n][a], fma(4.0, t[n][a], -T[a]), s);
        y[n] = s;
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int ea = Simplex<D>::edge_a(e), eb = Simplex<D>::edge_b(e);
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) s = fma(G.g[ea][a], t[eb][a], fma(G.g[eb][a], t[ea][a], s));
        y[NV + e] = 4.0 * s;
      }
    }
    if constexpr (FORM != F_STIFFNESS_ACTION) {
      // P2 mass action by index-coincidence classes (p2_mass_kind):
      //   vertex n: m0 u_n + m1 (Uv - u_n) + m2 sum_{e ni n} u_e + m3 (Ue - sum_{e ni n} u_e)
      //   edge e=(a,b): m2 (u_a + u_b) + m3 (Uv - u_a - u_b) + m4 u_e
      //                 + m5 sum_{f shares one vertex} u_f + m6 sum_{f disjoint} u_f
      constexpr double m0 = p2_mass_const<D>(0), m1 = p2_mass_const<D>(1), m2 = p2_mass_const<D>(2),
                       m3 = p2_mass_const<D>(3), m4 = p2_mass_const<D>(4), m5 = p2_mass_const<D>(5),
                       m6 = p2_mass_const<D>(6);
      const double kap = FORM == F_MASS_ACTION ? 1.0 : prm.p[0];
      double Uv = C[0], Ue = C[NV];
#pragma unroll
      for (int n = 1; n < NV; ++n) Uv += C[n];
#pragma unroll
      for (int e = 1; e < NE; ++e) Ue += C[NV + e];
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        double ein = 0.0;
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (Simplex<D>::edge_a(e) == n || Simplex<D>::edge_b(e) == n) ein += C[NV + e];
        const double m = fma(m0 - m1, C[n], fma(m1, Uv, fma(m2 - m3, ein, m3 * Ue)));
        y[n] = fma(kap, m, y[n]);
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int a = Simplex<D>::edge_a(e), b = Simplex<D>::edge_b(e);
        double dis = 0.0;
#pragma unroll
        for (int f = 0; f < NE; ++f) {
          const int c = Simplex<D>::edge_a(f), d = Simplex<D>::edge_b(f);
          if (f != e && c != a && c != b && d != a && d != b) dis += C[NV + f];
        }
        const double uab = C[a] + C[b];
        const double share = Ue - C[NV + e] - dis;
        double m = fma(m2 - m3, uab, m3 * Uv);
        m = fma(m4, C[NV + e], m);
        m = fma(m5, share, m);
        if (m6 != 0.0) m = fma(m6, dis, m);
        y[NV + e] = fma(kap, m, y[NV + e]);
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = G.V * y[i];
  }
};

// In-place exclusive scan of a[0..n) by one warp; returns the total.
__device__ __forceinline__ int warp_exclusive_scan(int* a, int n) {
  const int lane = threadIdx.x & 31;
  const int per = (n + 31) / 32, b = lane * per, e = min(n, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  int x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const int total = __shfl_sync(0xffffffffu, x, 31);
  int run = x - s;
  for (int i = b; i < e; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  return total;
}

template <class F>
__device__ __forceinline__ void patch_vertices(const PatchArgs& a, const int32_t* win_s, const uint16_t* rec,
                                               double (&X)[F::GD + 1][F::GD]) {
  constexpr int GD = F::GD;
#pragma unroll
  for (int v = 0; v <= GD; ++v) {
    const int64_t vid = win_s[rec[v]];
    if constexpr (GD == 2) {
      const double2 c = __ldg(reinterpret_cast<const double2*>(a.coords) + vid);
      X[v][0] = c.x;
      X[v][1] = c.y;
    } else {
#pragma unroll
      for (int c = 0; c < GD; ++c) X[v][c] = __ldg(a.coords + vid * GD + c);
    }
  }
}

// ---------------------------------------------------------------------------
// Shared-memory carve-up (byte offsets), identical on host and device.
struct PatchSmem {
  int seg, geo, rp0, segoff, plist, plist2, rcnt, tcnt, bm, pre, win, recs, rowof, oslot, ctr, total;
};
__host__ __device__ inline PatchSmem patch_smem(int gs, int nrn, bool mat, int max_win, int max_cells, int max_own,
                                                int max_pairs, int max_seg, int bw) {
  auto up = [](int x) { return (x + 15) & ~15; };
  PatchSmem L{};
  int o = 0;
  L.seg = o;    o += up(mat ? max_seg * 8 : max_own * 8); // Dats: per-row accumulators
  L.geo = o;    o += up(mat ? max_cells * gs * 8 : max_cells * nrn * 8); // Dats: element vectors
  L.rp0 = o;    o += up(mat ? max_own * 8 : 0);
  L.segoff = o; o += up(mat ? (max_own + 1) * 4 : 0);
  L.plist = o;  o += up(mat ? max_pairs * 4 : 0);
  L.plist2 = o; o += up(mat ? max_pairs * 4 : 0);
  L.rcnt = o;   o += up(mat ? max_own * 4 : 0);
  L.tcnt = o;   o += up(mat ? 3 * 65 * 4 : 0);
  L.bm = o;     o += up(mat ? max_own * bw * 4 : 0);
  L.pre = o;    o += up(mat ? max_own * bw : 0);
  L.win = o;    o += up((max_win + 4) * 4);
  L.recs = o;   o += up((max_cells * nrn + 8) * 2);
  L.rowof = o;  o += up(max_win * 2);
  L.oslot = o;  o += up(max_own * 2);
  L.ctr = o;    o += 16;
  L.total = o;
  return L;
}

template <class F>
struct PatchTraits {
  static constexpr int GD = F::GD;
  static constexpr int GS = GD * GD + 1; // Mats keep g_1..g_d and V per tile cell
};

__device__ __forceinline__ void smem_add(double* p, double v) { atomicAdd(p, v); }

// Stage-in shared by both kernels: window ids, tile-cell slots, owned rows.
// Ends with __syncthreads.
template <int NRN, int NT>
__device__ __forceinline__ void patch_stage(const PatchArgs& a, int p, const PatchSmem& L, unsigned char* sm,
                                           int4& h0, int4& h1) {
  const int tid = threadIdx.x;
  h0 = __ldg(a.hdr + 2 * p);
  h1 = __ldg(a.hdr + 2 * p + 1);
  const int nwin = h0.y, ncell = h0.w, nown = h1.y;
  int16_t* rowof = reinterpret_cast<int16_t*>(sm + L.rowof);
  {
    const int4* src = reinterpret_cast<const int4*>(a.win + h0.x);
    int4* dst = reinterpret_cast<int4*>(sm + L.win);
    for (int t = tid; t < (nwin + 3) >> 2; t += NT) dst[t] = __ldg(src + t);
  }
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.recs + h0.z);
    uint4* dst = reinterpret_cast<uint4*>(sm + L.recs);
    for (int t = tid; t < (ncell * NRN + 7) >> 3; t += NT) dst[t] = __ldg(src + t);
  }
  for (int t = tid; t < nwin; t += NT) rowof[t] = -1;
  __syncthreads();
  uint16_t* oslot = reinterpret_cast<uint16_t*>(sm + L.oslot);
  for (int k = tid; k < nown; k += NT) {
    const uint16_t sl = __ldg(a.own + h1.x + k);
    rowof[sl] = (int16_t)k;
    oslot[k] = sl;
  }
}

// Cell-owned patches for Dats (patch.cuh, halo = false): every cell is
// computed exactly once.  Each cell writes its element-vector entries into
// the patch's node-sorted incidence array (position = the node's incidence
// offset from the plan + an integer shared-memory counter: native ATOMS.ADD,
// no fp64 CAS), then one thread per window node sums its incidences and
// writes the node once -- or RED-adds it when the node is shared with another
// patch (bit 31 of its window id).
__host__ __device__ inline int patch_vec_smem(int max_win, int max_cells, int nrn, int gd, int* off_win, int* off_rec,
                                              int* off_ptr, int* off_fill, int* off_x) {
  auto up = [](int x) { return (x + 15) & ~15; };
  int o = up(max_cells * nrn * 8);
  *off_x = o; // per window node: coordinates (vertex nodes) and coefficient
  o += up(max_win * (gd + 1) * 8);
  *off_win = o;
  o += up((max_win + 4) * 4);
  *off_rec = o;
  o += up((max_cells * nrn + 8) * 2);
  *off_ptr = o;
  o += up((max_win + 16) * 2);
  *off_fill = o;
  o += up(max_win * 4);
  return o;
}

template <class F, int NT>
__global__ void __launch_bounds__(NT, 3) k_patch_vec(const __grid_constant__ PatchArgs a) {
  constexpr int NRN = F::NRN, GD = F::GD, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char sm[];
  int off_win, off_rec, off_ptr, off_fill, off_x;
  patch_vec_smem(a.max_win, a.max_cells, NRN, GD, &off_win, &off_rec, &off_ptr, &off_fill, &off_x);
  double* xs = reinterpret_cast<double*>(sm + off_x); // [nwin][GD + 1]: x_0..x_{GD-1}, coefficient
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* sev = reinterpret_cast<double*>(sm);
  int32_t* win_s = reinterpret_cast<int32_t*>(sm + off_win);
  uint16_t* rec_s = reinterpret_cast<uint16_t*>(sm + off_rec);
  uint16_t* ptr_s = reinterpret_cast<uint16_t*>(sm + off_ptr);
  int* fill = reinterpret_cast<int*>(sm + off_fill);
  for (int p = blockIdx.x; p < a.npatches; p += gridDim.x) {
    const int4 h0 = __ldg(a.hdr + 2 * p), h1 = __ldg(a.hdr + 2 * p + 1);
    const int nwin = h0.y, ncell = h0.w;
    {
      const int4* src = reinterpret_cast<const int4*>(a.win + h0.x);
      for (int t = tid; t < (nwin + 3) >> 2; t += NT) reinterpret_cast<int4*>(win_s)[t] = __ldg(src + t);
      const uint4* rsrc = reinterpret_cast<const uint4*>(a.recs + h0.z);
      for (int t = tid; t < (ncell * NRN + 7) >> 3; t += NT) reinterpret_cast<uint4*>(rec_s)[t] = __ldg(rsrc + t);
      const uint4* psrc = reinterpret_cast<const uint4*>(a.own + h1.x);
      for (int t = tid; t < (nwin + 8) >> 3; t += NT) reinterpret_cast<uint4*>(ptr_s)[t] = __ldg(psrc + t);
      for (int t = tid; t < nwin; t += NT) fill[t] = 0;
      // window-node gathers once per patch (a node is shared by ~7 of the
      // patch's cells): coefficient of every node, coordinates of vertex nodes
      for (int t = tid; t < nwin; t += NT) {
        const int64_t id = __ldg(a.win + h0.x + t) & 0x7fffffff;
        xs[t * (GD + 1) + GD] = __ldg(a.coeff + id);
        if (id < a.nverts) {
#pragma unroll
          for (int d = 0; d < GD; ++d) xs[t * (GD + 1) + d] = __ldg(a.coords + id * GD + d);
        }
      }
    }
    __syncthreads();
    for (int base = 0; base < ncell; base += NT) {
      const int c = base + tid; // consecutive cells: conflict-free slot reads (stride nrn u16)
      if (c < ncell) {
        const uint16_t* rec = rec_s + c * NRN;
        double X[GD + 1][GD];
#pragma unroll
        for (int v = 0; v <= GD; ++v)
#pragma unroll
          for (int d = 0; d < GD; ++d) X[v][d] = xs[rec[v] * (GD + 1) + d];
        Geom<GD> G;
        geometry<GD>(X, G);
        double C[F::NCOEFF];
#pragma unroll
        for (int q = 0; q < F::NCOEFF; ++q) C[q] = xs[rec[q] * (GD + 1) + GD];
        double y[NRN];
        ElemVec<F>::all(G, C, a.prm, y);
#pragma unroll
        for (int i = 0; i < NRN; ++i) {
          const int s = rec[i];
          sev[ptr_s[s] + atomicAdd(fill + s, 1)] = y[i];
        }
      }
    }
    __syncthreads();
    for (int t = tid; t < nwin; t += NT) {
      double sum = 0.0;
      for (int q = ptr_s[t], e = ptr_s[t + 1]; q < e; ++q) sum += sev[q];
      const int x = win_s[t];
      double* o = a.out + (x & 0x7fffffff);
      if (x < 0) atomicAdd(o, sum); // shared node: other patches add too
      else *o = a.accumulate ? *o + sum : sum;
    }
    __syncthreads();
  }
}

template <class F, int NT>
__global__ void __launch_bounds__(NT) k_patch_mat(const __grid_constant__ PatchArgs a) {
  constexpr int NRN = F::NRN, NCN = F::NCN, GD = F::GD, RD = F::RD, CD = F::CD, GS = PatchTraits<F>::GS;
  static_assert(NRN == NCN, "patch kernels serve square (row map == column map) forms");
  static_assert(NRN <= 16, "pair codes keep the local row in 4 bits");
  extern __shared__ __align__(16) unsigned char sm[];
  const PatchSmem L = patch_smem(GS, NRN, true, a.max_win, a.max_cells, a.max_own, a.max_pairs, a.max_seg, a.bw);
  const int tid = threadIdx.x;
  double* seg = reinterpret_cast<double*>(sm + L.seg);
  double* geo = reinterpret_cast<double*>(sm + L.geo);
  int64_t* rp0 = reinterpret_cast<int64_t*>(sm + L.rp0);
  int* segoff = reinterpret_cast<int*>(sm + L.segoff);
  int* plist = reinterpret_cast<int*>(sm + L.plist);
  int* plist2 = reinterpret_cast<int*>(sm + L.plist2);
  int* rcnt = reinterpret_cast<int*>(sm + L.rcnt);
  int* tcnt = reinterpret_cast<int*>(sm + L.tcnt); // [0,64) counts, [65,130) offsets, [130,194) fill
  uint32_t* bm = reinterpret_cast<uint32_t*>(sm + L.bm);
  uint8_t* pre = reinterpret_cast<uint8_t*>(sm + L.pre);
  const int32_t* win_s = reinterpret_cast<const int32_t*>(sm + L.win);
  const uint16_t* rec_s = reinterpret_cast<const uint16_t*>(sm + L.recs);
  const int16_t* rowof = reinterpret_cast<const int16_t*>(sm + L.rowof);
  int* ctr = reinterpret_cast<int*>(sm + L.ctr);
  const int bw = a.bw;
  for (int p = blockIdx.x; p < a.npatches; p += gridDim.x) {
    int4 h0, h1;
    patch_stage<NRN, NT>(a, p, L, sm, h0, h1);
    const int nwin = h0.y, ncell = h0.w, nown = h1.y, words = (nwin + 31) >> 5;
    for (int k = tid; k <= nown; k += NT) {
      segoff[k] = __ldg(a.oseg + h1.x + p + k);
      if (k < nown) {
        rp0[k] = __ldg(a.orp + h1.x + k);
        rcnt[k] = 0;
      }
    }
    for (int k = tid; k < nown; k += NT)
      for (int w = 0; w < words; ++w) bm[k * bw + w] = 0u;
    for (int t = tid; t < 3 * 65; t += NT) tcnt[t] = 0;
    if (tid == 0) ctr[0] = 0;
    __syncthreads();
    // per tile cell: geometry once; owned pairs: column bits, within-row
    // index t, pair list
    for (int c = tid; c < ncell; c += NT) {
      const uint16_t* rec = rec_s + c * NRN;
      double X[GD + 1][GD];
      patch_vertices<F>(a, win_s, rec, X);
      Geom<GD> G;
      geometry<GD>(X, G);
      double* o = geo + c * GS;
#pragma unroll
      for (int v = 1; v <= GD; ++v)
#pragma unroll
        for (int d = 0; d < GD; ++d) o[(v - 1) * GD + d] = G.g[v][d];
      o[GD * GD] = G.V;
      int sl[NCN];
#pragma unroll
      for (int j = 0; j < NCN; ++j) sl[j] = rec[j];
#pragma unroll
      for (int i = 0; i < NRN; ++i) {
        const int k = rowof[sl[i]];
        if (k >= 0) {
#pragma unroll
          for (int j = 0; j < NCN; ++j) atomicOr(bm + k * bw + (sl[j] >> 5), 1u << (sl[j] & 31));
          const int t = min(atomicAdd(rcnt + k, 1), 63);
          atomicAdd(tcnt + t, 1);
          plist[atomicAdd(ctr, 1)] = (c << 10) | (i << 6) | t;
        }
      }
    }
    // value segment: zero, or the Mat's current values (INC accumulates)
    const int tot = segoff[nown];
    if (a.accumulate) {
      for (int t = tid; t < tot; t += NT) {
        int lo = 0, hi = nown; // row of value t: segoff[lo] <= t < segoff[lo + 1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (segoff[mid] <= t) lo = mid;
          else hi = mid;
        }
        seg[t] = a.out[rp0[lo] + t - segoff[lo]];
      }
    } else {
      for (int t = tid; t < tot; t += NT) seg[t] = 0.0;
    }
    __syncthreads();
    if (tid < 32) { // offsets of the within-row-index groups
      int* toff = tcnt + 65;
      toff[tid] = tcnt[tid];
      toff[tid + 32] = tcnt[tid + 32];
      __syncwarp();
      const int total = warp_exclusive_scan(toff, 64);
      if (tid == 0) toff[64] = total;
    }
    for (int k = tid; k < nown; k += NT) {
      int run = 0;
      for (int w = 0; w < words; ++w) {
        pre[k * bw + w] = (uint8_t)run;
        run += __popc(bm[k * bw + w]);
      }
    }
    __syncthreads();
    const int npairs = ctr[0];
    // order the pairs by their within-row index t: inside one t group every
    // row appears at most once, so lanes adding concurrently hit distinct rows
    for (int q = tid; q < npairs; q += NT) {
      const int code = plist[q], t = code & 63;
      plist2[tcnt[65 + t] + atomicAdd(tcnt + 130 + t, 1)] = code;
    }
    __syncthreads();
    for (int q = tid; q < npairs; q += NT) {
      const int code = plist2[q], c = code >> 10, i = (code >> 6) & 15;
      const uint16_t* rec = rec_s + c * NRN;
      const int k = rowof[rec[i]];
      const uint32_t* B = bm + k * bw;
      const uint8_t* P = pre + k * bw;
      int rk[NCN];
#pragma unroll
      for (int j = 0; j < NCN; ++j) {
        const int s = rec[j];
        rk[j] = P[s >> 5] + __popc(B[s >> 5] & ((1u << (s & 31)) - 1u));
      }
      Geom<GD> G;
      const double* gc = geo + c * GS;
#pragma unroll
      for (int v = 1; v <= GD; ++v)
#pragma unroll
        for (int d = 0; d < GD; ++d) G.g[v][d] = gc[(v - 1) * GD + d];
#pragma unroll
      for (int d = 0; d < GD; ++d) {
        double s = G.g[1][d];
#pragma unroll
        for (int v = 2; v <= GD; ++v) s += G.g[v][d];
        G.g[0][d] = -s;
      }
      G.V = gc[GD * GD];
      const int Lk = (segoff[k + 1] - segoff[k]) / (RD * CD);
      double* sg = seg + segoff[k];
#pragma unroll
      for (int d = 0; d < RD; ++d) {
        double blk[F::NC];
        form_subrow<F>(i, d, G, nullptr, a.prm, blk);
        double* sr = sg + d * Lk * CD;
#pragma unroll
        for (int j = 0; j < NCN; ++j)
#pragma unroll
          for (int cc = 0; cc < CD; ++cc)
            if (!diag_block<F>::value || d == cc) smem_add(sr + rk[j] * CD + cc, blk[j * CD + cc]);
      }
    }
    __syncthreads();
    for (int t = tid; t < tot; t += NT) {
      int lo = 0, hi = nown;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (segoff[mid] <= t) lo = mid;
        else hi = mid;
      }
      a.out[rp0[lo] + t - segoff[lo]] = seg[t];
    }
    __syncthreads();
  }
}

} // namespace loam_gpu
