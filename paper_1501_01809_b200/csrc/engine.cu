#include <climits>
#include <chrono>
// engine.cu -- the B200 par_loop engine: registry, validate, execute.
//
// Replaces loam::execute (parloop.hpp:191-384).  Two device paths:
//
//  * OWNER-COMPUTES (default for catalogue forms with the assemble_* argument
//    pattern, assemble.hpp:91-99,123-129): one thread owns one row node and
//    gathers every (cell, local index) pair incident to it (plan.cuh), computes
//    its element rows in registers and writes each output entry exactly once
//    -- no atomics, no zero-fill pass, deterministic sums.  Mats accumulate a
//    warp's contiguous CSR segment in shared memory and store it coalesced.
//  * CELL-MAJOR generic staging engine for any registered kernel and any
//    access mix (the reference's stage-in / kernel / stage-out, parloop.hpp:
//    253-320): indirect INC through fp64 atomics, or -- when a loop writes
//    indirectly with WRITE/RW, or the colouring strategy is selected -- one
//    launch per colour of the bit-exact greedy colouring with plain stores.
//    Global reductions go through per-entity slots and a fixed-shape tree.
//
// There is no CPU fallback: an unregistered kernel is an error.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <unordered_map>

#include "async.cuh"
#include "stage.cuh"
#include "elements.cuh"
#include "engine.cuh"
#include "ctile.cuh"
#include "etile.cuh"
#include "ltile.cuh"
#include "thtile.cuh"
#include "wtile.cuh"
#include "ntile.cuh"
#include "rtile.cuh"
#include "patch.cuh"
#include "patch_kernels.cuh"
#include "plan.cuh"
#include "test_kernels.cuh"

namespace loam_gpu {

std::atomic<int64_t> g_launches{0};

Options& options() {
  static Options o;
  return o;
}

namespace {

constexpr int kMaxArgs = 8;
constexpr int kTPB = 256;

// ===========================================================================
// Generic cell-major staging engine
// ===========================================================================

struct GArg {
  int kind, access, dim;
  double* data;
  const int32_t* map;
  int arity;
  const int32_t* map2;
  int arity2;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  int nrows;
  int off, size;   // staging slot
  int slot_off;    // Global reduction slot offset within an entity's slots
};

struct GLaunch {
  int nargs;
  GArg a[kMaxArgs];
  const int32_t* order; // entity list (nullptr: identity)
  int count;
  int plain;            // entities of one launch are conflict-free: plain RMW
  int slot_stride;
  double* slots;        // [n * slot_stride] Global contributions
  FormParams prm;
  unsigned long long* err;
};

__device__ __forceinline__ double red_identity(int access) {
  return access == LOAM_SUM ? 0.0 : (access == LOAM_MIN ? __longlong_as_double(0x7ff0000000000000ll)
                                                        : __longlong_as_double(0xfff0000000000000ll));
}

__device__ __forceinline__ int64_t csr_find(const int64_t* rp, const int32_t* ci, int nrows, int row,
                                            int col) {
  if (row < 0 || row >= nrows) return -1;
  int64_t lo = rp[row], hi = rp[row + 1];
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ci[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return (lo == end || ci[lo] != col) ? -1 : lo;
}

template <class K>
__global__ void k_generic(const __grid_constant__ GLaunch L) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L.count) return;
  const int e = L.order ? L.order[t] : t;
  double stage[K::STAGE];
  double* ptrs[kMaxArgs];
  // ---- stage in (parloop.hpp:254-283)
  for (int k = 0; k < L.nargs; ++k) {
    const GArg& a = L.a[k];
    double* st = stage + a.off;
    ptrs[k] = st;
    if (a.kind == LOAM_ARG_DAT) {
      if (a.access == LOAM_WRITE || a.access == LOAM_INC) {
        for (int x = 0; x < a.size; ++x) st[x] = 0.0;
      } else if (!a.map) {
        for (int d = 0; d < a.dim; ++d) st[d] = a.data[(int64_t)e * a.dim + d];
      } else {
        for (int q = 0; q < a.arity; ++q) {
          const int64_t base = (int64_t)a.map[(int64_t)e * a.arity + q] * a.dim;
          for (int d = 0; d < a.dim; ++d) st[q * a.dim + d] = a.data[base + d];
        }
      }
    } else if (a.kind == LOAM_ARG_MAT) {
      for (int x = 0; x < a.size; ++x) st[x] = 0.0;
    } else {
      if (a.access == LOAM_READ)
        for (int d = 0; d < a.dim; ++d) st[d] = a.data[d];
      else
        for (int d = 0; d < a.dim; ++d) st[d] = red_identity(a.access);
    }
  }
  K::run(ptrs, L.prm);
  // ---- stage out (parloop.hpp:287-319)
  for (int k = 0; k < L.nargs; ++k) {
    const GArg& a = L.a[k];
    const double* st = stage + a.off;
    if (a.kind == LOAM_ARG_DAT) {
      if (a.access == LOAM_READ) continue;
      if (!a.map) {
        double* dst = a.data + (int64_t)e * a.dim;
        for (int d = 0; d < a.dim; ++d) dst[d] = a.access == LOAM_INC ? dst[d] + st[d] : st[d];
      } else {
        for (int q = 0; q < a.arity; ++q) {
          double* dst = a.data + (int64_t)a.map[(int64_t)e * a.arity + q] * a.dim;
          for (int d = 0; d < a.dim; ++d) {
            const double v = st[q * a.dim + d];
            if (a.access != LOAM_INC) dst[d] = v; // WRITE/RW: coloured launches only
            else if (L.plain) dst[d] += v;
            else atomicAdd(dst + d, v);
          }
        }
      }
    } else if (a.kind == LOAM_ARG_MAT) {
      // Mat::addto (data.hpp:205-222)
      for (int i = 0; i < a.arity; ++i) {
        const int row = a.map[(int64_t)e * a.arity + i];
        for (int j = 0; j < a.arity2; ++j) {
          const int col = a.map2[(int64_t)e * a.arity2 + j];
          const int64_t pos = csr_find(a.row_ptr, a.col_idx, a.nrows, row, col);
          if (pos < 0) {
            atomicCAS(L.err, 0ull, (1ull << 63) | ((unsigned long long)(uint32_t)row << 32) | (uint32_t)col);
            continue;
          }
          const double v = st[i * a.arity2 + j];
          if (a.access == LOAM_WRITE) a.data[pos] = v;
          else if (L.plain) a.data[pos] += v;
          else atomicAdd(a.data + pos, v);
        }
      }
    } else if (a.access != LOAM_READ) {
      double* slot = L.slots + (int64_t)e * L.slot_stride + a.slot_off;
      for (int d = 0; d < a.dim; ++d) slot[d] = st[d];
    }
  }
}

// Fixed-shape tree reduction of Global slots over entities 0..n-1 into dst.
__global__ void k_global_reduce(const double* __restrict__ slots, int n, int stride, int off,
                                int access, double* dst) {
  __shared__ double sh[kTPB];
  const int d = blockIdx.x;
  double acc = red_identity(access);
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const double v = slots[(int64_t)e * stride + off + d];
    acc = access == LOAM_SUM ? acc + v : (access == LOAM_MIN ? fmin(acc, v) : fmax(acc, v));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double a = sh[threadIdx.x], b = sh[threadIdx.x + w];
      sh[threadIdx.x] = access == LOAM_SUM ? a + b : (access == LOAM_MIN ? fmin(a, b) : fmax(a, b));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) dst[d] = sh[0];
}

__global__ void k_fill_identity(double* dst, int dim, int access) {
  if (threadIdx.x < dim) dst[threadIdx.x] = red_identity(access);
}

// Catalogue form as a staged kernel: A = element tensor(X, C)  (form.hpp:201-320).
template <class F>
struct FormKernel {
  static constexpr int STAGE = F::NR * F::NC + (F::GD + 1) * F::GD + (F::HAS_COEFF ? F::NCOEFF : 0);
  __device__ static void run(double* const* p, const FormParams& prm) {
    double X[F::GD + 1][F::GD];
#pragma unroll
    for (int v = 0; v <= F::GD; ++v)
#pragma unroll
      for (int d = 0; d < F::GD; ++d) X[v][d] = p[1][v * F::GD + d];
    Geom<F::GD> G;
    geometry<F::GD>(X, G);
    element_tensor<F>(G, F::HAS_COEFF ? p[2] : nullptr, prm, p[0]);
  }
};

// ===========================================================================
// Owner-computes kernels
// ===========================================================================

struct OwnerArgs {
  const int32_t* ptr;
  const int32_t* pairs;
  const uint8_t* ranks;
  const int32_t* xmap;
  int xstride;
  const double* coords;
  const int32_t* cmap;
  int cstride;
  const double* coeff;
  FormParams prm;
  double* out;
  const int64_t* row_ptr;
  const int32_t* chunk_row;
  int nchunks, seg_max, nrows_node, accumulate;
};

// Batched gather: the loads of U pairs are issued before any use so U
// independent pair -> cell-map -> coordinate chains are in flight per lane
// (the single-pair loop was latency bound: long-scoreboard stalls ~80%).
template <class F, int U>
struct PairBatch {
  static constexpr int GD = F::GD;
  int code[U];
  bool valid[U];
  double X[U][GD + 1][GD];
  double C[U][F::HAS_COEFF ? F::NCOEFF : 1];

  __device__ __forceinline__ void load(const OwnerArgs& a, int p, int p1) {
    int vid[U][GD + 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      valid[u] = p + u < p1;
      code[u] = __ldg(a.pairs + (valid[u] ? p + u : p));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = code[u] / F::NRN;
      const int32_t* xr = a.xmap + (int64_t)s * a.xstride;
#pragma unroll
      for (int v = 0; v <= GD; ++v) vid[u][v] = __ldg(xr + v);
    }
    if constexpr (F::HAS_COEFF) {
      int cid[U][F::NCOEFF];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t* cr = a.cmap + (int64_t)(code[u] / F::NRN) * a.cstride;
#pragma unroll
        for (int q = 0; q < F::NCOEFF; ++q) cid[u][q] = __ldg(cr + q);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < F::NCOEFF; ++q) C[u][q] = __ldg(a.coeff + cid[u][q]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v <= GD; ++v) {
        if constexpr (GD == 2) {
          const double2 c = __ldg(reinterpret_cast<const double2*>(a.coords) + vid[u][v]);
          X[u][v][0] = c.x;
          X[u][v][1] = c.y;
        } else {
#pragma unroll
          for (int d = 0; d < GD; ++d) X[u][v][d] = __ldg(a.coords + (int64_t)vid[u][v] * GD + d);
        }
      }
  }
};

// In-row ranks of the NCN column nodes of pair p, with the widest aligned loads.
template <int NCN>
__device__ __forceinline__ void load_ranks(const uint8_t* ranks, int64_t p, int (&rk)[NCN]) {
  const uint8_t* b = ranks + p * NCN;
  if constexpr (NCN % 4 == 0) {
#pragma unroll
    for (int w = 0; w < NCN / 4; ++w) {
      const uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(b) + w);
#pragma unroll
      for (int k = 0; k < 4; ++k) rk[4 * w + k] = (x >> (8 * k)) & 0xff;
    }
  } else if constexpr (NCN % 2 == 0) {
#pragma unroll
    for (int w = 0; w < NCN / 2; ++w) {
      const uint32_t x = __ldg(reinterpret_cast<const uint16_t*>(b) + w);
      rk[2 * w] = x & 0xff;
      rk[2 * w + 1] = x >> 8;
    }
  } else {
#pragma unroll
    for (int k = 0; k < NCN; ++k) rk[k] = __ldg(b + k);
  }
}

template <class F>
constexpr int batch_of() {
  return F::GD == 2 ? 4 : 2;
}

// Residual (Dat INC, dim 1): out[r] (+)= sum over pairs of row i of the action.
template <class F>
__global__ void __launch_bounds__(kTPB) k_owner_vec(const __grid_constant__ OwnerArgs a) {
  constexpr int U = batch_of<F>();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows_node) return;
  double acc = 0.0;
  const int p1 = __ldg(a.ptr + r + 1);
  for (int p = __ldg(a.ptr + r); p < p1; p += U) {
    PairBatch<F, U> B;
    B.load(a, p, p1);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!B.valid[u]) continue;
      const int i = B.code[u] % F::NRN;
      Geom<F::GD> G;
      geometry<F::GD>(B.X[u], G);
      double v;
      F::row(i, G, B.C[u], a.prm, &v);
      acc += v;
    }
  }
  a.out[r] = a.accumulate ? a.out[r] + acc : acc;
}

// Cell-centric scatter (the fp64-atomic strategies for catalogue forms): one
// thread per cell in locality order (sorted maps: coalesced map rows), the
// element tensor in registers with compile-time rows -- each cell's geometry
// is computed once, not once per row as the owner kernels must -- and one
// fp64 RED per entry (parloop.hpp:302-313 INC scatter / Mat::addto).  Matrix
// entries go to the precomputed per-cell slot: row_ptr[dof row] + in-row rank
// (the pair plan's ranks scattered to cell-major order, plan.cu:build_ranks),
// so no CSR search happens at assembly time.  AGG: lanes of a warp that hit
// the same address first combine through __match_any_sync + shuffles and the
// group leader issues one RED (the north star's warp-aggregated reduction).
struct CellArgs {
  int n;
  const int32_t* rmap; // sorted row map, NRN per cell
  const int32_t* xmap; // sorted coordinate map rows
  int xstride;
  const int32_t* cmap; // sorted coefficient map rows
  int cstride;
  const double* coords;
  const double* coeff;
  const uint8_t* cranks;  // (matrices) [n x NRN x NCN] in-row rank per entry
  const int64_t* row_ptr; // (matrices) CSR dof-row offsets
  FormParams prm;
  double* out;
  double* contrib; // deterministic mode: [n x NRN] element-vector entries, summed per row afterwards
};

template <bool AGG>
__device__ __forceinline__ void red_add(double* base, int64_t pos, double v, bool valid) {
  if constexpr (!AGG) {
    if (valid) atomicAdd(base + pos, v);
  } else {
    const int lane = threadIdx.x & 31;
    const int64_t key = valid ? pos : -1 - (int64_t)lane; // invalid lanes: unique keys
    const unsigned peers = __match_any_sync(0xffffffffu, (unsigned long long)key);
    const int leader = __ffs(peers) - 1;
    unsigned m = lane == leader ? peers & (peers - 1) : 0u; // the leader collects its peers
    double sum = v;
    while (__any_sync(0xffffffffu, m != 0)) {
      const int src = m ? __ffs(m) - 1 : lane;
      const double x = __shfl_sync(0xffffffffu, v, src);
      if (m) {
        sum += x;
        m &= m - 1;
      }
    }
    if (valid && lane == leader) atomicAdd(base + pos, sum);
  }
}

template <class F>
__device__ __forceinline__ void cell_gather(const CellArgs& a, int e, double (&X)[F::GD + 1][F::GD],
                                            double (&C)[F::HAS_COEFF ? F::NCOEFF : 1], int (&rows)[F::NRN]) {
  constexpr int GD = F::GD, NV = GD + 1;
  int vid[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) vid[v] = __ldg(a.xmap + (int64_t)e * a.xstride + v);
#pragma unroll
  for (int i = 0; i < F::NRN; ++i) rows[i] = __ldg(a.rmap + (int64_t)e * F::NRN + i);
  if constexpr (F::HAS_COEFF)
#pragma unroll
    for (int q = 0; q < F::NCOEFF; ++q) C[q] = __ldg(a.coeff + __ldg(a.cmap + (int64_t)e * a.cstride + q));
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int c = 0; c < GD; ++c) X[v][c] = __ldg(a.coords + (int64_t)vid[v] * GD + c);
}

#ifndef LOAM_GPU_CELL_MINB
#define LOAM_GPU_CELL_MINB 1
#endif
// The same with the warp's 32 map rows staged through shared memory by
// coalesced 16-byte loads: used when the row, coefficient and coordinate maps
// are one sorted map whose first gdim+1 entries are the vertices (P2 actions,
// config 3).  One thread's 10-entry row is 40 scattered bytes per lane
// otherwise -- 10 load instructions touching ~40 sectors each per warp.
// (build option: a register cap through min blocks per SM; the default leaves the
// allocation to ptxas -- 96 registers, 5 CTAs / SM.  A bound of 1 makes it take 122.)
#ifdef LOAM_GPU_CELLROWS_MINB
#define LOAM_GPU_CELLROWS_BOUNDS __launch_bounds__(128, LOAM_GPU_CELLROWS_MINB)
#else
#define LOAM_GPU_CELLROWS_BOUNDS __launch_bounds__(128)
#endif
template <class F>
__global__ void LOAM_GPU_CELLROWS_BOUNDS k_cell_vec_rows(const __grid_constant__ CellArgs a) {
  constexpr int NRN = F::NRN, GD = F::GD, NV = GD + 1;
  static_assert((32 * NRN) % 4 == 0, "row block of a warp must be a whole number of int4");
  __shared__ __align__(16) int32_t rows_s[4][32 * NRN];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * 4 + wl) * 32;
  if (c0 >= a.n) return;
  const int ncell = a.n - c0 < 32 ? (int)(a.n - c0) : 32;
  const int nint = ncell * NRN;
  const int32_t* src = a.rmap + c0 * NRN;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    for (int q = lane; q < nint / 4; q += 32)
      reinterpret_cast<int4*>(rows_s[wl])[q] = __ldg(reinterpret_cast<const int4*>(src) + q);
    for (int q = (nint / 4) * 4 + lane; q < nint; q += 32) rows_s[wl][q] = __ldg(src + q);
  } else {
    for (int q = lane; q < nint; q += 32) rows_s[wl][q] = __ldg(src + q);
  }
  __syncwarp();
  if (lane >= ncell) return;
  const int32_t* row = rows_s[wl] + lane * NRN;
  int nodes[NRN];
#pragma unroll
  for (int i = 0; i < NRN; ++i) nodes[i] = row[i];
  double X[NV][GD], C[F::NCOEFF];
#pragma unroll
  for (int q = 0; q < F::NCOEFF; ++q) C[q] = __ldg(a.coeff + nodes[q]);
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int c = 0; c < GD; ++c) X[v][c] = __ldg(a.coords + (int64_t)nodes[v] * GD + c);
  Geom<GD> G;
  geometry<GD>(X, G);
  double y[NRN];
  ElemVec<F>::all(G, C, a.prm, y);
  if (a.contrib) { // deterministic mode: entries in place, summed per row in a fixed order
    double* dst = a.contrib + (c0 + lane) * NRN;
#pragma unroll
    for (int i = 0; i < NRN; ++i) dst[i] = y[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < NRN; ++i) atomicAdd(a.out + nodes[i], y[i]);
}

template <class F, bool AGG>
__global__ void __launch_bounds__(128, LOAM_GPU_CELL_MINB) k_cell_vec(const __grid_constant__ CellArgs a) {
  const int e0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e0 < a.n;
  if (!AGG && !valid) return;
  const int e = valid ? e0 : 0;
  double X[F::GD + 1][F::GD], C[F::HAS_COEFF ? F::NCOEFF : 1];
  int rows[F::NRN];
  cell_gather<F>(a, e, X, C, rows);
  Geom<F::GD> G;
  geometry<F::GD>(X, G);
  double y[F::NRN];
  ElemVec<F>::all(G, C, a.prm, y); // whole element vector (P2: through grad u_h)
  if (!AGG && a.contrib) { // deterministic mode (see k_cell_vec_rows)
#pragma unroll
    for (int i = 0; i < F::NRN; ++i) a.contrib[(int64_t)e * F::NRN + i] = y[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < F::NRN; ++i) red_add<AGG>(a.out, rows[i], y[i], valid);
}

// Deterministic mode's second pass: every row sums its (cell, local row)
// entries in the pair plan's fixed order (cells ascending) -- bitwise the same
// on every run, unlike fp64 REDs whose order varies.
__global__ void k_pair_sum(const int32_t* __restrict__ ptr, const int32_t* __restrict__ pairs, int nrows,
                           const double* __restrict__ contrib, double* __restrict__ out, int accumulate) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double acc = 0.0;
  for (int p = ptr[r]; p < ptr[r + 1]; ++p) acc += contrib[pairs[p]];
  out[r] = accumulate ? out[r] + acc : acc;
}

template <class F, bool AGG>
__global__ void __launch_bounds__(128) k_cell_mat(const __grid_constant__ CellArgs a) {
  const int e0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e0 < a.n;
  if (!AGG && !valid) return;
  const int e = valid ? e0 : 0;
  double X[F::GD + 1][F::GD], C[1];
  int rows[F::NRN];
  cell_gather<F>(a, e, X, C, rows);
  Geom<F::GD> G;
  geometry<F::GD>(X, G);
#pragma unroll
  for (int i = 0; i < F::NRN; ++i) {
    int rk[F::NCN];
    load_ranks<F::NCN>(a.cranks, (int64_t)e * F::NRN + i, rk);
    double blk[F::RD * F::NC];
    F::row(i, G, C, a.prm, blk);
#pragma unroll
    for (int d = 0; d < F::RD; ++d) {
      const int64_t base = __ldg(a.row_ptr + (int64_t)rows[i] * F::RD + d);
#pragma unroll
      for (int j = 0; j < F::NCN; ++j)
#pragma unroll
        for (int c = 0; c < F::CD; ++c)
          if (!diag_block<F>::value || d == c)
            red_add<AGG>(a.out, base + rk[j] * F::CD + c, blk[d * F::NC + j * F::CD + c], valid);
    }
  }
}

template <class F>
void launch_cell(const CellArgs& a, bool agg, cudaStream_t s) {
  if (a.n == 0) return;
  const int grid = ceil_div(a.n, 128);
  if constexpr (F::BILINEAR) {
    if (agg) k_cell_mat<F, true><<<grid, 128, 0, s>>>(a);
    else k_cell_mat<F, false><<<grid, 128, 0, s>>>(a);
  } else {
    // one sorted map for rows, coefficients and (its vertex prefix) coordinates
    const bool one_map = F::HAS_COEFF && F::NCOEFF == F::NRN && a.rmap == a.cmap && a.xmap == a.cmap &&
                         a.cstride == F::NRN && a.xstride == F::NRN && !std::getenv("LOAM_GPU_NO_CELL_ROWS");
    if constexpr (F::HAS_COEFF && F::NCOEFF == F::NRN) {
      if (!agg && one_map) {
        k_cell_vec_rows<F><<<ceil_div(a.n, 128), 128, 0, s>>>(a);
        count_launch();
        LG_LAUNCH_CHECK();
        return;
      }
    }
    if (agg) k_cell_vec<F, true><<<grid, 128, 0, s>>>(a);
    else k_cell_vec<F, false><<<grid, 128, 0, s>>>(a);
  }
  count_launch();
  LG_LAUNCH_CHECK();
}

// Cell-centric Dat INC with a warp-level segmented reduction (P2 actions,
// config 3 residual): a warp takes a batch of 32 consecutive cells (locality
// order); each lane computes its cell's element vector and stores entry i at
// the plan's slot -- the batch's 32 x NRN contributions sorted by row node --
// then the lanes sum the runs of equal nodes (fixed order) and issue one fp64
// RED per distinct node: 2.9x fewer REDs than one per element entry on the
// Kuhn meshes (the REDs bound the plain atomic kernel).
struct CellSegArgs {
  CellArgs c;
  const uint16_t* slots;     // [batch][NRN][32] position of (lane, i) in the batch's sorted order
  const int32_t* seg_off;    // [nbatches + 1] into seg_start / seg_node
  const uint16_t* seg_start; // per batch: nseg + 1 run starts (batch-local)
  const int32_t* seg_node;   // per segment: the row node
  int nbatches;
};

template <class F>
__global__ void __launch_bounds__(128) k_cell_seg(const __grid_constant__ CellSegArgs a) {
  constexpr int NRN = F::NRN;
  __shared__ double stage[4][32 * NRN];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int b = blockIdx.x * 4 + wl;
  if (b >= a.nbatches) return;
  const int e = b * 32 + lane;
  if (e < a.c.n) {
    double X[F::GD + 1][F::GD], C[F::HAS_COEFF ? F::NCOEFF : 1];
    int rows[NRN];
    cell_gather<F>(a.c, e, X, C, rows);
    Geom<F::GD> G;
    geometry<F::GD>(X, G);
    double y[NRN];
    ElemVec<F>::all(G, C, a.c.prm, y);
#pragma unroll
    for (int i = 0; i < NRN; ++i) stage[wl][__ldg(a.slots + ((int64_t)b * NRN + i) * 32 + lane)] = y[i];
  }
  __syncwarp();
  const int s0 = __ldg(a.seg_off + b), ns = __ldg(a.seg_off + b + 1) - s0;
  const uint16_t* st = a.seg_start + s0 + b; // nseg + 1 starts per batch
  for (int q = lane; q < ns; q += 32) {
    const int lo = __ldg(st + q), hi = __ldg(st + q + 1);
    double sum = stage[wl][lo];
    for (int t = lo + 1; t < hi; ++t) sum += stage[wl][t];
    atomicAdd(a.c.out + __ldg(a.seg_node + s0 + q), sum);
  }
}

template <class F>
void launch_cell_seg(const CellSegArgs& a, cudaStream_t s) {
  if constexpr (!F::BILINEAR) {
    if (a.nbatches == 0) return;
    k_cell_seg<F><<<ceil_div(a.nbatches, 4), 128, 0, s>>>(a);
    count_launch();
    LG_LAUNCH_CHECK();
  }
}

// Matrix (Mat INC): one warp per chunk of consecutive row nodes; one lane per
// DOF row (node row x component); the chunk's contiguous CSR value segment
// is accumulated in shared memory (single owner per row: plain adds) and
// stored coalesced.
template <class F>
__global__ void __launch_bounds__(128) k_owner_mat(const __grid_constant__ OwnerArgs a) {
  constexpr int U = batch_of<F>();
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int chunk = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (chunk >= a.nchunks) return;
  double* seg = smem + (threadIdx.x >> 5) * a.seg_max;
  const int r0 = __ldg(a.chunk_row + chunk), r1 = __ldg(a.chunk_row + chunk + 1);
  const int64_t base = __ldg(a.row_ptr + (int64_t)r0 * F::RD);
  const int len = (int)(__ldg(a.row_ptr + (int64_t)r1 * F::RD) - base);
  if (a.accumulate)
    for (int t = lane; t < len; t += 32) seg[t] = a.out[base + t];
  else
    for (int t = lane; t < len; t += 32) seg[t] = 0.0;
  __syncwarp();
  const int node = lane / F::RD, d = lane - node * F::RD;
  const int r = r0 + node;
  if (node < 32 / F::RD && r < r1) {
    const int64_t rs = __ldg(a.row_ptr + (int64_t)r * F::RD);
    const int nlen = (int)((__ldg(a.row_ptr + (int64_t)r * F::RD + 1) - rs) / F::CD); // column nodes
    const int rstart = (int)(rs - base) + d * nlen * F::CD;
    const int p1 = __ldg(a.ptr + r + 1);
    for (int p = __ldg(a.ptr + r); p < p1; p += U) {
      PairBatch<F, U> B;
      B.load(a, p, p1);
      int rk[U][F::NCN];
#pragma unroll
      for (int u = 0; u < U; ++u) load_ranks<F::NCN>(a.ranks, B.valid[u] ? p + u : p, rk[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!B.valid[u]) continue;
        const int i = B.code[u] % F::NRN;
        Geom<F::GD> G;
        geometry<F::GD>(B.X[u], G);
        double blk[F::NC];
        form_subrow<F>(i, d, G, nullptr, a.prm, blk);
        // distinct ranks within a pair: all shared loads, then all stores
        double cur[F::NC];
#pragma unroll
        for (int j = 0; j < F::NCN; ++j)
#pragma unroll
          for (int c = 0; c < F::CD; ++c) cur[j * F::CD + c] = seg[rstart + rk[u][j] * F::CD + c];
#pragma unroll
        for (int j = 0; j < F::NCN; ++j)
#pragma unroll
          for (int c = 0; c < F::CD; ++c) seg[rstart + rk[u][j] * F::CD + c] = cur[j * F::CD + c] + blk[j * F::CD + c];
      }
    }
  }
  __syncwarp();
  for (int t = lane; t < len; t += 32) a.out[base + t] = seg[t];
}

// ---------------------------------------------------------------------------
// Neighbour-list tile kernel (plan.cuh NbrPlan): P1 forms whose row, column
// and coordinate maps are one node map.  Persistent CTAs walk tiles of
// consecutive rows through a 3-deep ring of shared-memory stages.  For tile
// k+2, thread 0 issues TMA bulk copies (cp.async.bulk + mbarrier tx count) of
//   * the tile's contiguous plan ranges: row offsets, pair offsets, pair
//     records (in-row ranks), window slots of the pattern entries, own ranks;
//   * the tile's VERTEX WINDOW: the few contiguous runs of coordinates (and
//     coefficients) the tile references -- no per-entry gathers at all;
// then every thread computes tile k from shared memory: one thread per dof
// row walks its pair records, reads the cell's vertices as
// window[widx[rank]], computes its element row (cells are pre-rotated so the
// row is local vertex 0) and accumulates it -- in registers with
// compile-time slots when rows are short (LMAX), else in a shared segment --
// writing every output value exactly once.

struct TileArgs {
  const int32_t* tiles;
  int ntiles;
  const int32_t* nptr;
  const int32_t* pptr;
  const uint8_t* recs;
  const uint16_t* widx;
  const uint8_t* selfr;
  const int32_t* runs;
  const double* coords;
  const double* coeff;
  FormParams prm;
  double* out;
  int accumulate, bits, max_len;
  long long* timing; // unused (kept for ABI of the phase-timing tool)
  // dynamic shared memory layout (bytes)
  int off_seg, off_buf, buf_bytes;
  int b_nptr, b_pptr, b_recs, b_widx, b_selfr, b_win, b_winc; // inside one ring stage
};

constexpr int kTileThreads = 256;                 // consumer threads (8 warps)
constexpr int kTileBlock = kTileThreads + 32;     // + one TMA producer warp

template <class F, class Rec, int LMAX>
__global__ void __launch_bounds__(kTileBlock, 3) k_tile(const __grid_constant__ TileArgs a) {
  constexpr int GD = F::GD, W = F::RD * F::CD;
  constexpr int ES = sizeof(Rec);
  constexpr bool REG = F::BILINEAR && LMAX > 0;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);  // [3] stage landed (tx bytes)
  uint64_t* empty = full + 3;                          // [3] stage released by the 8 consumer warps
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kTileThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int K = a.ntiles > (int)blockIdx.x ? (a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto tile_meta = [&](int k, int (&m)[8]) {
    const int4* t = reinterpret_cast<const int4*>(a.tiles + 8 * (blockIdx.x + k * gridDim.x));
    const int4 x = __ldg(t), y = __ldg(t + 1);
    m[0] = x.x; m[1] = x.y; m[2] = x.z; m[3] = x.w; m[4] = y.x; m[5] = y.y; m[6] = y.z; m[7] = y.w;
  };
  auto ring = [&](int k) { return sm + a.off_buf + (k % 3) * a.buf_bytes; };
  auto issue = [&](int k) { // thread 0
    int m[8];
    tile_meta(k, m);
    unsigned char* buf = ring(k);
    uint64_t* bar = &full[k % 3];
    uint32_t tx = 0;
    auto range = [&](unsigned char* dst, const void* src, int lo, int hi, int es) {
      const int64_t s0 = ((int64_t)lo * es) & ~int64_t(15), s1 = ((int64_t)hi * es + 15) & ~int64_t(15);
      const uint32_t n = (uint32_t)(s1 - s0);
      if (n) bulk_g2s(dst, reinterpret_cast<const unsigned char*>(src) + s0, n, bar);
    };
    auto range_bytes = [](int lo, int hi, int es) {
      const int64_t s0 = ((int64_t)lo * es) & ~int64_t(15), s1 = ((int64_t)hi * es + 15) & ~int64_t(15);
      return (uint32_t)(s1 - s0);
    };
    tx += 2 * range_bytes(m[0], m[1] + 1, 4) + range_bytes(m[4], m[5], ES) + range_bytes(m[2], m[3], 2) +
          range_bytes(m[0], m[1], 1);
    // vertex window runs: 16-byte multiples by TMA, an 8-byte tail by hand
    double* win = reinterpret_cast<double*>(buf + a.b_win);
    double* winc = reinterpret_cast<double*>(buf + a.b_winc);
    int slot = 0;
    for (int r = 0; r < m[7]; ++r) {
      const int lo = __ldg(a.runs + 2 * (m[6] + r)), hi = __ldg(a.runs + 2 * (m[6] + r) + 1);
      const uint32_t nb = (uint32_t)(hi - lo) * GD * 8;
      tx += nb & ~15u;
      if (nb & 15) { // odd vertex count at the end of the array (GD odd): copy the last 8 bytes
        const int64_t e = (int64_t)hi * GD - 1;
        win[(int64_t)(slot + hi - lo) * GD - 1] = a.coords[e];
      }
      if constexpr (F::HAS_COEFF) {
        const uint32_t nc = (uint32_t)(hi - lo) * 8;
        tx += nc & ~15u;
        if (nc & 15) winc[slot + hi - lo - 1] = a.coeff[hi - 1];
      }
      slot += hi - lo;
    }
    fence_async_shared();
    mbar_arrive_expect_tx(bar, tx);
    range(buf + a.b_nptr, a.nptr, m[0], m[1] + 1, 4);
    range(buf + a.b_pptr, a.pptr, m[0], m[1] + 1, 4);
    range(buf + a.b_recs, a.recs, m[4], m[5], ES);
    range(buf + a.b_widx, a.widx, m[2], m[3], 2);
    range(buf + a.b_selfr, a.selfr, m[0], m[1], 1);
    slot = 0;
    for (int r = 0; r < m[7]; ++r) {
      const int lo = __ldg(a.runs + 2 * (m[6] + r)), hi = __ldg(a.runs + 2 * (m[6] + r) + 1);
      const uint32_t nb = ((uint32_t)(hi - lo) * GD * 8) & ~15u;
      if (nb) bulk_g2s(win + (int64_t)slot * GD, a.coords + (int64_t)lo * GD, nb, bar);
      if constexpr (F::HAS_COEFF) {
        const uint32_t nc = ((uint32_t)(hi - lo) * 8) & ~15u;
        if (nc) bulk_g2s(winc + slot, a.coeff + lo, nc, bar);
      }
      slot += hi - lo;
    }
  };

  if (tid >= kTileThreads) { // ---- producer warp: TMA issue only, up to 3 tiles ahead
    if (tid == kTileThreads)
      for (int k = 0; k < K; ++k) {
        if (k >= 3) mbar_wait_sleep(&empty[k % 3], (k / 3 - 1) & 1);
        issue(k);
      }
    return;
  }
  // ---- consumer warps
  double* seg = reinterpret_cast<double*>(sm + a.off_seg);
  const uint32_t mask = (1u << a.bits) - 1;
  long long t_wait = 0, t_comp = 0;
  for (int k = 0; k < K; ++k) {
    const long long c0 = a.timing ? clock64() : 0;
    int m[8];
    tile_meta(k, m);
    const int R0 = m[0], nrows = m[1] - m[0], A0 = m[2], nA = m[3] - m[2], P0 = m[4];
    const int64_t E0 = (int64_t)A0 * W;
    if constexpr (F::BILINEAR && !REG) {
      const int len = nA * W;
      if (a.accumulate)
        for (int t = tid; t < len; t += kTileThreads) seg[t] = a.out[E0 + t];
      else
        for (int t = tid; t < len; t += kTileThreads) seg[t] = 0.0;
      named_bar(1, kTileThreads);
    }
    mbar_wait(&full[k % 3], (k / 3) & 1);
    const long long c1 = a.timing ? clock64() : 0;
    const unsigned char* buf = ring(k);
    const int32_t* nptr_s = reinterpret_cast<const int32_t*>(buf + a.b_nptr) + skew_of(R0, 4);
    const int32_t* pptr_s = reinterpret_cast<const int32_t*>(buf + a.b_pptr) + skew_of(R0, 4);
    const Rec* recs_s = reinterpret_cast<const Rec*>(buf + a.b_recs) + skew_of(P0, ES);
    const uint16_t* widx_s = reinterpret_cast<const uint16_t*>(buf + a.b_widx) + skew_of(A0, 2);
    const uint8_t* selfr_s = buf + a.b_selfr + skew_of(R0, 1);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    const double* winc = reinterpret_cast<const double*>(buf + a.b_winc);
    const int node = tid / F::RD, d = tid - node * F::RD;
    if (node < nrows) {
      const int a0 = nptr_s[node] - A0;
      const int L = nptr_s[node + 1] - A0 - a0;
      const int rstart = a0 * W + d * L * F::CD - a0 * F::CD;
      const int p1 = pptr_s[node + 1] - P0;
      const int self = a0 + selfr_s[node];
      double racc[REG ? LMAX : 1];
      double diag = 0.0, acc = 0.0;
      double dblk[F::CD];
#pragma unroll
      for (int c = 0; c < F::CD; ++c) dblk[c] = 0.0;
      if constexpr (REG)
#pragma unroll
        for (int q = 0; q < LMAX; ++q) racc[q] = 0.0;
      auto vertex = [&](int rank, double (&x)[GD]) {
        const int wv = widx_s[rank];
        if constexpr (GD == 2) {
          const double2 c2 = reinterpret_cast<const double2*>(win)[wv];
          x[0] = c2.x;
          x[1] = c2.y;
        } else {
#pragma unroll
          for (int c = 0; c < GD; ++c) x[c] = win[wv * GD + c];
        }
      };
      double X0[GD];
      if (L > 0) vertex(self, X0); // L == 0: a row no cell of the loop touches (no pairs)
      for (int p = pptr_s[node] - P0; p < p1; p += 2) { // two pairs per iteration (ILP)
        constexpr int N = F::NRN;
        const bool two = p + 1 < p1;
        const uint32_t rec[2] = {(uint32_t)recs_s[p], (uint32_t)recs_s[two ? p + 1 : p]};
        int rr[2][N];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          rr[u][0] = self;
#pragma unroll
          for (int j = 1; j < N; ++j) rr[u][j] = a0 + ((rec[u] >> ((j - 1) * a.bits)) & mask);
        }
        double X[2][GD + 1][GD];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int c = 0; c < GD; ++c) X[u][0][c] = X0[c];
#pragma unroll
          for (int v = 1; v <= GD; ++v) vertex(rr[u][v], X[u][v]);
        }
        Geom<GD> G[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) geometry<GD>(X[u], G[u]);
        if constexpr (F::BILINEAR) {
          double blk[2][F::NC];
#pragma unroll
          for (int u = 0; u < 2; ++u) form_subrow<F>(0, d, G[u], nullptr, a.prm, blk[u]);
          if constexpr (REG) { // rotated local vertex 0 is the row node: blk[0] is diagonal
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const double wgt = (u == 0 || two) ? 1.0 : 0.0;
              diag = fma(wgt, blk[u][0], diag);
#pragma unroll
              for (int j = 1; j < F::NCN; ++j) {
                const int sl = rr[u][j] - a0;
                const double v = wgt * blk[u][j];
#pragma unroll
                for (int q = 0; q < LMAX; ++q)
                  if (sl == q) racc[q] += v;
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u == 1 && !two) break;
              // column block 0 is the row node itself: kept in registers
#pragma unroll
              for (int c = 0; c < F::CD; ++c) dblk[c] += blk[u][c];
#pragma unroll
              for (int j = 1; j < F::NCN; ++j) {
                double o[F::CD];
#pragma unroll
                for (int c = 0; c < F::CD; ++c) o[c] = seg[rstart + rr[u][j] * F::CD + c];
#pragma unroll
                for (int c = 0; c < F::CD; ++c) seg[rstart + rr[u][j] * F::CD + c] = o[c] + blk[u][j * F::CD + c];
              }
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            double C[F::HAS_COEFF ? F::NCOEFF : 1];
            if constexpr (F::HAS_COEFF)
#pragma unroll
              for (int q = 0; q < F::NCOEFF; ++q) C[q] = winc[widx_s[rr[u][q]]];
            double v;
            F::row(0, G[u], C, a.prm, &v);
            if (u == 0 || two) acc += v;
          }
        }
      }
      if constexpr (!F::BILINEAR) a.out[R0 + node] = a.accumulate ? a.out[R0 + node] + acc : acc;
      if constexpr (F::BILINEAR && !REG)
        if (L > 0)
#pragma unroll
          for (int c = 0; c < F::CD; ++c) seg[rstart + self * F::CD + c] += dblk[c];
      if constexpr (REG) { // the row straight from registers (scalar rows: W == 1)
        double* o = a.out + E0 + a0;
#pragma unroll
        for (int q = 0; q < LMAX; ++q)
          if (q < L) {
            const double v = racc[q] + (q == self - a0 ? diag : 0.0);
            o[q] = a.accumulate ? o[q] + v : v;
          }
      }
    }
    __syncwarp();
    if (a.timing) {
      t_wait += c1 - c0;
      t_comp += clock64() - c1;
    }
    if ((tid & 31) == 0) mbar_arrive(&empty[k % 3]); // this warp is done with stage k%3
    if constexpr (F::BILINEAR && !REG) {
      named_bar(1, kTileThreads); // segment complete
      const int len = nA * W;
      for (int t = tid; t < len; t += kTileThreads) a.out[E0 + t] = seg[t];
      named_bar(1, kTileThreads); // segment drained before the next tile reuses it
    }
  }
  if (a.timing && (tid & 31) == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.timing), (unsigned long long)t_wait);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.timing) + 1, (unsigned long long)t_comp);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.timing) + 2, (unsigned long long)K);
  }
}

// ---------------------------------------------------------------------------
// Ring kernel (NbrPlan ring mode: P1 triangles on a manifold mesh).  Same
// producer/consumer TMA pipeline as k_tile, but each row's cells arrive in
// ring / fan order as one 16-bit record per chain vertex (window slot << 3 |
// in-row rank): a cell is (row vertex, previous chain vertex, new vertex), so
// one vertex is fetched per cell, and every off-diagonal entry is complete
// after two consecutive cells -- written once with a plain store.
struct RingArgs {
  const int32_t* tiles;
  int ntiles;
  int* next_tile;  // dynamic scheduler counter of this launch (zeroed by the previous launch)
  int* reset_tile; // counter of the next launch: zeroed here
  const int32_t* nptr;
  const int32_t* rptr;
  const uint16_t* recs;
  const uint32_t* rowinfo;
  const int32_t* runs;
  const double* coords;
  const double* coeff;
  FormParams prm;
  double* out;
  int accumulate;
  int off_seg, seg_stride, off_buf, buf_bytes; // seg_stride: doubles in the segment buffer
  int b_nptr, b_rptr, b_recs, b_info, b_win, b_winc;
  unsigned long long* timing; // LOAM_GPU_PHASE_TIMING: [first wait, waits, compute, tiles] in cycles
};

// One ring cell (s, p, n) of a P1 triangle form seen from the row vertex s,
// in closed form from the edge vectors a = x_p - x_s, b = x_n - x_s
// (aa = a.a, ab = a.b, bb = b.b, ad = |a x b| = 2 |T|):
//   K_sp = (ab - bb) / (2 ad),  K_sn = (ab - aa) / (2 ad),  K_ss = -(K_sp + K_sn)
//   M_ss = ad / 12,             M_sp = M_sn = ad / 24
// -- the same entries elements.cuh's barycentric-gradient row produces
// (cotangent form of grad l_i . grad l_j |T|; P1 mass |T|/12 (1 + delta_ij)),
// at a third of the arithmetic: b.b of one cell is a.a of the next.
template <class F>
struct RingCell {
  static constexpr int ID = F::ID;
  static constexpr bool K = ID != F_MASS && ID != F_MASS_ACTION;
  static constexpr bool M = ID != F_STIFFNESS && ID != F_STIFFNESS_ACTION;
  // bilinear: the s-row entries for s, p, n
  __device__ __forceinline__ static void entries(double aa, double ab, double bb, double ad, double kappa,
                                                 double& vs, double& vp, double& vn) {
    double kp = 0.0, kn = 0.0;
    if constexpr (K) {
      const double r = fast_half_rcp(ad);
      kp = (ab - bb) * r;
      kn = (ab - aa) * r;
    }
    if constexpr (!M) {
      vp = kp;
      vn = kn;
      vs = -(kp + kn);
    } else {
      const double m = ad * (1.0 / 24.0);
      const double km = K ? kappa * m : m;
      vp = kp + km;
      vn = kn + km;
      vs = K ? fma(2.0, km, -(kp + kn)) : 2.0 * m;
    }
  }
  // action: sum_j A_sj u_j
  __device__ __forceinline__ static double action(double aa, double ab, double bb, double ad, double kappa,
                                                  double us, double up, double un) {
    double v = 0.0;
    if constexpr (K) {
      const double r = fast_half_rcp(ad);
      v = ((ab - bb) * (up - us) + (ab - aa) * (un - us)) * r;
    }
    if constexpr (M) {
      const double m = ad * (1.0 / 24.0) * (2.0 * us + up + un);
      v = K ? fma(kappa, m, v) : m;
    }
    return v;
  }
};

// Vertex-star kernel for P1 triangle ACTIONS (config 1 shape): one thread per
// row vertex s.  Its star -- the link vertices v_0..v_{m-1} of the cells
// around s, in ring / fan order -- is one 32-byte record {m | closed << 4,
// v_0..v_6}; the cells are (s, v_k, v_{k+1}) (and (s, v_{m-1}, v_0) when the
// ring is closed); the header packs m (3 bits), closed (1), the in-row CSR
// rank of s (3) and of every v_k (3 each).  Two dependent gathers per row (record, then the
// neighbours' coordinates and coefficients), the action in closed form
// (RingCell::action), one store: no plan tiles, no shared memory, no
// atomics -- the short latency chain a 15 MB loop needs.
struct StarArgs {
  const int4* star; // 2 per row
  int nrows;
  const int64_t* row_ptr; // Mats: CSR offsets
  const double* coords;
  const double* coeff;
  FormParams prm;
  double* out;
  int accumulate;
};

struct CoeffLoad {
  const double* c;
  __device__ __forceinline__ double operator()(int v) const { return __ldg(c + v); }
};

template <class F, class Coef = CoeffLoad>
__device__ __forceinline__ double star_row(const StarArgs& a, int r, int4 h, int4 t, Coef coef = Coef{nullptr}) {
  if constexpr (std::is_same_v<Coef, CoeffLoad>) coef.c = a.coeff;
  const int m = h.x & 7;
  const bool closed = (h.x >> 3) & 1;
  const int v[7] = {h.y, h.z, h.w, t.x, t.y, t.z, t.w};
  const double2 xs = __ldg(reinterpret_cast<const double2*>(a.coords) + r);
  const double us = coef(r);
  // every neighbour gather is issued before the first use: one dependent
  // round trip after the star record instead of one per link vertex
  double2 X[7];
  double U[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const int vk = k < m ? v[k] : r;
    X[k] = __ldg(reinterpret_cast<const double2*>(a.coords) + vk);
    U[k] = coef(vk);
  }
  double px = 0, py = 0, up = 0, p0x = 0, p0y = 0, u0 = 0, aa = 0;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    if (k < m) {
      const double2 x = X[k];
      const double u = U[k];
      const double nx = x.x - xs.x, ny = x.y - xs.y, nn = nx * nx + ny * ny;
      if (k == 0) {
        p0x = nx;
        p0y = ny;
        u0 = u;
      } else { // cell (s, v_{k-1}, v_k)
        const double ab = px * nx + py * ny, ad = fabs(px * ny - py * nx);
        acc += RingCell<F>::action(aa, ab, nn, ad, a.prm.p[0], us, up, u);
      }
      px = nx;
      py = ny;
      up = u;
      aa = nn;
    }
  }
  if (closed && m > 2) { // closing cell (s, v_{m-1}, v_0)
    const double nn = p0x * p0x + p0y * p0y;
    const double ab = px * p0x + py * p0y, ad = fabs(px * p0y - py * p0x);
    acc += RingCell<F>::action(aa, ab, nn, ad, a.prm.p[0], us, up, u0);
  }
  return acc;
}

// RPT rows per thread (r, r + stride, ...): their independent record ->
// neighbour gather chains overlap, and the grid fits in one wave (one wave of
// 256-thread blocks at 48 registers holds 740 blocks; C1 has 263,169 rows).
template <class F, int RPT>
__global__ void __launch_bounds__(256) k_star_vec(const __grid_constant__ StarArgs a) {
  // PDL: let the next kernel's prologue start; load this row's star record
  // (plan data, library-owned) before waiting for the previous kernel
  if (threadIdx.x == 0) grid_dep_launch();
  const int r0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  int4 h[RPT], t[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = r0 + q * stride;
    if (r < a.nrows) {
      h[q] = __ldg(a.star + 2 * r);
      t[q] = __ldg(a.star + 2 * r + 1);
    }
  }
  grid_dep_wait(); // coordinates, coefficients and the output after the previous kernel
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = r0 + q * stride;
    if (r < a.nrows) {
      const double y = star_row<F>(a, r, h[q], t[q]);
      a.out[r] = a.accumulate ? a.out[r] + y : y;
    }
  }
}

// Bilinear P1 triangle forms (config 2 shape): the row's CSR segment is
// {s} u {v_k} (a manifold star), so the thread accumulates the diagonal and
// one register per link vertex over the cells (RingCell::entries, closed
// form) and writes the m + 1 values at row_ptr[s] + their packed ranks.
template <class F>
__global__ void __launch_bounds__(256) k_star_mat(const __grid_constant__ StarArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  const int4 h = __ldg(a.star + 2 * r), t = __ldg(a.star + 2 * r + 1);
  const int hdr = h.x, m = hdr & 7;
  const bool closed = (hdr >> 3) & 1;
  const int v[7] = {h.y, h.z, h.w, t.x, t.y, t.z, t.w};
  const int64_t base = __ldg(a.row_ptr + r);
  const double2 xs = __ldg(reinterpret_cast<const double2*>(a.coords) + r);
  double acc[7], self = 0.0;
  double px = 0, py = 0, p0x = 0, p0y = 0, aa = 0;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    acc[k] = 0.0;
    if (k < m) {
      const double2 x = __ldg(reinterpret_cast<const double2*>(a.coords) + v[k]);
      const double nx = x.x - xs.x, ny = x.y - xs.y, nn = nx * nx + ny * ny;
      if (k == 0) {
        p0x = nx;
        p0y = ny;
      } else { // cell (s, v_{k-1}, v_k)
        const double ab = px * nx + py * ny, ad = fabs(px * ny - py * nx);
        double vs, vp, vn;
        RingCell<F>::entries(aa, ab, nn, ad, a.prm.p[0], vs, vp, vn);
        self += vs;
        acc[k - 1] += vp;
        acc[k] += vn;
      }
      px = nx;
      py = ny;
      aa = nn;
    }
  }
  if (closed && m > 2) { // closing cell (s, v_{m-1}, v_0)
    const double nn = p0x * p0x + p0y * p0y;
    const double ab = px * p0x + py * p0y, ad = fabs(px * p0y - py * p0x);
    double vs, vp, vn;
    RingCell<F>::entries(aa, ab, nn, ad, a.prm.p[0], vs, vp, vn);
    self += vs;
#pragma unroll
    for (int k = 0; k < 7; ++k)
      if (k == m - 1) acc[k] += vp;
    acc[0] += vn;
  }
  double* o = a.out + base;
  const int rs = (hdr >> 4) & 7;
  o[rs] = a.accumulate ? o[rs] + self : self;
#pragma unroll
  for (int k = 0; k < 7; ++k)
    if (k < m) {
      const int rk = (hdr >> (7 + 3 * k)) & 7;
      o[rk] = a.accumulate ? o[rk] + acc[k] : acc[k];
    }
}

template <class F>
void launch_star(const StarArgs& a, cudaStream_t s) {
  if (a.nrows == 0) return;
  if constexpr (F::BILINEAR) k_star_mat<F><<<ceil_div(a.nrows, 256), 256, 0, s>>>(a);
  else {
    static const int rpt = std::getenv("LOAM_GPU_STAR_RPT") ? std::atoi(std::getenv("LOAM_GPU_STAR_RPT")) : 1;
    if (rpt >= 4) launch_pdl(k_star_vec<F, 4>, dim3(ceil_div(a.nrows, 256 * 4)), dim3(256), 0, s, a);
    else if (rpt == 2) launch_pdl(k_star_vec<F, 2>, dim3(ceil_div(a.nrows, 256 * 2)), dim3(256), 0, s, a);
    else launch_pdl(k_star_vec<F, 1>, dim3(ceil_div(a.nrows, 256)), dim3(256), 0, s, a);
  }
  count_launch();
  LG_LAUNCH_CHECK();
}

// ---- the run_wave time step fused into the vertex-star action -------------
// bench::run_wave (bench.hpp:267-289) per step:
//   phi -= dt/2 p;  b = K phi;  p += b * pc;  p[bc] = forcing;  phi -= dt/2 p;  |p|_inf
// Every update but the action is pointwise and the star kernel owns its
// vertex row, so one kernel does the step: the half-kick phi - (dt/2) p of
// every gathered neighbour is formed on the fly from the previous step's
// fields (ping-pong buffers: no thread reads what another writes), then the
// owner applies the kick, the Dirichlet forcing and the second half-kick to
// its vertex and folds |p| into the step's maximum.  The arithmetic is the
// pointwise engine's (__dmul_rn / __dsub_rn / __dadd_rn, no contraction)
// and the star kernel's, so the fields equal the unfused chain bitwise.
struct WaveFields {
  const double* p_in;
  const double* phi_in;
  double* p_out;
  double* phi_out;
  const double* pc;
  const uint8_t* bc;  // 1 on the Dirichlet vertices
  double half_dt;
  double* state;      // [1] forcing value, [2] |p|_inf (max-folded; zeroed by the clock)
};

struct HalfKick {
  const double* phi;
  const double* p;
  double h;
  __device__ __forceinline__ double operator()(int v) const {
    return __dsub_rn(__ldg(phi + v), __dmul_rn(h, __ldg(p + v)));
  }
};

template <class F>
__global__ void __launch_bounds__(256) k_wave_step(const __grid_constant__ StarArgs a, const __grid_constant__ WaveFields w) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (r < a.nrows) {
    const int4 h = __ldg(a.star + 2 * r), t = __ldg(a.star + 2 * r + 1);
    const HalfKick hk{w.phi_in, w.p_in, w.half_dt};
    const double b = star_row<F>(a, r, h, t, hk);
    double p = __dadd_rn(__ldg(w.p_in + r), __dmul_rn(b, __ldg(w.pc + r)));
    if (w.bc[r]) p = w.state[1];
    w.p_out[r] = p;
    w.phi_out[r] = __dsub_rn(hk(r), __dmul_rn(w.half_dt, p));
    m = fabs(p);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) m = fmax(m, wm[q]);
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(w.state + 2), (unsigned long long)__double_as_longlong(m));
  }
}

// Star records of the node map (host build; false if a star is not a single
// ring or fan of <= 7 link vertices).
// build_stars on the device: one thread per vertex, its link edges from the
// pair plan (cells ascending, as the host loop meets them), the same chain
// and header -- bitwise the host's records (tests/test_ring_plan_gpu.py).
__global__ void k_star_plan(const int32_t* __restrict__ cv, const int32_t* __restrict__ ptr,
                            const int32_t* __restrict__ pairs, int nverts, int4* __restrict__ rec, int* fail) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nverts) return;
  const int b = ptr[r], nl = ptr[r + 1] - b;
  int lx[7], ly[7], chain[8], m = 0;
  bool closed = false;
  if (nl > 7) { atomicExch(fail, 1); return; }
  for (int k = 0; k < nl; ++k) {
    const int code = pairs[b + k], c = code / 3, i = code - 3 * c;
    lx[k] = cv[(int64_t)c * 3 + (i + 1) % 3];
    ly[k] = cv[(int64_t)c * 3 + (i + 2) % 3];
  }
  if (nl > 0) {
    auto deg = [&](int x) {
      int d = 0;
      for (int k = 0; k < nl; ++k) d += (lx[k] == x) + (ly[k] == x);
      return d;
    };
    int start = lx[0], ends = 0;
    for (int k = 0; k < nl; ++k)
      for (int u = 0; u < 2; ++u) {
        const int x = u ? ly[k] : lx[k];
        const int d = deg(x);
        if (d > 2 || x == r) { atomicExch(fail, 1); return; }
        if (d == 1) ++ends;
      }
    if (ends != 0 && ends != 2) { atomicExch(fail, 1); return; }
    if (ends == 2) { // the smaller end id, deterministic
      start = INT_MAX;
      for (int k = 0; k < nl; ++k)
        for (int u = 0; u < 2; ++u) {
          const int x = u ? ly[k] : lx[k];
          if (deg(x) == 1) start = min(start, x);
        }
    }
    closed = ends == 0;
    unsigned used = 0u;
    int cur = start;
    chain[m++] = cur;
    for (int step = 0; step < nl; ++step) {
      int nxt = -1;
      for (int k = 0; k < nl; ++k) {
        if (used >> k & 1u) continue;
        if (lx[k] == cur) nxt = ly[k];
        else if (ly[k] == cur) nxt = lx[k];
        else continue;
        used |= 1u << k;
        break;
      }
      if (nxt < 0) { atomicExch(fail, 1); return; } // several components
      if (closed && step == nl - 1) {
        if (nxt != start) { atomicExch(fail, 1); return; }
        break;
      }
      if (m == 8) { atomicExch(fail, 1); return; }
      chain[m++] = nxt;
      cur = nxt;
    }
    if (m > 7 || (closed ? m != nl : m != nl + 1)) { atomicExch(fail, 1); return; }
  }
  int v[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < m; ++k) v[k] = chain[k];
  int hdr = m | (closed ? 8 : 0);
  int rank_self = 0;
  for (int k = 0; k < m; ++k) rank_self += v[k] < r;
  hdr |= rank_self << 4;
  for (int k = 0; k < m; ++k) {
    int rk = v[k] > r;
    for (int q = 0; q < m; ++q) rk += v[q] < v[k];
    hdr |= rk << (7 + 3 * k);
  }
  rec[2 * r] = make_int4(hdr, v[0], v[1], v[2]);
  rec[2 * r + 1] = make_int4(v[3], v[4], v[5], v[6]);
}

bool build_stars_dev(const int32_t* dmap, int ncells, int nverts, DevBuf<int4>& out, cudaStream_t s) {
  PairPlan pp;
  build_pairs(dmap, ncells, 3, nverts, pp, s);
  out.alloc(2 * (size_t)std::max(nverts, 1), s);
  DevBuf<int> fail(1, s);
  LG_CUDA(cudaMemsetAsync(fail.get(), 0, sizeof(int), s));
  if (nverts) {
    k_star_plan<<<ceil_div(nverts, 256), 256, 0, s>>>(dmap, pp.ptr.get(), pp.pairs.get(), nverts, out.get(), fail.get());
    count_launch();
    LG_LAUNCH_CHECK();
  }
  int h = 0;
  LG_CUDA(cudaMemcpyAsync(&h, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

bool build_stars(const int32_t* dmap, int ncells, int nverts, DevBuf<int4>& out, cudaStream_t s) {
  std::vector<int32_t> cv((size_t)ncells * 3);
  LG_CUDA(cudaMemcpyAsync(cv.data(), dmap, sizeof(int32_t) * cv.size(), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  // link edges {p, q} of every vertex, CSR by vertex
  std::vector<int32_t> cnt(nverts + 1, 0);
  for (size_t e = 0; e < (size_t)ncells; ++e)
    for (int i = 0; i < 3; ++i) ++cnt[cv[e * 3 + i] + 1];
  for (int v = 0; v < nverts; ++v) cnt[v + 1] += cnt[v];
  std::vector<int2> link(cnt[nverts]);
  {
    std::vector<int32_t> f(cnt.begin(), cnt.end() - 1);
    for (size_t e = 0; e < (size_t)ncells; ++e)
      for (int i = 0; i < 3; ++i) {
        const int r = cv[e * 3 + i];
        link[f[r]++] = make_int2(cv[e * 3 + (i + 1) % 3], cv[e * 3 + (i + 2) % 3]);
      }
  }
  std::vector<int4> rec(2 * (size_t)nverts);
  for (int r = 0; r < nverts; ++r) {
    const int b = cnt[r], e = cnt[r + 1], nl = e - b;
    int chain[8], m = 0;
    bool closed = false;
    if (nl > 0) {
      if (nl > 7) return false;
      // link-graph degrees; start at a degree-1 end (fan) or anywhere (ring)
      auto deg = [&](int x) {
        int d = 0;
        for (int k = b; k < e; ++k) d += (link[k].x == x) + (link[k].y == x);
        return d;
      };
      int start = link[b].x, ends = 0;
      for (int k = b; k < e; ++k)
        for (int x : {link[k].x, link[k].y}) {
          const int d = deg(x);
          if (d > 2 || x == r) return false;
          if (d == 1) ++ends;
        }
      if (ends != 0 && ends != 2) return false;
      if (ends == 2) { // the smaller end id, deterministic
        start = INT32_MAX;
        for (int k = b; k < e; ++k)
          for (int x : {link[k].x, link[k].y})
            if (deg(x) == 1) start = std::min(start, x);
      }
      closed = ends == 0;
      uint32_t used = 0;
      int cur = start;
      chain[m++] = cur;
      for (int step = 0; step < nl; ++step) {
        int nxt = -1;
        for (int k = b; k < e; ++k) {
          if (used >> (k - b) & 1u) continue;
          if (link[k].x == cur) nxt = link[k].y;
          else if (link[k].y == cur) nxt = link[k].x;
          else continue;
          used |= 1u << (k - b);
          break;
        }
        if (nxt < 0) return false; // several components
        if (closed && step == nl - 1) {
          if (nxt != start) return false;
          break;
        }
        chain[m++] = nxt;
        cur = nxt;
      }
      if (m > 7 || (closed ? m != nl : m != nl + 1)) return false;
    }
    int v[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < m; ++k) v[k] = chain[k];
    // in-row ranks (CSR columns ascending): of the row vertex and of each link vertex
    int hdr = m | (closed ? 8 : 0);
    {
      int rank_self = 0;
      for (int k = 0; k < m; ++k) rank_self += v[k] < r;
      hdr |= rank_self << 4;
      for (int k = 0; k < m; ++k) {
        int rk = v[k] > r;
        for (int q = 0; q < m; ++q) rk += v[q] < v[k];
        hdr |= rk << (7 + 3 * k);
      }
    }
    rec[2 * r] = make_int4(hdr, v[0], v[1], v[2]);
    rec[2 * r + 1] = make_int4(v[3], v[4], v[5], v[6]);
  }
  out.alloc(rec.size(), s);
  LG_CUDA(cudaMemcpyAsync(out.get(), rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

#ifndef LOAM_GPU_RING_STAGES
#define LOAM_GPU_RING_STAGES 3
#endif
#ifndef LOAM_GPU_RING_MINB
#define LOAM_GPU_RING_MINB 3
#endif
#ifndef LOAM_GPU_RING_STG
#define LOAM_GPU_RING_STG 0
#endif
constexpr bool kRingStg = LOAM_GPU_RING_STG != 0;    // warp slices by coalesced st.global instead of TMA (measured slower: 22.8 vs 22.3 us)
constexpr int kRS = LOAM_GPU_RING_STAGES;            // ring pipeline stages
constexpr int kRingMinBlocks = LOAM_GPU_RING_MINB;   // CTAs per SM the registers are sized for
static_assert(2 * 8 * kRS + 4 * kRS <= 128, "ring barriers + stage ids fit the 128-byte header");

template <class F, bool ACC>
__global__ void __launch_bounds__(kTileBlock, kRingMinBlocks) k_ring(const __grid_constant__ RingArgs a) {
  static_assert(F::GD == 2 && F::NRN == 3, "ring kernel: P1 triangles");
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + kRS;
  int* slot_tile = reinterpret_cast<int*>(full + 2 * kRS); // [kRS] tile id carried by each ring stage (-1: done)
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < kRS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kTileThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // PDL: the next PDL-launched kernel may start its prologue (it waits for
  // this grid's completion before touching anything this grid writes)
  if (tid == 0) grid_dep_launch();
  auto ring = [&](int k) { return sm + a.off_buf + (k % kRS) * a.buf_bytes; };
  // tile records of this CTA, 8 tiles per batch, double-buffered (cp.async);
  // the meta of the tile in each ring stage, handed to the consumers with it
  __shared__ __align__(16) int meta_s[2][8 * 16];
  __shared__ int stage_meta[kRS][8];
  if (tid >= kTileThreads) { // ---- producer warp
    // Static schedule: tile k of this CTA is blockIdx + k * grid (tiles cost
    // about the same).  The 64-byte tile records (meta + the first window
    // runs) arrive 8 tiles at a time by cp.async, one batch ahead, so the
    // producer's per-tile chain holds no dependent global round trip (the
    // former dynamic counter cost an atomic, a record load and a run load
    // per tile, ~3 round trips -- the consumers waited ~1k cycles per tile).
    const int lane = tid & 31;
    auto load_batch = [&](int b) { // tiles 8b..8b+7 -> meta_s[b & 1]; lane = (tile in batch, 16-byte part)
      const int kk = 8 * b + (lane >> 2), part = lane & 3;
      const int tile = blockIdx.x + kk * gridDim.x;
      if (tile < a.ntiles) cp_async16(&meta_s[b & 1][(lane >> 2) * 16 + part * 4], a.tiles + 16 * tile + part * 4);
      cp_async_commit();
    };
    load_batch(0);
    load_batch(1);
    for (int k = 0;; ++k) {
      const int tile = blockIdx.x + k * gridDim.x;
      if (k % 8 == 0) {
        cp_async_wait<1>(); // batch k / 8 has landed (the next one may still be in flight)
        __syncwarp();
      }
      const int* rec = &meta_s[(k / 8) & 1][(k % 8) * 16];
      int m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int2 run0 = make_int2(0, 0);
      if (tile < a.ntiles) { // (past the end the batch slot was never filled)
#pragma unroll
        for (int q = 0; q < 8; ++q) m[q] = rec[q];
        const int cnt = m[7];
        if (lane < cnt)
          run0 = lane < kRingInlineRuns ? reinterpret_cast<const int2*>(rec + 8)[lane]
                                        : __ldg(reinterpret_cast<const int2*>(a.runs) + m[6] + lane);
      }
      if (k % 8 == 7) {
        __syncwarp(); // every lane has read batch k / 8: refill its buffer
        load_batch(k / 8 + 2);
      }
      if (k >= kRS) mbar_wait_sleep(&empty[k % kRS], (k / kRS - 1) & 1);
      if (tile >= a.ntiles) { // publish "no more tiles" through the stage
        if (lane == 0) {
          slot_tile[k % kRS] = -1;
          mbar_arrive(&full[k % kRS]);
        }
        break;
      }
      if (lane < 8) stage_meta[k % kRS][lane] = m[lane];
      if (lane == 0) slot_tile[k % kRS] = tile;
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % kRS];
      auto rb = [](int lo, int hi, int es, int64_t& s0) {
        s0 = ((int64_t)lo * es) & ~int64_t(15);
        return (uint32_t)((((int64_t)hi * es + 15) & ~int64_t(15)) - s0);
      };
      int64_t g0, g1, g2, g3;
      const uint32_t n0 = F::BILINEAR ? rb(m[0], m[1] + 1, 4, g0) : (g0 = 0, 0u);
      const uint32_t n1 = rb(m[0], m[1] + 1, 4, g1), n2 = rb(m[4], m[5], 2, g2), n3 = rb(m[0], m[1], 4, g3);
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + m[6], m[7], a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), 2};
      const RunSet rk{reinterpret_cast<const int2*>(a.runs) + m[6], F::HAS_COEFF ? m[7] : 0, a.coeff,
                      reinterpret_cast<double*>(buf + a.b_winc), 1};
      // plan ranges (library-owned, immutable: safe before the PDL wait)
      if (lane == 0) {
        mbar_expect_tx(bar, n0 + n1 + n2 + n3);
        if (n0) bulk_g2s(buf + a.b_nptr, reinterpret_cast<const unsigned char*>(a.nptr) + g0, n0, bar);
        bulk_g2s(buf + a.b_rptr, reinterpret_cast<const unsigned char*>(a.rptr) + g1, n1, bar);
        if (n2) bulk_g2s(buf + a.b_recs, reinterpret_cast<const unsigned char*>(a.recs) + g2, n2, bar);
        if (n3) bulk_g2s(buf + a.b_info, reinterpret_cast<const unsigned char*>(a.rowinfo) + g3, n3, bar);
      }
      // the caller's data (coordinates / coefficients) only after every
      // prerequisite grid has completed
      if (k == 0) grid_dep_wait();
      const uint32_t tx = stage_runs<false>(rc, lane, bar, run0) + stage_runs<false>(rk, lane, bar, run0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(bar, tx);
      __syncwarp();
      stage_runs<true>(rc, lane, bar, run0);
      stage_runs<true>(rk, lane, bar, run0);
    }
    if (a.ntiles <= (int)blockIdx.x) grid_dep_wait(); // (no tile: still order the exit)
    cp_async_wait<0>();
    return;
  }
  // ---- consumers: one thread per row vertex
  double* seg = reinterpret_cast<double*>(sm + a.off_seg);
  const double kappa = a.prm.p[0];
  const long long t_start = clock64();
  long long t_first = 0, t_wait = 0, t_comp = 0, t_n = 0, t_early = 0, t_last = 0;
  for (int k = 0;; ++k) {
    const long long c0 = a.timing ? clock64() : 0;
    mbar_wait(&full[k % kRS], (k / kRS) & 1);
    const long long c1 = a.timing ? clock64() : 0;
    const int tile = slot_tile[k % kRS];
    if (a.timing) {
      if (k == 0) t_first += c1 - c0;
      else if (tile < 0) t_last += c1 - c0;
      else if (k < kRS) t_early += c1 - c0;
      else t_wait += c1 - c0;
    }
    if (tile < 0) break;
    if (k == 0) grid_dep_wait(); // (returns at once: the producer has waited)
    int m[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) m[q] = stage_meta[k % kRS][q];
    const int R0 = m[0], nrows = m[1] - m[0], P0 = m[4];
    (void)m[3];
    // every warp owns its 32 rows' CSR values (a contiguous range [W0, W1))
    // in its own shared slice, skewed so wsegb[t] and out[W0 + t] agree mod
    // 16 bytes, and stores it with its own bulk copy: no CTA-wide barrier
    // per tile (the previous store of this warp must have read the slice)
    const int wl = tid >> 5, lane = tid & 31;
    const int* nptr_w = reinterpret_cast<const int32_t*>(ring(k) + a.b_nptr) + skew_of(R0, 4);
    const int W0 = F::BILINEAR ? nptr_w[min(32 * wl, nrows)] : 0;
    const int W1 = F::BILINEAR ? nptr_w[min(32 * wl + 32, nrows)] : 0;
    double* segb = seg + wl * a.seg_stride + (W0 & 1) - W0; // indexed by the global CSR offset
    if constexpr (F::BILINEAR) {
      if (!kRingStg && lane == 0) bulk_wait_read<0>();
      __syncwarp();
      if constexpr (ACC) {
        for (int t = W0 + lane; t < W1; t += 32) segb[t] = a.out[t];
        __syncwarp();
      }
    }
    const long long c1b = a.timing ? clock64() : 0;
    const unsigned char* buf = ring(k);
    const int32_t* nptr_s = reinterpret_cast<const int32_t*>(buf + a.b_nptr) + skew_of(R0, 4);
    const int32_t* rptr_s = reinterpret_cast<const int32_t*>(buf + a.b_rptr) + skew_of(R0, 4);
    const uint16_t* rec_s = reinterpret_cast<const uint16_t*>(buf + a.b_recs) + skew_of(P0, 2);
    const uint32_t* info_s = reinterpret_cast<const uint32_t*>(buf + a.b_info) + skew_of(R0, 4);
    const double2* win = reinterpret_cast<const double2*>(buf + a.b_win);
    const double* winc = reinterpret_cast<const double*>(buf + a.b_winc);
    if (tid < nrows) {
      const uint32_t info = info_s[tid];
      const int self_slot = info & 0xffff, self_rank = (info >> 16) & 0xff;
      const int q0 = rptr_s[tid] - P0, q1 = rptr_s[tid + 1] - P0;
      double* row = segb + (F::BILINEAR ? nptr_s[tid] : 0);
      auto put = [&](int rank, double v) {
        if constexpr (ACC) row[rank] += v;
        else row[rank] = v;
      };
      const double2 xs = win[self_slot];
      const double us = F::HAS_COEFF ? winc[self_slot] : 0.0;
      // a chain record is (window slot << 4 | in-row rank): the slot's byte
      // offset in the double2 window is the record with the rank masked off
      const unsigned char* winb = reinterpret_cast<const unsigned char*>(win);
      auto wx = [&](uint32_t r) { return *reinterpret_cast<const double2*>(winb + (r & 0xfff0u)); };
      auto wc = [&](uint32_t r) { return winc[r >> 4]; };
      // chain vertex 0 (a row with no cell has q1 == q0 + 1 and no pair)
      const uint32_t h0 = rec_s[q0];
      const int rk0 = h0 & 7;
      double2 ea;
      {
        const double2 x = wx(h0);
        ea = make_double2(x.x - xs.x, x.y - xs.y);
      }
      double aa = ea.x * ea.x + ea.y * ea.y;
      double up = F::HAS_COEFF ? wc(h0) : 0.0;
      // pure stiffness: the diagonal is minus the sum of the row's
      // off-diagonal entries (the same cell terms, summed per entry)
      constexpr bool kDiagBySum = F::BILINEAR && RingCell<F>::K && !RingCell<F>::M;
      double diag = 0.0, first = 0.0, carry = 0.0, acc = 0.0;
      int rkp = rk0;
      // one cell (s, chain vertex with edge e0 / e0.e0 = a0, chain vertex at x):
      // returns its edge and |edge|^2 for the next cell
      auto cell = [&](const double2& e0, double a0, const double2& x, double2& e1, double& b1, double un,
                      double& vp, double& vn) {
        e1 = make_double2(x.x - xs.x, x.y - xs.y);
        b1 = e1.x * e1.x + e1.y * e1.y;
        const double ab = e0.x * e1.x + e0.y * e1.y;
        // |cross| with the sign bit cleared on the integer pipe (the FP64
        // pipe is this loop's busiest unit)
        const double cr = e0.x * e1.y - e0.y * e1.x;
        const double ad = __hiloint2double(__double2hiint(cr) & 0x7fffffff, __double2loint(cr));
        if constexpr (F::BILINEAR) {
          double vs;
          RingCell<F>::entries(a0, ab, b1, ad, kappa, vs, vp, vn);
          if constexpr (!kDiagBySum) diag += vs;
        } else {
          acc += RingCell<F>::action(a0, ab, b1, ad, kappa, us, up, un);
          up = un;
        }
      };
      auto emit = [&](int rank, double v) {
        if constexpr (F::BILINEAR) {
          put(rank, v);
          if constexpr (kDiagBySum) diag -= v;
        }
      };
      if (q1 - q0 > 1) {
        double vp = 0.0, vn = 0.0;
        uint32_t r = rec_s[q0 + 1];
        {
          double2 e1;
          double b1;
          cell(ea, aa, wx(r), e1, b1, F::HAS_COEFF ? wc(r) : 0.0, first, carry);
          ea = e1;
          aa = b1;
        }
        rkp = r & 7;
        int q = q0 + 2;
        // two cells per iteration; the second writes the loop-carried edge in
        // place (no register rotation)
        for (; q + 1 < q1; q += 2) {
          const uint32_t r1 = rec_s[q], r2 = rec_s[q + 1];
          const double2 x1 = wx(r1), x2 = wx(r2);
          const double u1 = F::HAS_COEFF ? wc(r1) : 0.0, u2 = F::HAS_COEFF ? wc(r2) : 0.0;
          double2 e1;
          double b1;
          cell(ea, aa, x1, e1, b1, u1, vp, vn);
          emit(rkp, carry + vp);
          carry = vn;
          cell(e1, b1, x2, ea, aa, u2, vp, vn);
          emit(r1 & 7, carry + vp);
          carry = vn;
          rkp = r2 & 7;
        }
        if (q < q1) {
          r = rec_s[q];
          double2 e1;
          double b1;
          cell(ea, aa, wx(r), e1, b1, F::HAS_COEFF ? wc(r) : 0.0, vp, vn);
          emit(rkp, carry + vp);
          carry = vn;
          rkp = r & 7;
        }
        if constexpr (F::BILINEAR) {
          if (rkp == rk0) emit(rk0, first + carry); // closed ring
          else {
            emit(rk0, first);
            emit(rkp, carry);
          }
        }
      }
      if constexpr (F::BILINEAR) put(self_rank, diag);
      else a.out[R0 + tid] = ACC ? a.out[R0 + tid] + acc : acc;
    }
    __syncwarp();
    const long long c1c = a.timing ? clock64() : 0;
    if (lane == 0) mbar_arrive(&empty[k % kRS]);
    if constexpr (F::BILINEAR && kRingStg) {
      // the warp's slice complete -> a coalesced warp-wide copy to its range
      // of the CSR values (plain stores: no async-proxy fence, no TMA store
      // whose shared-memory reads the next tile would have to wait for)
      for (int t = W0 + lane; t < W1; t += 32) a.out[t] = segb[t];
      __syncwarp();
    }
    if constexpr (F::BILINEAR && !kRingStg) {
      // the warp's slice complete -> one bulk store by its lane 0 (head /
      // tail doubles off the 16-byte grid stored directly)
      fence_async_shared();
      __syncwarp();
      if (lane == 0 && W1 > W0) {
        const int nw = W1 - W0, h = W0 & 1, t1 = nw - ((W0 + nw) & 1);
        double* dst = a.out + W0;
        const double* src = segb + W0;
        if (h) dst[0] = src[0];
        if (t1 > h) {
          bulk_s2g(dst + h, src + h, (uint32_t)(t1 - h) * 8);
          bulk_commit();
        }
        if (t1 < nw && t1 >= h) dst[t1] = src[t1];
      }
    }
    if (a.timing) {
      const long long c2 = clock64();
      t_comp += c2 - c1;
      ++t_n;
      if (tid == 0 && tile < 16384) { // per-tile record (warp 0): wait | start barrier, rows, end (16 bits each)
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.timing[16 + 4 * 2048 + 2 * tile] = (unsigned long long)(c1 - c0) | ((unsigned long long)blockIdx.x << 32) |
                                            ((unsigned long long)smid << 48) | ((unsigned long long)(k & 15) << 60);
        a.timing[17 + 4 * 2048 + 2 * tile] = (unsigned long long)(c1b - c1) | ((unsigned long long)(c1c - c1b) << 20) |
                                            ((unsigned long long)(c2 - c1c) << 40);
      }
    }
  }
  // the segment must outlive its bulk store's shared-memory reads; the global
  // writes themselves complete with the grid
  if (F::BILINEAR && (tid & 31) == 0) bulk_wait_read<0>();
  tile_counter_release(a.next_tile, a.reset_tile, kTileThreads, tid);
  if (a.timing && (tid & 31) == 0) {
    atomicAdd(a.timing, (unsigned long long)t_first);
    atomicAdd(a.timing + 1, (unsigned long long)t_wait);
    atomicAdd(a.timing + 2, (unsigned long long)t_comp);
    atomicAdd(a.timing + 3, (unsigned long long)t_n);
    atomicAdd(a.timing + 4, 1ull);
    atomicAdd(a.timing + 5, (unsigned long long)t_early);
    atomicAdd(a.timing + 6, (unsigned long long)t_last);
    atomicAdd(a.timing + 7, (unsigned long long)(clock64() - t_start));
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    atomicMax(a.timing + 9, gt);
  }
  if (a.timing && tid == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    const unsigned long long st = gt - (unsigned long long)((clock64() - t_start) / 2); // ~start (ns, 2 GHz)
    atomicMin(a.timing + 8, st);
    atomicAdd(a.timing + 10, (unsigned long long)(clock64() - t_start));
    atomicMax(a.timing + 11, st);
    atomicMin(a.timing + 12, gt);
    a.timing[16 + 4 * blockIdx.x] = st;
    a.timing[17 + 4 * blockIdx.x] = gt;
    a.timing[18 + 4 * blockIdx.x] = t_n;
    unsigned sm_id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
    a.timing[19 + 4 * blockIdx.x] = sm_id;
  }
}

// PDL for the persistent tile kernels (LOAM_GPU_NO_PDL=1 disables it).
bool pdl_enabled() {
  static const bool on = std::getenv("LOAM_GPU_NO_PDL") == nullptr;
  return on;
}

template <class F>
void launch_ring(const RingArgs& a, size_t smem, cudaStream_t s) {
  if constexpr (F::GD == 2 && F::NRN == 3 && F::RD == 1 && F::CD == 1) {
    if (a.ntiles == 0) return;
    static size_t attr = 0;
    auto kern = a.accumulate ? k_ring<F, true> : k_ring<F, false>;
    if (attr < smem) {
      LG_CUDA(cudaFuncSetAttribute(k_ring<F, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LG_CUDA(cudaFuncSetAttribute(k_ring<F, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kTileBlock, smem));
    const int grid = std::min(a.ntiles, std::max(blocks, 1) * kNumSMs);
    // programmatic dependent launch: the kernel's prologue (barriers, tile
    // records, plan ranges) overlaps the previous kernel's tail; it waits
    // (griddepcontrol.wait) before reading the caller's data or writing
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTileBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr_pdl[1];
    attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr_pdl[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr_pdl;
    cfg.numAttrs = 1;
    LG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    count_launch();
    LG_LAUNCH_CHECK();
  } else {
    fail(LOAM_ERR(InvalidArgument), "ring kernel needs a scalar P1 triangle form");
  }
}

// ---------------------------------------------------------------------------
// Canonical pair-tile kernel (plan.cuh PTilePlan) for every catalogue form:
// P2 tets and triangles, vector P1 elasticity, Taylor-Hood blocks.  The plan
// permuted each cell's local numbering so the owning row is local vertex 0
// (vertex rows) or the first local edge (P2 edge rows): the element row is a
// compile-time index and one thread computes its node row's whole RD x NC
// block once per pair.  TMA producer warp + consumer warps as in k_tile; the
// cell vertices (and coefficients) come from TMA-loaded vertex windows via the
// u16 slots in the pair record; no per-pair global gathers remain.
struct PTileArgs {
  const int32_t* tiles;
  int ntiles;
  int* next_tile;
  int* reset_tile;
  const int32_t* pptr;
  const int32_t* nptr;
  const uint8_t* recs;
  const int32_t* runs;
  const int32_t* cruns;
  const double* coords;
  const double* coeff;
  FormParams prm;
  double* out;
  int accumulate;
  int off_seg, off_buf, buf_bytes;
  int b_pptr, b_nptr, b_recs, b_win, b_winc;
  int cas; // concurrent G-lane adds by shared-memory CAS instead of serialised sub-steps
};

template <class F>
struct PRec { // record layout (plan.cu:build_ptile)
  static constexpr int NV = F::GD + 1;
  static constexpr int NCF = F::HAS_COEFF ? F::NCOEFF : 0;
  static constexpr int OFF_CF = 2 * NV, OFF_RK = OFF_CF + 2 * NCF, OFF_CI = OFF_RK + F::NCN;
  static constexpr int BYTES = (OFF_CI + 1 + 3) & ~3;
};

template <class F, int NT, int kPS>
__global__ void __launch_bounds__(NT + 32, 1) k_ptile(const __grid_constant__ PTileArgs a) {
  constexpr int GD = F::GD, NV = GD + 1, W = F::RD * F::CD;
  using RL = PRec<F>;
  constexpr int RB = RL::BYTES;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + kPS;
  int* slot_tile = reinterpret_cast<int*>(full + 6);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < kPS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) grid_dep_launch(); // PDL: the next kernel's prologue may start
  auto tile_meta = [&](int tile, int (&m)[12]) {
    const int4* t = reinterpret_cast<const int4*>(a.tiles + 12 * tile);
    const int4 x = __ldg(t), y = __ldg(t + 1), z = __ldg(t + 2);
    m[0] = x.x; m[1] = x.y; m[2] = x.z; m[3] = x.w; m[4] = y.x; m[5] = y.y; m[6] = y.z; m[7] = y.w;
    m[8] = z.x; m[9] = z.y; m[10] = z.z; m[11] = z.w;
  };
  auto ring = [&](int k) { return sm + a.off_buf + (k % kPS) * a.buf_bytes; };
  if (tid >= NT) { // ---- producer warp (software-pipelined as in k_ring)
    const int lane = tid & 31;
    auto grab = [&]() {
      int t = 0;
      if (lane == 0) t = atomicAdd(a.next_tile, 1);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    int nt = grab(), nm[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    int2 nrun = make_int2(0, 0), ncrun = make_int2(0, 0);
    auto prefetch = [&]() {
      if (nt < a.ntiles) {
        tile_meta(nt, nm);
        nrun = first_run(reinterpret_cast<const int2*>(a.runs) + nm[6], nm[7], lane);
        if constexpr (F::HAS_COEFF) ncrun = first_run(reinterpret_cast<const int2*>(a.cruns) + nm[8], nm[9], lane);
      }
    };
    prefetch();
    grid_dep_wait(); // the caller's data only after the previous kernel (PDL)
    for (int k = 0;; ++k) {
      const int tile = nt;
      int m[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) m[q] = nm[q];
      const int2 run0 = nrun, crun0 = ncrun;
      if (k >= kPS) mbar_wait_sleep(&empty[k % kPS], (k / kPS - 1) & 1);
      if (tile >= a.ntiles) {
        if (lane == 0) {
          slot_tile[k % kPS] = -1;
          mbar_arrive(&full[k % kPS]);
        }
        break;
      }
      if (lane == 0) slot_tile[k % kPS] = tile;
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % kPS];
      auto rb = [](int64_t lo_b, int64_t hi_b, int64_t& s0) {
        s0 = lo_b & ~int64_t(15);
        return (uint32_t)(((hi_b + 15) & ~int64_t(15)) - s0);
      };
      int64_t g0, g1, g2;
      const uint32_t n0 = rb((int64_t)m[0] * 4, (int64_t)(m[1] + 1) * 4, g0);
      const uint32_t n1 = F::BILINEAR ? rb((int64_t)m[0] * 4, (int64_t)(m[1] + 1) * 4, g1) : (g1 = 0, 0u);
      const uint32_t n2 = rb((int64_t)m[4] * RB, (int64_t)m[5] * RB, g2);
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + m[6], m[7], a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), GD};
      const RunSet rk{reinterpret_cast<const int2*>(a.cruns) + m[8], F::HAS_COEFF ? m[9] : 0, a.coeff,
                      reinterpret_cast<double*>(buf + a.b_winc), 1};
      const uint32_t tx = n0 + n1 + n2 + stage_runs<false>(rc, lane, bar, run0) + stage_runs<false>(rk, lane, bar, crun0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, tx);
        bulk_g2s(buf + a.b_pptr, reinterpret_cast<const unsigned char*>(a.pptr) + g0, n0, bar);
        if (n1) bulk_g2s(buf + a.b_nptr, reinterpret_cast<const unsigned char*>(a.nptr) + g1, n1, bar);
        if (n2) bulk_g2s(buf + a.b_recs, a.recs + g2, n2, bar);
      }
      __syncwarp();
      stage_runs<true>(rc, lane, bar, run0);
      stage_runs<true>(rk, lane, bar, crun0);
      nt = grab();
      prefetch();
    }
    return;
  }
  grid_dep_wait(); // (PDL) before the consumers read or write anything of the caller's
  // ---- consumers: one thread per node row
  double* seg = reinterpret_cast<double*>(sm + a.off_seg);
  for (int k = 0;; ++k) {
    mbar_wait(&full[k % kPS], (k / kPS) & 1);
    const int tile = slot_tile[k % kPS];
    if (tile < 0) break;
    int m[12];
    tile_meta(tile, m);
    const int R0 = m[0], nrows = m[1] - m[0], A0 = m[2], nA = m[3] - m[2], P0 = m[4];
    const int64_t E0 = (int64_t)A0 * W;
    if constexpr (F::BILINEAR) {
      const int len = nA * W;
      if (a.accumulate)
        for (int t = tid; t < len; t += NT) seg[t] = a.out[E0 + t];
      else
        for (int t = tid; t < len; t += NT) seg[t] = 0.0;
      named_bar(1, NT);
    }
    const unsigned char* buf = ring(k);
    const int32_t* pptr_s = reinterpret_cast<const int32_t*>(buf + a.b_pptr) + skew_of(R0, 4);
    const int32_t* nptr_s = reinterpret_cast<const int32_t*>(buf + a.b_nptr) + skew_of(R0, 4);
    const unsigned char* rec0 = buf + a.b_recs + (((int64_t)P0 * RB) & 15);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    const double* winc = reinterpret_cast<const double*>(buf + a.b_winc);
    // G lanes per row (tile field 10): lane `sub` takes pairs sub, sub+G, ...;
    // the group's element rows are added to the row segment in G serialized
    // sub-steps (no shared-memory atomics: f64 ATOMS is a CAS loop)
    const int G = m[10], sub = tid & (G - 1), RPP = NT / G;
    for (int base = 0; base < nrows; base += RPP) {
      const int node = base + tid / G;
      const bool live = node < nrows;
      int a0 = 0, L = 0, p0 = 0, p1 = 0;
      if (live) {
        if constexpr (F::BILINEAR) {
          a0 = nptr_s[node] - A0;
          L = nptr_s[node + 1] - A0 - a0;
        }
        p0 = pptr_s[node] - P0;
        p1 = pptr_s[node + 1] - P0;
      }
      const int iters = __reduce_max_sync(0xffffffffu, (p1 - p0 + G - 1) / G);
      double acc = 0.0;
      for (int it = 0; it < iters; ++it) {
        const int p = p0 + it * G + sub;
        const bool has = p < p1;
        double blk[F::RD * F::NC];
        const unsigned char* rec = rec0 + (int64_t)(has ? p : p0) * RB;
        if (has) {
          double X[NV][GD];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int sl = *reinterpret_cast<const uint16_t*>(rec + 2 * v);
            if constexpr (GD == 2) {
              const double2 c2 = reinterpret_cast<const double2*>(win)[sl];
              X[v][0] = c2.x;
              X[v][1] = c2.y;
            } else {
#pragma unroll
              for (int c = 0; c < GD; ++c) X[v][c] = win[sl * GD + c];
            }
          }
          double C[F::HAS_COEFF ? F::NCOEFF : 1];
          if constexpr (F::HAS_COEFF)
#pragma unroll
            for (int q = 0; q < F::NCOEFF; ++q) C[q] = winc[*reinterpret_cast<const uint16_t*>(rec + RL::OFF_CF + 2 * q)];
          Geom<GD> Gm;
          geometry<GD>(X, Gm);
          const int ci = rec[RL::OFF_CI];
          if constexpr (F::NRN > NV) { // P2 row space: vertex or edge canonical row
            if (ci == 0) F::row(0, Gm, C, a.prm, blk);
            else F::row(NV, Gm, C, a.prm, blk);
          } else {
            F::row(0, Gm, C, a.prm, blk);
          }
          if constexpr (!F::BILINEAR) acc += blk[0];
        }
        if constexpr (F::BILINEAR) {
          if (a.cas) { // the G lanes of a row add concurrently (fp64 CAS in shared memory)
            if (has) {
#pragma unroll
              for (int j = 0; j < F::NCN; ++j) {
                const int rk = rec[RL::OFF_RK + j];
#pragma unroll
                for (int d = 0; d < F::RD; ++d)
#pragma unroll
                  for (int c = 0; c < F::CD; ++c)
                    if (!diag_block<F>::value || d == c)
                      atomicAdd(&seg[a0 * W + d * L * F::CD + rk * F::CD + c], blk[d * F::NC + j * F::CD + c]);
              }
            }
          } else
          for (int st = 0; st < G; ++st) {
            if (has && st == sub) {
              // the column nodes of one pair have distinct ranks: issue every
              // shared load of the element row first, then the stores (a
              // load-add-store chain per entry serialises on shared latency)
              int pos[F::NCN];
#pragma unroll
              for (int j = 0; j < F::NCN; ++j) pos[j] = a0 * W + rec[RL::OFF_RK + j] * F::CD;
#pragma unroll
              for (int d = 0; d < F::RD; ++d) {
                double cur[F::NCN * F::CD];
#pragma unroll
                for (int j = 0; j < F::NCN; ++j)
#pragma unroll
                  for (int c = 0; c < F::CD; ++c)
                    if (!diag_block<F>::value || d == c) cur[j * F::CD + c] = seg[pos[j] + d * L * F::CD + c];
#pragma unroll
                for (int j = 0; j < F::NCN; ++j)
#pragma unroll
                  for (int c = 0; c < F::CD; ++c)
                    if (!diag_block<F>::value || d == c)
                      seg[pos[j] + d * L * F::CD + c] = cur[j * F::CD + c] + blk[d * F::NC + j * F::CD + c];
              }
            }
            if (G > 1) __syncwarp();
          }
        }
      }
      if constexpr (!F::BILINEAR) {
        for (int o = 1; o < G; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (live && sub == 0) a.out[R0 + node] = a.accumulate ? a.out[R0 + node] + acc : acc;
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % kPS]);
    if constexpr (F::BILINEAR) {
      named_bar(1, NT);
      const int len = nA * W;
      for (int t = tid; t < len; t += NT) a.out[E0 + t] = seg[t];
      named_bar(1, NT);
    }
  }
  tile_counter_release(a.next_tile, a.reset_tile, NT, tid);
}

constexpr int kPTileThreads = 128;

// pipeline stages (LOAM_GPU_PT_STAGES, 1..3): fewer stages = less shared
// memory per CTA = more CTAs per SM; the best count depends on the form
// (profiles/r01/strategies_ptile_stages.txt)
inline int ptile_stages(int form) {
  static const int env = std::getenv("LOAM_GPU_PT_STAGES") ? std::atoi(std::getenv("LOAM_GPU_PT_STAGES")) : 0;
  if (env >= 1 && env <= 3) return env;
  return form == F_STOKES_A || form == F_STOKES_B || form == F_STOKES_BT ? 2 : 1;
}

template <class F>
void launch_ptile(const PTileArgs& a, size_t smem_base, size_t buf, cudaStream_t s) {
  if (a.ntiles == 0) return;
  auto go = [&](auto kern, int stages) {
    const size_t smem = smem_base + stages * buf;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kPTileThreads + 32, smem));
    const int grid = std::min(a.ntiles, std::max(blocks, 1) * kNumSMs);
    launch_pdl(kern, dim3(grid), dim3(kPTileThreads + 32), smem, s, a);
  };
  const int st = ptile_stages(F::ID);
  if (st == 1) go(k_ptile<F, kPTileThreads, 1>, 1);
  else if (st == 2) go(k_ptile<F, kPTileThreads, 2>, 2);
  else go(k_ptile<F, kPTileThreads, 3>, 3);
  count_launch();
  LG_LAUNCH_CHECK();
}

// ===========================================================================
// Registry
// ===========================================================================

using GenericFn = void (*)(const GLaunch&, cudaStream_t);
using OwnerFn = void (*)(const OwnerArgs&, int grid, size_t smem, cudaStream_t);
using NbrFn = void (*)(const TileArgs&, int rec_bytes, size_t smem, cudaStream_t);
using RingFn = void (*)(const RingArgs&, size_t smem, cudaStream_t);
using PTileFn = void (*)(const PTileArgs&, size_t smem_base, size_t buf, cudaStream_t);
using CellFn = void (*)(const CellArgs&, bool agg, cudaStream_t);
using CellSegFn = void (*)(const CellSegArgs&, cudaStream_t);
using PatchFn = void (*)(const PatchArgs&, size_t smem, cudaStream_t);
using StarFn = void (*)(const StarArgs&, cudaStream_t);

struct Entry {
  KernelInfo info;
  GenericFn generic = nullptr;
  int stage = 0;
  // catalogue form traits (form < 0: plain staged kernel)
  int form = -1, gd = 0, nrn = 0, ncn = 0, rd = 1, cd = 1, ncoeff = 0;
  bool bilinear = false, has_coeff = false;
  OwnerFn owner = nullptr;
  NbrFn nbr = nullptr;   // P1 forms only
  RingFn ring = nullptr; // scalar P1 triangle forms only
  PTileFn ptile = nullptr;
  CellFn cell = nullptr;
  CellSegFn cell_seg = nullptr; // actions: warp-segmented cell reduction
  PatchFn patch = nullptr; // square Mats and actions whose coordinate map is the row map's vertex prefix
  StarFn star = nullptr;   // P1 triangle actions
};

template <class K>
void launch_generic(const GLaunch& L, cudaStream_t s) {
  if (L.count == 0) return;
  k_generic<K><<<ceil_div(L.count, kTPB), kTPB, 0, s>>>(L);
  count_launch();
  LG_LAUNCH_CHECK();
}

template <class F>
void launch_owner(const OwnerArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (grid == 0) return;
  if constexpr (F::BILINEAR) {
    static bool attr = [] {
      cudaFuncSetAttribute(k_owner_mat<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      return true;
    }();
    (void)attr;
    k_owner_mat<F><<<grid, 128, smem, s>>>(a);
  } else {
    k_owner_vec<F><<<grid, kTPB, 0, s>>>(a);
  }
  count_launch();
  LG_LAUNCH_CHECK();
}

template <class F>
void launch_nbr(const TileArgs& a, int rec_bytes, size_t smem, cudaStream_t s) {
  if (a.ntiles == 0) return;
  auto go = [&](auto kern) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kTileBlock, smem));
    const int per_sm = blocks > 0 ? blocks : 1;
    const int grid = std::min(a.ntiles, per_sm * kNumSMs);
    kern<<<grid, kTileBlock, smem, s>>>(a);
  };
  if constexpr (F::BILINEAR && F::RD == 1 && F::CD == 1) {
    if (a.max_len <= 8 && std::getenv("LOAM_GPU_REG")) { // register-slot accumulator (experimental)
      if (rec_bytes == 1) go(k_tile<F, uint8_t, 8>);
      else if (rec_bytes == 2) go(k_tile<F, uint16_t, 8>);
      else go(k_tile<F, uint32_t, 8>);
      count_launch();
      LG_LAUNCH_CHECK();
      return;
    }
  }
  if (rec_bytes == 1) go(k_tile<F, uint8_t, 0>);
  else if (rec_bytes == 2) go(k_tile<F, uint16_t, 0>);
  else go(k_tile<F, uint32_t, 0>);
  count_launch();
  LG_LAUNCH_CHECK();
}

constexpr int kPatchThreads = 256;

template <class F>
void launch_patch(const PatchArgs& a, size_t smem, cudaStream_t s) {
  if (a.npatches == 0) return;
  auto go = [&](auto kern) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kPatchThreads, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "patch kernel does not fit on an SM");
    static const bool one_per_cta = std::getenv("LOAM_GPU_PATCH_GRID") != nullptr;
    const int grid = one_per_cta ? a.npatches : std::min(a.npatches, blocks * kNumSMs);
    kern<<<grid, kPatchThreads, smem, s>>>(a);
  };
  if constexpr (F::BILINEAR) {
    if constexpr (F::NRN == F::NCN) go(k_patch_mat<F, kPatchThreads>);
  } else {
    go(k_patch_vec<F, kPatchThreads>);
  }
  count_launch();
  LG_LAUNCH_CHECK();
}

template <class K>
Entry plain_entry(const char* name, std::vector<std::string> names, std::vector<std::vector<int>> ext) {
  Entry e;
  e.info = KernelInfo{name, std::move(names), std::move(ext)};
  e.generic = &launch_generic<K>;
  e.stage = K::STAGE;
  return e;
}

template <int FORM, int D, int P>
Entry form_entry(const std::string& name) {
  using F = FormT<FORM, D, P>;
  Entry e;
  e.info.name = name;
  e.info.param_names = {"A", "X"};
  if (F::BILINEAR) e.info.extents = {{F::NR, F::NC}, {D + 1, D}};
  else e.info.extents = {{F::NR}, {D + 1, D}};
  if (F::HAS_COEFF) {
    e.info.param_names.push_back("C");
    e.info.extents.push_back({F::NCOEFF});
  }
  e.generic = &launch_generic<FormKernel<F>>;
  e.stage = FormKernel<F>::STAGE;
  e.form = FORM;
  e.gd = D;
  e.nrn = F::NRN;
  e.ncn = F::NCN;
  e.rd = F::RD;
  e.cd = F::CD;
  e.ncoeff = F::NCOEFF;
  e.bilinear = F::BILINEAR;
  e.has_coeff = F::HAS_COEFF;
  e.owner = &launch_owner<F>;
  e.ptile = &launch_ptile<F>;
  e.cell = &launch_cell<F>;
  if constexpr (!F::BILINEAR) e.cell_seg = &launch_cell_seg<F>;
  if constexpr (!F::BILINEAR ? F::NCOEFF == F::NRN : F::NRN == F::NCN) e.patch = &launch_patch<F>;
  if constexpr (P == 1 && F::NRN == D + 1 && (!F::BILINEAR || F::NCN == F::NRN)) e.nbr = &launch_nbr<F>;
  if constexpr (P == 1 && D == 2 && F::RD == 1 && F::CD == 1) e.ring = &launch_ring<F>;
  if constexpr (P == 1 && D == 2 && F::RD == 1 && F::CD == 1) e.star = &launch_star<F>;
  return e;
}

template <int D, int P>
void add_scalar_forms(std::map<std::string, Entry>& r) {
  const std::string sfx = std::string("_p") + std::to_string(P) + (D == 2 ? "_tri" : "_tet");
  // names as compile_cell_kernel builds them (form.hpp:214-222)
  r["mass" + sfx] = form_entry<F_MASS, D, P>("mass" + sfx);
  r["stiffness" + sfx] = form_entry<F_STIFFNESS, D, P>("stiffness" + sfx);
  r["helmholtz" + sfx] = form_entry<F_HELMHOLTZ, D, P>("helmholtz" + sfx);
  r["mass_action" + sfx] = form_entry<F_MASS_ACTION, D, P>("mass_action" + sfx);
  r["source" + sfx] = form_entry<F_MASS_ACTION, D, P>("source" + sfx); // interpolated density
  r["stiffness_action" + sfx] = form_entry<F_STIFFNESS_ACTION, D, P>("stiffness_action" + sfx);
  r["helmholtz_action" + sfx] = form_entry<F_HELMHOLTZ_ACTION, D, P>("helmholtz_action" + sfx);
}

const std::map<std::string, Entry>& registry() {
  static const std::map<std::string, Entry> r = [] {
    std::map<std::string, Entry> m;
    add_scalar_forms<2, 1>(m);
    add_scalar_forms<2, 2>(m);
    add_scalar_forms<3, 1>(m);
    add_scalar_forms<3, 2>(m);
    m["elasticity_p1_tet"] = form_entry<F_ELASTICITY, 3, 1>("elasticity_p1_tet");
    m["stokes_a_p2_tri"] = form_entry<F_STOKES_A, 2, 2>("stokes_a_p2_tri");
    m["stokes_b_p2_tri"] = form_entry<F_STOKES_B, 2, 2>("stokes_b_p2_tri");
    m["stokes_bt_p2_tri"] = form_entry<F_STOKES_BT, 2, 2>("stokes_bt_p2_tri");
    return m;
  }();
  return r;
}

// The kernels the reference's own test suite builds (test_parloop.cpp,
// test_data.cpp: add_one, ones_block, ...): a separate registry, visible only
// when LOAM_OPT_TEST_KERNELS is set (the parity tests), not product kernels.
const std::map<std::string, Entry>& test_registry() {
  static const std::map<std::string, Entry> r = [] {
    std::map<std::string, Entry> m;
    using namespace testk;
    m["double_direct"] = plain_entry<DoubleDirect>("double_direct", {"A", "B"}, {{1}, {1}});
    m["add_one"] = plain_entry<AddOne>("add_one", {"V"}, {{3}});
    m["ones_block"] = plain_entry<OnesBlock>("ones_block", {"A"}, {{3, 3}});
    m["weighted_scatter"] = plain_entry<WeightedScatter>("weighted_scatter", {"V", "X"}, {{3}, {1}});
    m["bump"] = plain_entry<Bump>("bump", {"V"}, {{3}});
    m["fill"] = plain_entry<Fill>("fill", {"V"}, {{2}});
    m["sum"] = plain_entry<Sum>("sum", {"G", "X"}, {{1}, {1}});
    m["maxval"] = plain_entry<MaxVal>("maxval", {"G", "X"}, {{1}, {1}});
    m["sumcells"] = plain_entry<SumCells>("sumcells", {"G", "X"}, {{1}, {1}});
    m["dw"] = plain_entry<Dw>("dw", {"A", "B"}, {{1}, {1}});
    m["drw"] = plain_entry<Drw>("drw", {"A", "B"}, {{1}, {1}});
    m["dinc"] = plain_entry<Dinc>("dinc", {"A", "B"}, {{1}, {1}});
    m["gw"] = plain_entry<Gw>("gw", {"A", "V"}, {{1}, {3}});
    m["iinc"] = plain_entry<WeightedScatter>("iinc", {"V", "C"}, {{3}, {1}});
    m["iincv"] = plain_entry<Iincv>("iincv", {"V", "C"}, {{3, 2}, {1}});
    m["gsum"] = plain_entry<Gsum>("gsum", {"G", "B", "S"}, {{1}, {1}, {1}});
    m["gmm"] = plain_entry<Gmm>("gmm", {"LO", "HI", "B"}, {{1}, {1}, {1}});
    return m;
  }();
  return r;
}

const Entry* find_entry(const std::string& name) {
  auto it = registry().find(name);
  if (it != registry().end()) return &it->second;
  if (options().test_kernels) {
    auto jt = test_registry().find(name);
    if (jt != test_registry().end()) return &jt->second;
  }
  return nullptr;
}

const Entry& lookup(const char* name) {
  require(name != nullptr, LOAM_ERR(InvalidArgument), "parloop without kernel");
  const Entry* e = find_entry(name);
  require(e != nullptr, LOAM_ERR(InvalidArgument),
          std::string("kernel ") + name + " has no device implementation (no CPU fallback)");
  return *e;
}

// ===========================================================================
// Validation (parloop.hpp:89-146)
// ===========================================================================

const char* access_name(int a) {
  static const char* n[] = {"READ", "WRITE", "RW", "INC", "SUM", "MIN", "MAX"};
  return a >= 0 && a < 7 ? n[a] : "?";
}

bool same_id(uint64_t a, uint64_t b) { return a == 0 || b == 0 || a == b; }
bool writes(int access) { return access != LOAM_READ; }

std::vector<int> staged_extents(const loam_arg_desc& a) { // parloop.hpp:63-70
  if (a.kind == LOAM_ARG_GLOBAL) return {a.dim};
  if (a.kind == LOAM_ARG_MAT) return {a.map->arity, a.col_map->arity};
  if (!a.map) return {a.dim};
  if (a.dim == 1) return {a.map->arity};
  return {a.map->arity, a.dim};
}

void validate_args(const Entry& k, int n, uint64_t iter, const loam_arg_desc* args, int nargs) {
  require(n >= 0, LOAM_ERR(InvalidArgument), "iteration set size must be non-negative");
  require(nargs >= 0 && nargs <= kMaxArgs, LOAM_ERR(InvalidArgument), "too many arguments");
  for (int q = 0; q < nargs; ++q) {
    const loam_arg_desc& a = args[q];
    require(a.kind >= 0 && a.kind <= 2, LOAM_ERR(InvalidArgument), "argument must target exactly one object");
    if (a.kind == LOAM_ARG_DAT) {
      require(a.access == LOAM_READ || a.access == LOAM_WRITE || a.access == LOAM_RW || a.access == LOAM_INC,
              LOAM_ERR(IllegalAccess), std::string("access ") + access_name(a.access) + " not legal for Dats");
      require(a.col_map == nullptr, LOAM_ERR(InvalidArgument), "Dat argument with several maps");
      require(a.dim > 0, LOAM_ERR(InvalidArgument), "Dat dim must be positive");
      if (!a.map) {
        require(a.set_size == n && same_id(a.set_id, iter), LOAM_ERR(MapSourceMismatch),
                "direct argument not defined on the iteration set");
      } else {
        require(a.map->source_size == n && same_id(a.map->source_id, iter), LOAM_ERR(MapSourceMismatch),
                "map source differs from iteration set");
        require(a.map->target_size == a.set_size && same_id(a.map->target_id, a.set_id),
                LOAM_ERR(MapSourceMismatch), "map target differs from set of dat");
      }
    } else if (a.kind == LOAM_ARG_MAT) {
      require(a.access == LOAM_WRITE || a.access == LOAM_INC, LOAM_ERR(IllegalAccess),
              "Mats are write-only: only WRITE and INC are permitted");
      require(a.map && a.col_map && a.sparsity, LOAM_ERR(InvalidArgument),
              "Mat argument requires row and column maps");
      require(a.map->source_size == n && same_id(a.map->source_id, iter) && a.col_map->source_size == n &&
                  same_id(a.col_map->source_id, iter),
              LOAM_ERR(MapSourceMismatch), "map source differs from iteration set");
      require(a.map->target_size == a.sparsity->nrows && a.col_map->target_size == a.sparsity->ncols,
              LOAM_ERR(ShapeMismatch), "matrix shape does not match its maps");
    } else {
      require(a.access == LOAM_READ || a.access == LOAM_SUM || a.access == LOAM_MIN || a.access == LOAM_MAX,
              LOAM_ERR(IllegalAccess), std::string("access ") + access_name(a.access) + " not legal for Globals");
      require(!a.map && !a.col_map, LOAM_ERR(InvalidArgument), "Global argument cannot carry a map");
      require(a.dim > 0, LOAM_ERR(InvalidArgument), "Global dim must be positive");
    }
  }
  for (int i = 0; i < nargs; ++i) // written-alias rejection (parloop.hpp:131-137)
    for (int j = i + 1; j < nargs; ++j) {
      const bool same = (args[i].obj_id && args[i].obj_id == args[j].obj_id) ||
                        (!args[i].obj_id && args[i].data && args[i].data == args[j].data);
      if (same)
        require(!writes(args[i].access) && !writes(args[j].access), LOAM_ERR(IllegalAccess),
                "aliased argument is written by this parloop");
    }
  const auto& ext = k.info.extents;
  require((int)ext.size() == nargs, LOAM_ERR(ShapeMismatch),
          "kernel parameter count does not match argument count");
  for (int q = 0; q < nargs; ++q)
    require(ext[q] == staged_extents(args[q]), LOAM_ERR(ShapeMismatch),
            "staged shape of argument " + std::to_string(q) + " does not match kernel parameter " +
                k.info.param_names[q]);
}

// ===========================================================================
// Plans and their cache (the reference caches colourings, parloop.hpp:153-168)
// ===========================================================================

struct NodeMap { // node-level view of a map (undoing a declared dof expansion)
  MapView v;
  int dim = 1;
  uint64_t id = 0;
};

NodeMap node_view(const loam_map_desc* m) {
  NodeMap r;
  r.id = m->id;
  if (m->expand_dim > 1 && m->node_values) {
    r.v = MapView{m->node_values, m->source_size, m->node_arity, m->node_target_size};
    r.dim = m->expand_dim;
    r.id = m->node_id; // the node map's identity (0 = unknown)
  } else {
    r.v = MapView{m->values, m->source_size, m->arity, m->target_size};
  }
  return r;
}

// A Mat argument whose (row, col) maps are, at node level, the maps its
// sparsity was built from (loam_sparsity_desc provenance) has exactly that
// pattern: every entry is reached by some cell of the loop.
bool pattern_provenance_exact(const loam_arg_desc& a) {
  if (a.kind != LOAM_ARG_MAT || !a.sparsity || !a.map || !a.col_map) return false;
  const loam_sparsity_desc* sp = a.sparsity;
  if (!sp->pattern_row_map || !sp->pattern_col_map) return false;
  const NodeMap R = node_view(a.map), C = node_view(a.col_map);
  return R.id == sp->pattern_row_map && C.id == sp->pattern_col_map && R.dim == sp->pattern_row_dim &&
         C.dim == sp->pattern_col_dim;
}

// Tile counters of the persistent tile kernels, one pair per launch in
// flight.  A kernel takes tiles from counter [0] and the last CTA puts [0] and
// the exit count [1] back to zero (stage.cuh:tile_counter_release), so a pair
// may be reused by the next launch that is ORDERED after it: a launch on the
// same stream, or any launch once the recorded event of the previous user has
// completed.  Two launches of one cached plan that may overlap (two streams, a
// graph replay beside a direct execute) therefore never share a pair.  A launch
// captured into a CUDA graph keeps its pair for good (its pointer is frozen in
// the graph; replays of one graph are ordered among themselves).
struct TileCounters {
  static constexpr int kSlots = 32;
  struct Slot {
    cudaEvent_t done = nullptr;
    cudaStream_t stream = nullptr;
    int state = 0; // 0 unused, 1 direct launches, 2 owned by a captured graph
  };
  DevBuf<int> mem;
  Slot slot[kSlots];
  std::mutex mu;

  void init(cudaStream_t s) {
    mem.alloc(2 * kSlots, s);
    LG_CUDA(cudaMemsetAsync(mem.get(), 0, mem.bytes(), s));
  }
  ~TileCounters() {
    for (Slot& q : slot)
      if (q.done) cudaEventDestroy(q.done);
  }
  // index of a pair this launch may use on stream s
  int acquire(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LG_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
      for (int i = 0; i < kSlots; ++i)
        if (slot[i].state == 0) {
          slot[i].state = 2;
          return i;
        }
      fail(LOAM_ERR(InvalidArgument), "more than 32 CUDA-graph captures of one par_loop plan");
    }
    for (int i = 0; i < kSlots; ++i) {
      Slot& q = slot[i];
      if (q.state == 0 || (q.state == 1 && (q.stream == s || cudaEventQuery(q.done) == cudaSuccess))) return i;
    }
    // every pair is in flight on other streams: order after the first one
    for (int i = 0; i < kSlots; ++i)
      if (slot[i].state == 1) {
        LG_CUDA(cudaStreamWaitEvent(s, slot[i].done, 0));
        return i;
      }
    fail(LOAM_ERR(InvalidArgument), "no tile counter available");
    return -1;
  }
  // after the launch that used pair i (no-op for captured pairs)
  void commit(int i, cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    Slot& q = slot[i];
    if (q.state == 2) return;
    if (!q.done) LG_CUDA(cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming));
    LG_CUDA(cudaEventRecord(q.done, s));
    q.stream = s;
    q.state = 1;
  }
  int* next(int i) const { return mem.get() + 2 * i; }
  int* exits(int i) const { return mem.get() + 2 * i + 1; }
};

__global__ void k_mark_nodes(const int32_t* __restrict__ m, int64_t len, uint8_t* __restrict__ mark) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    mark[m[i]] = 1;
}
__global__ void k_count_unmarked(const uint8_t* __restrict__ mark, int n, int* __restrict__ cnt) {
  int c = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) c += mark[i] == 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// Does every target node appear in the map?  (A Dat INC through it then
// reaches every entry of the Dat.)
bool map_covers_target(const MapView& m, cudaStream_t s) {
  if (m.target == 0) return true;
  DevBuf<uint8_t> mark((size_t)m.target, s);
  DevBuf<int> cnt(1, s);
  LG_CUDA(cudaMemsetAsync(mark.get(), 0, (size_t)m.target, s));
  LG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int), s));
  const int64_t len = (int64_t)m.n * m.arity;
  if (len) k_mark_nodes<<<kNumSMs * 4, 256, 0, s>>>(m.v, len, mark.get());
  k_count_unmarked<<<kNumSMs * 4, 256, 0, s>>>(mark.get(), m.target, cnt.get());
  count_launch(len ? 2 : 1);
  LG_LAUNCH_CHECK();
  int h = 0;
  LG_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

// The scatter strategy in effect: deterministic mode runs the auto paths only
// (their RED-based pieces switch to fixed-order variants).
int strategy() { return options().deterministic ? 0 : options().inc_strategy; }

struct FastPlan {
  TileCounters counter; // dynamic tile scheduler of the persistent tile kernels
  bool exact = false;   // the loop's (row, col) pattern IS the Mat's pattern (provenance / checked)

  bool use_nbr = false;
  NbrPlan nb;
  bool use_ptile = false;
  PTilePlan pt;
  bool use_etile = false;  // edge tiles (scalar P2 matrices, etile.cuh)
  EtilePlan et;
  bool use_wtile = false;  // link-walk tiles (scalar P2 tetrahedra on manifold meshes, wtile.cuh)
  WtilePlan wt;
  bool use_ntile = false;  // node-block tiles (vector P1 elasticity, ntile.cuh)
  NtilePlan nt;
  bool use_ltile = false;  // edge-link tiles (the same loops on manifold meshes, ltile.cuh)
  LtilePlan lt;
  bool use_rtile = false;  // row tiles with shared cell geometry (Taylor-Hood B / B^T, rtile.cuh)
  RtilePlan rt;
  bool use_star = false;   // vertex-star kernel (P1 triangle actions)
  DevBuf<int4> star;
  bool use_patch = false;  // cell-patch row-owner kernels (patch.cuh)
  PatchPlan patch;
  bool use_cell = false;   // cell-centric atomic scatter
  bool det_cell = false;   // deterministic mode: cell entries + fixed-order pair sums
  bool use_ctile = false;  // P2 actions: cell tiles (ctile.cu)
  CtilePlan ct;
  bool use_cseg = false;   // (actions, auto) warp-segmented reduction of the cell scatter
  DevBuf<uint16_t> cs_slots, cs_start;
  DevBuf<int32_t> cs_off, cs_node;
  int cs_nbatches = 0;
  SortedMap crows;         // (cell mode) sorted row map
  DevBuf<uint8_t> cranks;  // (cell mode, matrices) per-cell in-row ranks
  LocalityPlan loc;
  SortedMap xmap, cmap;
  const int32_t* xptr = nullptr;
  const int32_t* cptr = nullptr;
  int xstride = 0, cstride = 0;
  PairPlan pp;
};

struct ColorCacheEntry {
  ColorPlan cp;
};

std::mutex g_cache_mutex;
std::map<std::vector<uint64_t>, std::shared_ptr<FastPlan>> g_fast_cache;
std::map<std::vector<uint64_t>, std::shared_ptr<ColorCacheEntry>> g_color_cache;

__global__ void k_prefix_equal(const int32_t* __restrict__ a, int sa, const int32_t* __restrict__ b,
                               int sb, int ncols, int n, int* bad) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  for (int c = 0; c < ncols; ++c)
    if (a[(int64_t)e * sa + c] != b[(int64_t)e * sb + c]) { *bad = 1; return; }
}

bool prefix_equal(const int32_t* a, int sa, const int32_t* b, int sb, int ncols, int n, cudaStream_t s) {
  if (n == 0) return true;
  DevBuf<int> bad(1, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  k_prefix_equal<<<ceil_div(n, kTPB), kTPB, 0, s>>>(a, sa, b, sb, ncols, n, bad.get());
  count_launch();
  LG_LAUNCH_CHECK();
  int h = 0;
  LG_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

constexpr int kSegMax = 2048;  // doubles of shared memory per warp (16 KB), pair-list kernels
constexpr int kTileSeg = 4096;   // matrix values per neighbour-list tile (32 KB)
constexpr int kTileSlots = 1024; // vertices in a tile's window
constexpr int kTileRuns = 32;    // contiguous runs per window

// Strategy 6 selects the patch kernels; auto uses them for the forms they
// win on (profiles/r01/strategies_patch*).
bool patch_wanted(const Entry& k) {
  const int strat = strategy();
  if (strat == 6) return true;
  if (strat != 0 || std::getenv("LOAM_GPU_NO_PATCH")) return false;
  return std::getenv("LOAM_GPU_PATCH_AUTO") != nullptr && (k.nrn > k.gd + 1 || k.rd > 1);
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

size_t patch_smem_bytes(const Entry& k, const PatchPlan& pp) {
  if (!k.bilinear) {
    int ow, orc, op, of, ox;
    return (size_t)patch_vec_smem(pp.max_win, pp.max_cells, k.nrn, k.gd, &ow, &orc, &op, &of, &ox);
  }
  const int gs = k.gd * k.gd + 1; // (Dats size their element vectors from nrn)
  return (size_t)patch_smem(gs, k.nrn, k.bilinear, pp.max_win, pp.max_cells, pp.max_own, pp.max_pairs,
                            (int)pp.max_seg, (pp.max_win + 31) / 32).total;
}

// Cell-patch plan (patch.cuh) when the loop has the shape the patch kernels
// serve: the coordinate map is the row map's vertex prefix, actions read their
// coefficient through the row map, Mats are square with exactly the (map, map)
// pattern (the in-kernel ranks are derived from the maps, not read from
// col_idx).  Returns false (caller uses another plan) otherwise.
bool try_build_patch(const Entry& k, int n, const loam_arg_desc* args, FastPlan& P, cudaStream_t s) {
  if (!k.patch) return false;
  const NodeMap R = node_view(args[0].map);
  if ((reinterpret_cast<uintptr_t>(args[1].data) & 15) != 0) return false;
  auto same_as_rows = [&](const MapView& m) {
    return m.arity == R.v.arity && m.target == R.v.target &&
           (m.v == R.v.v || prefix_equal(m.v, m.arity, R.v.v, R.v.arity, m.arity, n, s));
  };
  const loam_sparsity_desc* sp = nullptr;
  if (k.has_coeff) {
    const loam_map_desc* Cm = args[2].map;
    if (!same_as_rows(MapView{Cm->values, n, Cm->arity, Cm->target_size})) return false;
  }
  if (k.bilinear) {
    const NodeMap Cn = node_view(args[0].col_map);
    if (Cn.dim != k.cd || R.dim != k.rd || !same_as_rows(Cn.v)) return false;
    sp = args[0].sparsity;
    if (!P.exact &&
        !pattern_is_map_pattern(R.v.v, n, R.v.arity, R.v.target, R.dim, Cn.dim, sp->row_ptr, sp->col_idx, sp->nnz, s))
      return false;
    P.exact = true;
  }
  PatchSpec spec;
  spec.gd = k.gd;
  spec.nrn = k.nrn;
  spec.rd = k.rd;
  spec.cd = k.cd;
  spec.bilinear = k.bilinear;
  spec.budget = env_int("LOAM_GPU_PATCH_BUDGET", 3072);
  spec.max_cells = env_int("LOAM_GPU_PATCH_CELLS", k.bilinear ? 1024 : 512);
  spec.halo = k.bilinear; // Dats: cell-owned patches, shared nodes by fp64 RED
  const loam_map_desc* X = args[1].map;
  for (int attempt = 0; attempt < 6; ++attempt) {
    if (!build_patch(P.patch, spec, n, R.v.target, R.v.v, X->values, X->arity, args[1].data,
                     sp ? sp->row_ptr : nullptr, s))
      return false;
    if (patch_smem_bytes(k, P.patch) <= 200 * 1024) return true;
    spec.budget = spec.budget * 2 / 3;
    spec.max_cells = spec.max_cells * 2 / 3;
  }
  return false;
}

// Warp batches of 32 consecutive (locality-ordered) cells: each batch's
// 32 x arity contributions sorted by row node (then lane, entry), the slot of
// every contribution, and the runs of equal nodes.
void build_cell_segments(const int32_t* sorted_rows, int n, int arity, FastPlan& P, cudaStream_t s) {
  std::vector<int32_t> rows((size_t)n * arity);
  LG_CUDA(cudaMemcpyAsync(rows.data(), sorted_rows, sizeof(int32_t) * rows.size(), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  const int nb = ceil_div(n, 32);
  std::vector<uint16_t> slots((size_t)nb * arity * 32, 0), start;
  std::vector<int32_t> off(nb + 1, 0), node;
  std::vector<std::pair<int32_t, int>> c; // (node, lane * arity + i)
  for (int b = 0; b < nb; ++b) {
    c.clear();
    for (int l = 0; l < 32 && b * 32 + l < n; ++l)
      for (int i = 0; i < arity; ++i) c.emplace_back(rows[((size_t)b * 32 + l) * arity + i], l * arity + i);
    std::sort(c.begin(), c.end());
    off[b] = (int32_t)node.size();
    for (size_t q = 0; q < c.size(); ++q) {
      const int l = c[q].second / arity, i = c[q].second % arity;
      slots[((size_t)b * arity + i) * 32 + l] = (uint16_t)q;
      if (q == 0 || c[q].first != c[q - 1].first) {
        node.push_back(c[q].first);
        start.push_back((uint16_t)q);
      }
    }
    start.push_back((uint16_t)c.size()); // closing start of the batch (nseg + 1 per batch)
  }
  off[nb] = (int32_t)node.size();
  P.cs_nbatches = nb;
  P.cs_slots.alloc(slots.size() + 1, s);
  P.cs_start.alloc(start.size() + 1, s);
  P.cs_off.alloc(off.size(), s);
  P.cs_node.alloc(node.size() + 1, s);
  LG_CUDA(cudaMemcpyAsync(P.cs_slots.get(), slots.data(), 2 * slots.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(P.cs_start.get(), start.data(), 2 * start.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(P.cs_off.get(), off.data(), 4 * off.size(), cudaMemcpyHostToDevice, s));
  if (!node.empty())
    LG_CUDA(cudaMemcpyAsync(P.cs_node.get(), node.data(), 4 * node.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  P.use_cseg = true;
}

std::shared_ptr<FastPlan> build_fast_plan(const Entry& k, int n, const loam_arg_desc* args, bool cell_mode,
                                          cudaStream_t s) {
  plan_tick("plan start", s);
  auto P = std::make_shared<FastPlan>();
  P->counter.init(s);
  P->exact = k.bilinear ? pattern_provenance_exact(args[0]) : map_covers_target(node_view(args[0].map).v, s);
  if (!cell_mode && patch_wanted(k) && try_build_patch(k, n, args, *P, s)) {
    P->use_patch = true;
    return P;
  }
  const NodeMap R = node_view(args[0].map);
  const loam_map_desc* X = args[1].map;
  const loam_map_desc* Cm = k.has_coeff ? args[2].map : nullptr;
  // locality order of the cells, by their smallest row node
  if (options().locality) {
    build_locality(R.v, P->loc, s);
  } else {
    P->loc.n = n;
    P->loc.perm.alloc(n, s);
    std::vector<int32_t> id(n);
    for (int e = 0; e < n; ++e) id[e] = e;
    LG_CUDA(cudaMemcpyAsync(P->loc.perm.get(), id.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    LG_CUDA(cudaStreamSynchronize(s));
  }
  plan_tick("locality order", s);
  const int32_t* perm = P->loc.perm.get();
  SortedMap srows;
  gather_rows(R.v, perm, srows, s);
  plan_tick("gather rows", s);
  if (cell_mode) { // sorted row / coordinate / coefficient maps (+ per-cell slot ranks)
    P->use_cell = true;
    if (k.bilinear) {
      const NodeMap Cn = node_view(args[0].col_map);
      SortedMap scols;
      const int32_t* sc = srows.v.get();
      if (!(Cn.v.v == R.v.v && Cn.v.arity == R.v.arity)) {
        gather_rows(Cn.v, perm, scols, s);
        sc = scols.v.get();
      }
      const loam_sparsity_desc* sp = args[0].sparsity;
      CsrView csr{sp->row_ptr, sp->col_idx, sp->nrows, sp->ncols, sp->nnz, R.dim, Cn.dim};
      PairPlan pp;
      build_pairs(srows.v.get(), n, R.v.arity, R.v.target, pp, s);
      build_ranks(pp, srows.v.get(), sc, Cn.v.arity, csr, s); // OutsideSparsity / ShapeMismatch here
      cell_major_ranks(pp, P->cranks, s);
    }
    // deterministic mode: the rows' (cell, local row) pair lists for the
    // fixed-order second pass (k_pair_sum)
    if (!k.bilinear && options().deterministic && R.dim == 1) {
      build_pairs(srows.v.get(), n, R.v.arity, R.v.target, P->pp, s);
      P->det_cell = true;
    }
    // (measured slower than one RED per entry on config 3, 0.128 vs 0.081 ms: the
    // plain kernel is bound by its dependent gathers, not by the L2 atomics)
    if (!k.bilinear && k.cell_seg && strategy() == 0 && !options().deterministic && std::getenv("LOAM_GPU_CSEG"))
      build_cell_segments(srows.v.get(), n, R.v.arity, *P, s);
    P->crows = std::move(srows);
    gather_rows(MapView{X->values, n, X->arity, X->target_size}, perm, P->xmap, s);
    P->xptr = P->xmap.v.get();
    P->xstride = X->arity;
    if (Cm) {
      if (Cm->values == R.v.v && Cm->arity == R.v.arity) {
        P->cptr = P->crows.v.get();
      } else {
        gather_rows(MapView{Cm->values, n, Cm->arity, Cm->target_size}, perm, P->cmap, s);
        P->cptr = P->cmap.v.get();
      }
      P->cstride = Cm->arity;
      // vertex ids = the coefficient map's first gdim+1 entries (P2 vertices
      // first): one sorted map serves rows, coefficients and coordinates
      if (P->cptr == P->crows.v.get() && prefix_equal(Cm->values, Cm->arity, X->values, X->arity, X->arity, n, s)) {
        P->xptr = P->cptr;
        P->xstride = P->cstride;
        P->xmap.v.release();
      }
    }
    // P2 actions on one sorted map (rows = coefficients, vertex prefix =
    // coordinates): cell tiles with TMA-staged windows and one RED per
    // distinct node of a tile instead of one per element entry.  Opt-in
    // (LOAM_GPU_CTILE=1): measured slower than the cell kernel on config 3
    // (83 vs 68 us per step; DESIGN 15) -- the cell kernel's gathers hit L2.
    const bool action = k.form == F_MASS_ACTION || k.form == F_STIFFNESS_ACTION || k.form == F_HELMHOLTZ_ACTION;
    if (!k.bilinear && action && !P->det_cell && R.dim == 1 && k.nrn == (k.gd == 3 ? 10 : 6) && Cm &&
        P->xptr == P->crows.v.get() && P->cptr == P->crows.v.get() && std::getenv("LOAM_GPU_CTILE") &&
        (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0 && (reinterpret_cast<uintptr_t>(args[2].data) & 15) == 0 &&
        build_ctile(P->ct, k.gd, k.nrn, n, P->crows.v.get(), R.v.target, X->target_size, s))
      P->use_ctile = true;
    return P;
  }
  // Neighbour-list plan when row, column, coordinate (and coefficient) maps
  // are one node map (P1 forms): no per-pair cell ids or map rows at all.
  const int strat = strategy();
  if (k.nbr && (strat == 0 || strat == 4)) {
    auto same = [&](const MapView& m) {
      return m.arity == R.v.arity && (m.v == R.v.v || prefix_equal(m.v, m.arity, R.v.v, R.v.arity, m.arity, n, s));
    };
    // (3D vector rows -- elasticity -- are still faster on the pair-list kernel)
    bool ok = (R.dim == 1 || k.bilinear) && (R.dim == 1 || strat == 4);
    ok = ok && same(MapView{X->values, n, X->arity, X->target_size}) && X->target_size == R.v.target;
    if (Cm) ok = ok && same(MapView{Cm->values, n, Cm->arity, Cm->target_size});
    CsrView csr{};
    if (k.bilinear) {
      const NodeMap Cn = node_view(args[0].col_map);
      ok = ok && same(Cn.v) && Cn.v.target == R.v.target;
      const loam_sparsity_desc* sp = args[0].sparsity;
      csr = CsrView{sp->row_ptr, sp->col_idx, sp->nrows, sp->ncols, sp->nnz, R.dim, Cn.dim};
      if (ok && (R.dim > 1 || Cn.dim > 1)) { // blockedness of the pattern
        DevBuf<int> dummy;
        PairPlan probe;
        probe.nrows_node = R.v.target;
        probe.npairs = 0;
        build_ranks(probe, srows.v.get(), srows.v.get(), 0, csr, s); // throws ShapeMismatch if not blocked
      }
    }
    // the window TMA needs 16-byte aligned coordinate / coefficient arrays
    ok = ok && (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0 &&
         (!Cm || (reinterpret_cast<uintptr_t>(args[2].data) & 15) == 0);
    // Mats: the star kernel writes the (map, map) pattern's rows, so the Mat's
    // pattern must be exactly that one (not a superset)
    const bool star_ok = ok && k.star && strat == 0 && !std::getenv("LOAM_GPU_NO_STAR") &&
                         (!k.bilinear || std::getenv("LOAM_GPU_STAR_MAT")) &&
                         (!k.bilinear || P->exact ||
                          pattern_is_map_pattern(R.v.v, n, R.v.arity, R.v.target, 1, 1, csr.row_ptr, csr.col_idx,
                                                 csr.nnz, s));
    plan_tick("nbr checks", s);
    if (star_ok && (std::getenv("LOAM_GPU_HOST_RING") ? build_stars(R.v.v, n, R.v.target, P->star, s)
                                                       : build_stars_dev(R.v.v, n, R.v.target, P->star, s))) {
      plan_tick("stars", s);
      if (k.bilinear) P->exact = true;
      P->use_star = true;
      return P;
    }
    // tile rows: at most one per consumer thread; for the ring kernel's static
    // schedule (3 CTAs per SM) the row count is evened out so every CTA gets
    // the same number of tiles (no tail of CTAs with one tile more)
    int tile_rows = kTileThreads / R.dim;
    if (k.ring && R.dim == 1 && k.bilinear) {
      const int G = kRingMinBlocks * kNumSMs;
      const int per_cta = ceil_div(ceil_div(R.v.target, tile_rows), G);
      tile_rows = std::max(32, ceil_div(R.v.target, (int64_t)per_cta * G));
    }
    // the ring plan on the device (LOAM_GPU_HOST_RING=1: the host builder)
    if (ok && k.ring && k.bilinear && R.dim == 1 && R.v.arity == 3 && !std::getenv("LOAM_GPU_NO_RING") &&
        !std::getenv("LOAM_GPU_HOST_RING") &&
        build_ring_dev(P->nb, srows.v.get(), n, R.v.target, csr, tile_rows, kTileSeg, kTileSlots, s)) {
      plan_tick("ring tiles (device)", s);
      P->use_nbr = true;
      return P;
    }
    if (ok && build_nbr(P->nb, srows.v.get(), n, R.v.arity, R.v.target, csr, tile_rows,
                        k.bilinear ? kTileSeg : (1 << 30), kTileSlots, kTileRuns, s)) {
      plan_tick("nbr / ring tiles", s);
      P->use_nbr = true;
      return P;
    }
  }
  build_pairs(srows.v.get(), n, R.v.arity, R.v.target, P->pp, s);
  if (k.bilinear) {
    const NodeMap Cn = node_view(args[0].col_map);
    SortedMap scols;
    const int32_t* sc = srows.v.get();
    if (!(Cn.v.v == R.v.v && Cn.v.arity == R.v.arity)) {
      gather_rows(Cn.v, perm, scols, s);
      sc = scols.v.get();
    }
    const loam_sparsity_desc* sp = args[0].sparsity;
    CsrView csr{sp->row_ptr, sp->col_idx, sp->nrows, sp->ncols, sp->nnz, R.dim, Cn.dim};
    plan_tick("pairs", s);
    build_ranks(P->pp, srows.v.get(), sc, Cn.v.arity, csr, s);
    plan_tick("ranks", s);
    build_chunks(P->pp, csr, kSegMax, 32 / R.dim, s);
    plan_tick("chunks", s);
    // edge tiles: scalar P2 mass / stiffness / helmholtz on one (map, map) pattern
    const bool et_form = ((k.form == F_MASS || k.form == F_STIFFNESS || k.form == F_HELMHOLTZ) &&
                          k.nrn == (k.gd == 2 ? 6 : 10) && k.ncn == k.nrn && k.rd == 1 && k.cd == 1) ||
                         (k.form == F_STOKES_A && k.rd == 2 && k.cd == 2);
    if (strat == 0 && et_form && !std::getenv("LOAM_GPU_NO_ETILE") && !(k.form == F_STOKES_A && rtile_form(k.form)) &&
        R.dim == k.rd && Cn.dim == k.cd &&
        (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0 && Cn.v.arity == R.v.arity &&
        (Cn.v.v == R.v.v || prefix_equal(Cn.v.v, Cn.v.arity, R.v.v, R.v.arity, R.v.arity, n, s)) &&
        (P->exact ||
         pattern_is_map_pattern(R.v.v, n, R.v.arity, R.v.target, k.rd, k.cd, sp->row_ptr, sp->col_idx, sp->nnz, s))) {
      P->exact = true;
      SortedMap sx;
      gather_rows(MapView{X->values, n, X->arity, X->target_size}, perm, sx, s);
      // scalar P2 tetrahedra: the edge rows walk their links (wtile.cuh); the
      // edge tiles stay for triangles, the Stokes A block and non-manifold meshes
      if (k.gd == 3 && k.rd == 1 && k.cd == 1 && k.nrn == 10 && !std::getenv("LOAM_GPU_NO_WTILE")) {
        WtileSpec ws;
        ws.tile_rows = env_int("LOAM_GPU_WT_ROWS", ws.tile_rows);
        ws.det = options().deterministic != 0;
        if (build_wtile(P->wt, ws, n, R.v.target, X->target_size, srows.v.get(), sx.v.get(), P->pp, sp->row_ptr,
                        sp->col_idx, sp->nnz, s)) {
          plan_tick("walk tiles", s);
          P->use_wtile = true;
          return P;
        }
        require(!std::getenv("LOAM_GPU_WT_REQUIRE"), LOAM_ERR(UnsupportedForm),
                "walk-tile plan declined (LOAM_GPU_WT_REQUIRE is set: tests of that path)");
        P->wt = WtilePlan{};
      }
      EtileSpec es;
      es.tile_rows = env_int("LOAM_GPU_ET_ROWS", es.tile_rows);
      es.tile_seg = env_int("LOAM_GPU_ET_SEG", es.tile_seg);
      es.tile_cells = env_int("LOAM_GPU_ET_CELLS", es.tile_cells);
      es.det = options().deterministic != 0;
      if (build_etile(P->et, es, k.gd, n, R.v.target, srows.v.get(), sx.v.get(), X->target_size, P->pp,
                      sp->row_ptr, sp->nnz, k.rd, s)) {
        plan_tick("edge tiles", s);
        P->use_etile = true;
        return P;
      }
    }
    // node-block tiles: vector P1 elasticity on its (map, map) 3x3-blocked pattern
    if (strat == 0 && k.form == F_ELASTICITY && !std::getenv("LOAM_GPU_NO_NTILE") && R.dim == 3 && Cn.dim == 3 &&
        (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0 && Cn.v.arity == R.v.arity &&
        (Cn.v.v == R.v.v || prefix_equal(Cn.v.v, Cn.v.arity, R.v.v, R.v.arity, R.v.arity, n, s))) {
      SortedMap sx;
      gather_rows(MapView{X->values, n, X->arity, X->target_size}, perm, sx, s);
      if (!std::getenv("LOAM_GPU_NO_LTILE")) { // manifold meshes: a block walks its edge's link
        LtileSpec ls;
        ls.tile_nodes = env_int("LOAM_GPU_LT_NODES", ls.tile_nodes);
        // (the coordinate map IS the node map for vector P1: one sorted copy serves both)
        const int32_t* lx = (X->values == R.v.v && X->arity == R.v.arity) ? srows.v.get() : sx.v.get();
        if (build_ltile(P->lt, ls, n, R.v.target, srows.v.get(), lx, X->target_size, P->pp, sp->row_ptr,
                        sp->nnz, s)) {
          plan_tick("link tiles", s);
          P->use_ltile = true;
          return P;
        }
        P->lt = LtilePlan{};
      }
      NtileSpec ns;
      ns.tile_nodes = env_int("LOAM_GPU_NT_NODES", ns.tile_nodes);
      ns.tile_items = env_int("LOAM_GPU_NT_ITEMS", ns.tile_items);
      ns.tile_pairs = env_int("LOAM_GPU_NT_PAIRS", ns.tile_pairs);
      ns.tile_cells = env_int("LOAM_GPU_NT_CELLS", ns.tile_cells);
      ns.tile_slots = env_int("LOAM_GPU_NT_SLOTS", ns.tile_slots);
      if (build_ntile(P->nt, ns, n, R.v.target, srows.v.get(), sx.v.get(), X->target_size, P->pp, sp->row_ptr,
                      sp->nnz, s)) {
        plan_tick("node tiles", s);
        P->use_ntile = true;
        return P;
      }
    }
    // row tiles: the Taylor-Hood coupling blocks
    if (strat == 0 && rtile_form(k.form) && !std::getenv("LOAM_GPU_NO_RTILE") && R.dim == k.rd && Cn.dim == k.cd &&
        (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0) {
      SortedMap sx;
      gather_rows(MapView{X->values, n, X->arity, X->target_size}, perm, sx, s);
      RtileSpec rs;
      rs.tile_rows = env_int("LOAM_GPU_RT_ROWS", rs.tile_rows);
      if (build_rtile(P->rt, rs, k.form, k.gd, k.nrn, k.ncn, k.rd, k.cd, n, R.v.target, srows.v.get(), sx.v.get(),
                      X->target_size, P->pp, sp->row_ptr, sp->nnz, s)) {
        plan_tick("row tiles", s);
        P->use_rtile = true;
        return P;
      }
    }
  }
  // canonical pair tiles: default for the scalar / 2-vector bilinear forms the
  // ring / neighbour paths do not take (P2 matrices, Taylor-Hood blocks).  P2
  // actions are coefficient-window bound and 3-vector rows overflow the tile
  // segment; both stay on the pair-list kernel (profiles/r01/strategies_*).
  const bool ptile_form = (k.bilinear && k.rd * k.cd <= 4) || std::getenv("LOAM_GPU_PTILE_ALL");
  if (strat == 0 && ptile_form && !std::getenv("LOAM_GPU_NO_PTILE") && (reinterpret_cast<uintptr_t>(args[1].data) & 15) == 0 &&
      (!Cm || (reinterpret_cast<uintptr_t>(args[2].data) & 15) == 0)) {
    SortedMap sx, scf;
    gather_rows(MapView{X->values, n, X->arity, X->target_size}, perm, sx, s);
    if (Cm) gather_rows(MapView{Cm->values, n, Cm->arity, Cm->target_size}, perm, scf, s);
    PTileSpec spec;
    spec.gd = k.gd;
    spec.nrn = k.nrn;
    spec.ncn = k.bilinear ? k.ncn : 0;
    spec.ncoeff = k.has_coeff ? k.ncoeff : 0;
    spec.rd = k.rd;
    spec.cd = k.cd;
    spec.tile_rows = kPTileThreads;
    spec.tile_seg = env_int("LOAM_GPU_PT_SEG", 4096);
    spec.tile_pairs = env_int("LOAM_GPU_PT_PAIRS", 768);
    spec.tile_slots = env_int("LOAM_GPU_PT_SLOTS", 1024);
    spec.tile_runs = env_int("LOAM_GPU_PT_RUNS", 48);
    CsrView csr{};
    if (k.bilinear) {
      const loam_sparsity_desc* sp = args[0].sparsity;
      csr = CsrView{sp->row_ptr, sp->col_idx, sp->nrows, sp->ncols, sp->nnz, R.dim, node_view(args[0].col_map).dim};
    }
    if (build_ptile(P->pt, spec, n, R.v.target, srows.v.get(), nullptr, sx.v.get(), X->target_size,
                    Cm ? scf.v.get() : nullptr, Cm ? Cm->target_size : 0, P->pp, csr, s)) {
      plan_tick("pair tiles", s);
      P->use_ptile = true;
      return P;
    }
  }
  // sorted coordinate / coefficient maps; share storage where maps coincide
  const MapView xv{X->values, n, X->arity, X->target_size};
  if (Cm) {
    const MapView cv{Cm->values, n, Cm->arity, Cm->target_size};
    if (Cm->values == R.v.v && Cm->arity == R.v.arity) {
      P->cmap = std::move(srows);
    } else {
      gather_rows(cv, perm, P->cmap, s);
    }
    P->cptr = P->cmap.v.get();
    P->cstride = Cm->arity;
    // vertex ids are the first gdim+1 entries of the coefficient map (P1, and P2 vertices first)
    if (prefix_equal(Cm->values, Cm->arity, X->values, X->arity, X->arity, n, s)) {
      P->xptr = P->cptr;
      P->xstride = P->cstride;
    }
  }
  if (!P->xptr) {
    if (X->values == R.v.v && X->arity == R.v.arity && srows.v.get()) {
      P->xmap = std::move(srows);
    } else {
      gather_rows(xv, perm, P->xmap, s);
    }
    P->xptr = P->xmap.v.get();
    P->xstride = X->arity;
  }
  return P;
}

// The argument pattern of assemble_matrix / assemble_vector
// (assemble.hpp:91-99, 123-129) that the owner-computes path serves.
bool fast_pattern(const Entry& k, const loam_arg_desc* args, int nargs) {
  if (k.form < 0 || !k.owner) return false;
  if (nargs != 2 + (k.has_coeff ? 1 : 0)) return false;
  const loam_arg_desc& A = args[0];
  if (A.access != LOAM_INC) return false;
  if (k.bilinear) {
    if (A.kind != LOAM_ARG_MAT) return false;
    const NodeMap R = node_view(A.map), C = node_view(A.col_map);
    if (R.v.arity != k.nrn || R.dim != k.rd || C.v.arity != k.ncn || C.dim != k.cd) return false;
  } else {
    if (A.kind != LOAM_ARG_DAT || !A.map || A.dim != 1 || A.map->arity != k.nrn) return false;
  }
  const loam_arg_desc& X = args[1];
  if (X.kind != LOAM_ARG_DAT || X.access != LOAM_READ || !X.map || X.dim != k.gd ||
      X.map->arity != k.gd + 1)
    return false;
  if (k.has_coeff) {
    const loam_arg_desc& C = args[2];
    if (C.kind != LOAM_ARG_DAT || C.access != LOAM_READ || !C.map || C.dim != 1 ||
        C.map->arity != k.ncoeff)
      return false;
  }
  return true;
}

// set while wave_step() asks run_fast for the loop's plan instead of a launch
thread_local std::shared_ptr<FastPlan>* g_plan_probe = nullptr;

void run_fast(const Entry& k, int n, const loam_arg_desc* args, int nargs, const FormParams& prm,
              cudaStream_t s, bool cell_mode = false) {
  std::vector<uint64_t> key{(uint64_t)k.form, (uint64_t)k.gd, (uint64_t)k.nrn, (uint64_t)k.ncn,
                            (uint64_t)options().locality, (uint64_t)strategy(), (uint64_t)cell_mode,
                            (uint64_t)options().deterministic};
  bool cacheable = true;
  for (int q = 0; q < nargs; ++q) {
    const loam_arg_desc& a = args[q];
    for (const loam_map_desc* m : {a.map, a.col_map})
      if (m) {
        key.push_back(m->id);
        cacheable &= m->id != 0;
      }
    if (a.kind == LOAM_ARG_MAT) {
      key.push_back(a.sparsity->id);
      cacheable &= a.sparsity->id != 0;
    }
  }
  std::shared_ptr<FastPlan> P;
  if (cacheable) {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    auto it = g_fast_cache.find(key);
    if (it != g_fast_cache.end()) P = it->second;
  }
  if (!P) {
    P = build_fast_plan(k, n, args, cell_mode, s);
    // the plan's device arrays are complete before any kernel reads them: the
    // PDL kernels load plan data before griddepcontrol.wait
    LG_CUDA(cudaStreamSynchronize(s));
    if (cacheable) {
      std::lock_guard<std::mutex> g(g_cache_mutex);
      g_fast_cache[key] = P;
    }
  }
  if (g_plan_probe) {
    *g_plan_probe = P;
    return;
  }
  // A fresh output the loop may not reach entirely (a sub-mesh loop into a
  // whole-mesh Mat or Dat): zero it here and let the owner-computes kernels
  // accumulate, so untouched entries stay zero as in the reference
  // (data.hpp:37-39,185-187).  The cell-centric path zero-fills on its own.
  std::vector<loam_arg_desc> local;
  if ((args[0].flags & LOAM_ARG_ZERO) && !P->exact && !P->use_cell) {
    const size_t len = k.bilinear ? (size_t)args[0].sparsity->nnz : (size_t)args[0].set_size * args[0].dim;
    LG_CUDA(cudaMemsetAsync(args[0].data, 0, sizeof(double) * len, s));
    local.assign(args, args + nargs);
    local[0].flags &= ~LOAM_ARG_ZERO;
    args = local.data();
  }
  if (P->use_star) {
    StarArgs t{};
    t.star = P->star.get();
    t.nrows = k.bilinear ? args[0].sparsity->nrows : args[0].set_size;
    t.row_ptr = k.bilinear ? args[0].sparsity->row_ptr : nullptr;
    t.coords = args[1].data;
    t.coeff = k.has_coeff ? args[2].data : nullptr;
    t.prm = prm;
    t.out = args[0].data;
    t.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
    k.star(t, s);
    return;
  }
  if (P->use_patch) {
    const PatchPlan& pp = P->patch;
    PatchArgs t{};
    t.hdr = pp.hdr.get();
    t.npatches = pp.npatches;
    t.win = pp.win.get();
    t.recs = pp.recs.get();
    t.own = pp.own.get();
    t.orp = pp.orp.get();
    t.oseg = pp.oseg.get();
    t.coords = args[1].data;
    t.coeff = k.has_coeff ? args[2].data : nullptr;
    t.prm = prm;
    t.out = args[0].data;
    t.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
    t.max_win = pp.max_win;
    t.max_cells = pp.max_cells;
    t.max_own = pp.max_own;
    t.max_pairs = pp.max_pairs;
    t.max_seg = (int)pp.max_seg;
    t.bw = (pp.max_win + 31) / 32;
    t.nverts = args[1].map->target_size;
    if (!k.bilinear && !t.accumulate) // shared nodes are RED-accumulated; nodes in no cell stay zero
      LG_CUDA(cudaMemsetAsync(args[0].data, 0, sizeof(double) * (size_t)args[0].set_size * args[0].dim, s));
    k.patch(t, patch_smem_bytes(k, pp), s);
    return;
  }
  if (P->use_ctile) {
    const int ctr = P->counter.acquire(s);
    launch_ctile(k.form, P->ct, args[1].data, args[2].data, args[0].data, (int64_t)args[0].set_size * args[0].dim,
                 prm, !(args[0].flags & LOAM_ARG_ZERO), P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_cell) {
    CellArgs c{};
    c.cranks = P->cranks.get();
    c.row_ptr = k.bilinear ? args[0].sparsity->row_ptr : nullptr;
    c.n = n;
    c.rmap = P->crows.v.get();
    c.xmap = P->xptr;
    c.xstride = P->xstride;
    c.cmap = P->cptr;
    c.cstride = P->cstride;
    c.coords = args[1].data;
    c.coeff = k.has_coeff ? args[2].data : nullptr;
    c.prm = prm;
    c.out = args[0].data;
    if (P->det_cell) { // deterministic: entries in place, then fixed-order row sums
      DevBuf<double> contrib((size_t)n * k.nrn, s);
      c.contrib = contrib.get();
      k.cell(c, false, s);
      const int nrows = P->pp.nrows_node;
      k_pair_sum<<<ceil_div(nrows, 256), 256, 0, s>>>(P->pp.ptr.get(), P->pp.pairs.get(), nrows, contrib.get(),
                                                      args[0].data, (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1);
      count_launch();
      LG_LAUNCH_CHECK();
      return;
    }
    if (args[0].flags & LOAM_ARG_ZERO) {
      const size_t len = k.bilinear ? (size_t)args[0].sparsity->nnz : (size_t)args[0].set_size * args[0].dim;
      LG_CUDA(cudaMemsetAsync(args[0].data, 0, sizeof(double) * len, s));
    }
    if (P->use_cseg) {
      CellSegArgs g{};
      g.c = c;
      g.slots = P->cs_slots.get();
      g.seg_off = P->cs_off.get();
      g.seg_start = P->cs_start.get();
      g.seg_node = P->cs_node.get();
      g.nbatches = P->cs_nbatches;
      k.cell_seg(g, s);
      return;
    }
    k.cell(c, strategy() == 5, s);
    return;
  }
  if (P->use_nbr && P->nb.ring && k.ring && !std::getenv("LOAM_GPU_NO_RING")) {
    const NbrPlan& nb = P->nb;
    RingArgs t{};
    t.tiles = nb.rtiles.get();
    t.ntiles = nb.ntiles;
    const int ctr = P->counter.acquire(s);
    t.next_tile = P->counter.next(ctr);   // tile counter
    t.reset_tile = P->counter.exits(ctr); // exit count (tile_counter_release)
    t.nptr = nb.nptr.get();
    t.rptr = nb.rptr.get();
    t.recs = nb.rrecs.get();
    t.rowinfo = nb.rowinfo.get();
    t.runs = nb.runs.get();
    t.coords = args[1].data;
    t.coeff = k.has_coeff ? args[2].data : nullptr;
    t.prm = prm;
    t.out = args[0].data;
    t.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
    auto up16 = [](int x) { return (x + 15) & ~15; };
    int off = 128; // 6 mbarriers + 3 stage tile ids
    t.off_seg = off;
    // one slice per consumer warp: 32 rows of at most max_len entries (+ skew)
    t.seg_stride = k.bilinear ? up16((32 * nb.max_len + 2) * 8) / 8 : 0;
    off += (kTileThreads / 32) * t.seg_stride * 8;
    t.off_buf = off;
    int b = 0;
    t.b_nptr = b;
    b += up16((nb.max_rows + 1) * 4 + 32);
    t.b_rptr = b;
    b += up16((nb.max_rows + 1) * 4 + 32);
    t.b_recs = b;
    b += up16(nb.max_pairs * 2 + 32);
    t.b_info = b;
    b += up16(nb.max_rows * 4 + 32);
    t.b_win = b;
    b += up16(nb.max_slots * 16);
    t.b_winc = b;
    b += up16(k.has_coeff ? nb.max_slots * 8 : 0);
    t.buf_bytes = b;
    off += kRS * b;
    static const bool timing = std::getenv("LOAM_GPU_PHASE_TIMING") != nullptr;
    DevBuf<unsigned long long> tbuf;
    if (timing) {
      tbuf.alloc(16 + 4 * 2048 + 2 * 16384, s);
      LG_CUDA(cudaMemsetAsync(tbuf.get(), 0, tbuf.bytes(), s));
      LG_CUDA(cudaMemsetAsync(tbuf.get() + 8, 0xff, 8, s));
      LG_CUDA(cudaMemsetAsync(tbuf.get() + 12, 0xff, 8, s));
      t.timing = tbuf.get();
    }
    k.ring(t, (size_t)off, s);
    P->counter.commit(ctr, s);
    if (timing) {
      std::vector<unsigned long long> hv(16 + 4 * 2048 + 2 * 16384);
      unsigned long long* h = hv.data();
      LG_CUDA(cudaMemcpyAsync(h, tbuf.get(), sizeof(unsigned long long) * hv.size(), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
      if (const char* dump = std::getenv("LOAM_GPU_PHASE_DUMP")) {
        FILE* f = fopen(dump, "w");
        for (int b = 0; b < 2048 && h[17 + 4 * b]; ++b)
          fprintf(f, "%d %.3f %.3f %llu %llu\n", b, (h[16 + 4 * b] - h[8]) * 1e-3, (h[17 + 4 * b] - h[8]) * 1e-3,
                  h[18 + 4 * b], h[19 + 4 * b]);
        fclose(f);
        f = fopen((std::string(dump) + ".tiles").c_str(), "w");
        for (int t = 0; t < std::min(nb.ntiles, 16384); ++t)
          fprintf(f, "%d %llu %llu\n", t, h[16 + 4 * 2048 + 2 * t], h[17 + 4 * 2048 + 2 * t]);
        fclose(f);
      }
      const double nw = std::max(1.0, (double)h[4]), nt = std::max(1.0, (double)h[3]);
      fprintf(stderr, "[ring timing] cycles per consumer warp: total %.0f = first wait %.0f + stage 1-2 waits %.0f + "
              "steady waits %.0f + final wait %.0f + compute %.0f (%.1f tiles/warp; tiles %d, warps %.0f, smem %d B)\n",
              h[7] / nw, h[0] / nw, h[5] / nw, h[1] / nw, h[6] / nw, h[2] / nw, nt / nw, nb.ntiles, nw, off);
      fprintf(stderr, "[ring timing] CTA starts span %.2f us, CTA ends from %.2f to %.2f us after the first start\n",
              (double)(h[11] - h[8]) * 1e-3, (double)(h[12] - h[8]) * 1e-3, (double)(h[9] - h[8]) * 1e-3);
    }
    return;
  }
  if (P->use_rtile) {
    const int ctr = P->counter.acquire(s);
    launch_rtile(P->rt, args[1].data, args[0].data, prm, !(args[0].flags & LOAM_ARG_ZERO),
                 P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_wtile) {
    const int ctr = P->counter.acquire(s);
    launch_wtile(P->wt, k.form, args[1].data, args[0].data, prm, !(args[0].flags & LOAM_ARG_ZERO),
                 P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_ltile) {
    const int ctr = P->counter.acquire(s);
    launch_ltile(P->lt, args[1].data, args[0].data, prm, !(args[0].flags & LOAM_ARG_ZERO),
                 P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_ntile) {
    const int ctr = P->counter.acquire(s);
    launch_ntile(P->nt, args[1].data, args[0].data, prm, !(args[0].flags & LOAM_ARG_ZERO),
                 P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_etile) {
    const int ctr = P->counter.acquire(s);
    launch_etile(k.form, P->et, args[1].data, args[0].data, prm, !(args[0].flags & LOAM_ARG_ZERO),
                 P->counter.next(ctr), P->counter.exits(ctr), s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_ptile) {
    const PTilePlan& pt = P->pt;
    PTileArgs t{};
    t.tiles = pt.tiles.get();
    t.ntiles = pt.ntiles;
    const int ctr = P->counter.acquire(s);
    t.next_tile = P->counter.next(ctr);   // tile counter
    t.reset_tile = P->counter.exits(ctr); // exit count (tile_counter_release)
    t.pptr = pt.pptr.get();
    t.nptr = pt.nptr.get();
    t.recs = pt.recs.get();
    t.runs = pt.runs.get();
    t.cruns = pt.cruns.get();
    t.coords = args[1].data;
    t.coeff = k.has_coeff ? args[2].data : nullptr;
    t.prm = prm;
    t.out = args[0].data;
    t.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
    t.cas = env_int("LOAM_GPU_PTILE_CAS", 0);
    auto up16 = [](int x) { return (x + 15) & ~15; };
    int off = 128;
    t.off_seg = off;
    off += up16(k.bilinear ? pt.max_seg * 8 : 0);
    t.off_buf = off;
    int b = 0;
    t.b_pptr = b;
    b += up16((pt.max_rows + 1) * 4 + 32);
    t.b_nptr = b;
    b += up16(k.bilinear ? (pt.max_rows + 1) * 4 + 32 : 0);
    t.b_recs = b;
    b += up16(pt.max_pairs * pt.rec_bytes + 32);
    t.b_win = b;
    b += up16(pt.max_slots * k.gd * 8 + 16);
    t.b_winc = b;
    b += up16(k.has_coeff ? pt.max_cslots * 8 + 16 : 0);
    t.buf_bytes = b;
    k.ptile(t, (size_t)off, (size_t)b, s);
    P->counter.commit(ctr, s);
    return;
  }
  if (P->use_nbr) {
    const NbrPlan& nb = P->nb;
    TileArgs t{};
    t.tiles = nb.tiles.get();
    t.ntiles = nb.ntiles;
    t.nptr = nb.nptr.get();
    t.pptr = nb.pptr.get();
    t.recs = nb.recs.get();
    t.widx = nb.widx.get();
    t.selfr = nb.selfr.get();
    t.runs = nb.runs.get();
    t.coords = args[1].data;
    t.coeff = k.has_coeff ? args[2].data : nullptr;
    t.prm = prm;
    t.out = args[0].data;
    t.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
    t.bits = nb.bits;
    t.max_len = nb.max_len;
    auto up16 = [](int x) { return (x + 15) & ~15; };
    int off = 64; // 6 mbarriers
    t.off_seg = off;
    const bool reg = k.bilinear && k.rd == 1 && k.cd == 1 && nb.max_len <= 8 && std::getenv("LOAM_GPU_REG");
    off += up16(k.bilinear && !reg ? nb.max_seg * 8 : 0);
    t.off_buf = off;
    int b = 0;
    t.b_nptr = b;
    b += up16((nb.max_rows + 1) * 4 + 32);
    t.b_pptr = b;
    b += up16((nb.max_rows + 1) * 4 + 32);
    t.b_recs = b;
    b += up16(nb.max_pairs * nb.rec_bytes + 32);
    t.b_widx = b;
    b += up16(nb.max_adj * 2 + 32);
    t.b_selfr = b;
    b += up16(nb.max_rows + 32);
    t.b_win = b;
    b += up16(nb.max_slots * k.gd * 8);
    t.b_winc = b;
    b += up16(k.has_coeff ? nb.max_slots * 8 : 0);
    t.buf_bytes = b;
    off += 3 * b;
    static const bool timing = std::getenv("LOAM_GPU_PHASE_TIMING") != nullptr;
    DevBuf<long long> tbuf;
    if (timing) {
      tbuf.alloc(4, s);
      LG_CUDA(cudaMemsetAsync(tbuf.get(), 0, tbuf.bytes(), s));
      t.timing = tbuf.get();
    }
    k.nbr(t, nb.rec_bytes, (size_t)off, s);
    if (timing) {
      long long h[4];
      LG_CUDA(cudaMemcpyAsync(h, tbuf.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
      fprintf(stderr, "[phase timing] per warp-tile cycles: wait %.0f compute %.0f (tiles %d, smem %d B)\n",
              (double)h[0] / std::max<long long>(h[2], 1), (double)h[1] / std::max<long long>(h[2], 1), nb.ntiles, off);
    }
    return;
  }
  OwnerArgs a{};
  a.ptr = P->pp.ptr.get();
  a.pairs = P->pp.pairs.get();
  a.ranks = P->pp.ranks.get();
  a.xmap = P->xptr;
  a.xstride = P->xstride;
  a.coords = args[1].data;
  a.cmap = P->cptr;
  a.cstride = P->cstride;
  a.coeff = k.has_coeff ? args[2].data : nullptr;
  a.prm = prm;
  a.out = args[0].data;
  a.nrows_node = P->pp.nrows_node;
  a.accumulate = (args[0].flags & LOAM_ARG_ZERO) ? 0 : 1;
  if (k.bilinear) {
    a.row_ptr = args[0].sparsity->row_ptr;
    a.chunk_row = P->pp.chunk_row.get();
    a.nchunks = P->pp.nchunks;
    a.seg_max = P->pp.seg_max;
    const int warps = 4;
    k.owner(a, ceil_div(a.nchunks, warps), (size_t)warps * a.seg_max * sizeof(double), s);
  } else {
    k.owner(a, ceil_div(a.nrows_node, kTPB), 0, s);
  }
}

// --- generic path ----------------------------------------------------------

std::shared_ptr<ColorCacheEntry> get_coloring(int n, uint64_t iter, const std::vector<const loam_map_desc*>& maps,
                                              cudaStream_t s) {
  std::vector<uint64_t> key{iter, (uint64_t)n};
  bool cacheable = iter != 0;
  std::vector<const loam_map_desc*> uniq;
  for (auto* m : maps) {
    bool dup = false;
    for (auto* u : uniq) dup |= (u == m) || (m->id && u->id == m->id);
    if (!dup) uniq.push_back(m);
  }
  std::sort(uniq.begin(), uniq.end(), [](auto* a, auto* b) { return a->id < b->id; });
  for (auto* m : uniq) {
    key.push_back(m->id);
    cacheable &= m->id != 0;
  }
  if (cacheable) {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    auto it = g_color_cache.find(key);
    if (it != g_color_cache.end()) return it->second;
  }
  auto c = std::make_shared<ColorCacheEntry>();
  std::vector<MapView> mv;
  for (auto* m : uniq) mv.push_back(MapView{m->values, m->source_size, m->arity, m->target_size});
  color_dev(n, mv, c->cp, s);
  if (cacheable) {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    g_color_cache[key] = c;
  }
  return c;
}

void run_generic(const Entry& k, int n, uint64_t iter, const loam_arg_desc* args, int nargs,
                 const FormParams& prm, cudaStream_t s) {
  GLaunch L{};
  L.nargs = nargs;
  L.prm = prm;
  int off = 0, slot_stride = 0;
  bool need_color = options().inc_strategy == 3 || options().deterministic; // colouring: the reference's order
  std::vector<const loam_map_desc*> conflict;
  for (int q = 0; q < nargs; ++q) {
    const loam_arg_desc& a = args[q];
    GArg& g = L.a[q];
    g.kind = a.kind;
    g.access = a.access;
    g.dim = a.dim;
    g.data = a.data;
    std::vector<int> ext = staged_extents(a);
    g.size = 1;
    for (int x : ext) g.size *= x;
    g.off = off;
    off += g.size;
    if (a.map) {
      g.map = a.map->values;
      g.arity = a.map->arity;
    }
    if (a.kind == LOAM_ARG_MAT) {
      g.map2 = a.col_map->values;
      g.arity2 = a.col_map->arity;
      g.row_ptr = a.sparsity->row_ptr;
      g.col_idx = a.sparsity->col_idx;
      g.nrows = a.sparsity->nrows;
      conflict.push_back(a.map);
      conflict.push_back(a.col_map);
      if (a.access == LOAM_WRITE) need_color = true;
    } else if (a.kind == LOAM_ARG_DAT && a.map && writes(a.access)) { // parloop.hpp:212-215
      conflict.push_back(a.map);
      if (a.access != LOAM_INC) need_color = true;
    } else if (a.kind == LOAM_ARG_GLOBAL && a.access != LOAM_READ) {
      g.slot_off = slot_stride;
      slot_stride += a.dim;
    }
  }
  require(off == k.stage, LOAM_ERR(ShapeMismatch), "staged size mismatch");
  // lazily zero-initialised targets (LOAM_ARG_ZERO): this path accumulates
  for (int q = 0; q < nargs; ++q) {
    const loam_arg_desc& a = args[q];
    if (!(a.flags & LOAM_ARG_ZERO) || a.access == LOAM_READ || a.kind == LOAM_ARG_GLOBAL) continue;
    const size_t count = a.kind == LOAM_ARG_MAT ? (size_t)a.sparsity->nnz : (size_t)a.set_size * a.dim;
    if (count) {
      LG_CUDA(cudaMemsetAsync(a.data, 0, sizeof(double) * count, s));
      count_launch();
    }
  }
  L.slot_stride = slot_stride;
  DevBuf<double> slots;
  if (slot_stride) {
    slots.alloc((size_t)std::max(n, 1) * slot_stride, s);
    L.slots = slots.get();
  }
  DevBuf<unsigned long long> err(1, s);
  LG_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(unsigned long long), s));
  L.err = err.get();
  if (need_color && !conflict.empty() && n > 0) {
    auto c = get_coloring(n, iter, conflict, s);
    L.plain = 1;
    for (int col = 0; col < c->cp.ncolors; ++col) {
      L.order = c->cp.order.get() + c->cp.offsets[col];
      L.count = c->cp.offsets[col + 1] - c->cp.offsets[col];
      k.generic(L, s);
    }
  } else {
    L.order = nullptr;
    L.count = n;
    L.plain = 0;
    k.generic(L, s);
  }
  // Global reductions, then overwrite (parloop.hpp:354-383)
  for (int q = 0; q < nargs; ++q) {
    const loam_arg_desc& a = args[q];
    if (a.kind != LOAM_ARG_GLOBAL || a.access == LOAM_READ) continue;
    if (n == 0) {
      k_fill_identity<<<1, 32, 0, s>>>(a.data, a.dim, a.access);
    } else {
      k_global_reduce<<<a.dim, kTPB, 0, s>>>(L.slots, n, slot_stride, L.a[q].slot_off, a.access, a.data);
    }
    count_launch();
    LG_LAUNCH_CHECK();
  }
  if (options().check_sparsity) {
    bool has_mat = false;
    for (int q = 0; q < nargs; ++q) has_mat |= args[q].kind == LOAM_ARG_MAT;
    if (has_mat) {
      unsigned long long h = 0;
      LG_CUDA(cudaMemcpyAsync(&h, err.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
      if (h >> 63)
        fail(LOAM_ERR(OutsideSparsity), "mat: entry (" + std::to_string((int)((h >> 32) & 0x7fffffff)) +
                                            ", " + std::to_string((int)(uint32_t)h) + ") outside sparsity");
    }
  }
}

} // namespace

// ===========================================================================
// Public engine API
// ===========================================================================

const KernelInfo* find_kernel(const std::string& name) {
  const Entry* e = find_entry(name);
  return e ? &e->info : nullptr;
}

const std::string& kernel_names() {
  static const std::string prod = [] {
    std::string r;
    for (auto& [name, e] : registry()) r += name + "\n";
    return r;
  }();
  static const std::string all = [] {
    std::string r = prod;
    for (auto& [name, e] : test_registry()) r += name + "\n";
    return r;
  }();
  return options().test_kernels ? all : prod;
}

void validate(const loam_kernel_desc* kd, int n, uint64_t iter, const loam_arg_desc* args, int nargs) {
  require(kd != nullptr, LOAM_ERR(InvalidArgument), "parloop without kernel");
  validate_args(lookup(kd->name), n, iter, args, nargs);
}

void execute(const loam_kernel_desc* kd, int n, uint64_t iter, const loam_arg_desc* args, int nargs,
             cudaStream_t s) {
  require(kd != nullptr, LOAM_ERR(InvalidArgument), "parloop without kernel");
  const Entry& k = lookup(kd->name);
  validate_args(k, n, iter, args, nargs); // before any mutation (parloop.hpp:193)
  FormParams prm{{0, 0, 0, 0}};
  for (int i = 0; i < kd->nparams && i < 4; ++i) prm.p[i] = kd->params[i];
  // deterministic mode: the auto paths only (the atomic / warp-aggregated /
  // patch strategies sum in a varying order); the RED-based pieces of auto run
  // their fixed-order variants (cell entries + pair sums, edge-tile diagonals)
  const int strat = strategy();
  // auto: P2 tetrahedral actions (C3 residual) are fastest with one fp64 RED
  // per element entry -- 10 rows per cell, each recomputed by its owner would
  // redo the cell geometry 10 times (profiles/r01/strategies_*: 0.34 vs 0.80 ms)
  const bool atomic_auto = strat == 0 && !std::getenv("LOAM_GPU_PTILE_ALL") && !k.bilinear && k.form >= 0 && k.gd == 3 && k.nrn > k.gd + 1;
  // catalogue forms under the atomic strategies (and P2-tet actions under
  // auto): the cell-centric kernel, plain or warp-aggregated REDs
  if (n > 0 && k.cell && (atomic_auto || strat == 1 || strat == 5) && fast_pattern(k, args, nargs)) {
    try {
      run_fast(k, n, args, nargs, prm, s, true);
      return;
    } catch (const Error& e) {
      if (e.code() != LOAM_ERR(ShapeMismatch)) throw; // unblocked pattern: generic engine
    }
  }
  if (n > 0 && !atomic_auto && (strat == 0 || strat == 2 || strat == 4 || strat == 6) && fast_pattern(k, args, nargs)) {
    try {
      run_fast(k, n, args, nargs, prm, s);
      return;
    } catch (const Error& e) {
      // a pattern that is not blocked by the maps' dof expansion is served by
      // the generic path; every other failure propagates
      if (e.code() != LOAM_ERR(ShapeMismatch)) throw;
    }
  }
  run_generic(k, n, iter, args, nargs, prm, s);
}

// ---------------------------------------------------------------------------
// fem::assemble_blocks (fem/assemble.hpp:439-448): the loops of a nested block
// matrix issued together.  The Taylor-Hood triple (stokes_a / stokes_b /
// stokes_bt over one cell set, velocity map, pressure map and coordinate Dat)
// runs as ONE launch (thtile.cuh) when its plan builds; any other list -- and
// the triple on a mesh or pattern the plan declines -- runs loop by loop,
// exactly as the reference does.
struct ThFused { // (static tile schedule: no counters, any number of launches in flight)
  ThtilePlan plan;
  bool ok = false;
};
std::map<std::vector<uint64_t>, std::shared_ptr<ThFused>> g_th_cache;

bool try_taylor_hood(const LoopDesc* loops, int nloops, cudaStream_t s) {
  if (nloops != 3 || strategy() != 0 || std::getenv("LOAM_GPU_NO_THTILE")) return false;
  int ia = -1, ib = -1, it = -1;
  for (int i = 0; i < 3; ++i) {
    if (!loops[i].kernel || !loops[i].kernel->name) return false;
    const Entry& k = lookup(loops[i].kernel->name);
    if (k.form == F_STOKES_A && ia < 0) ia = i;
    else if (k.form == F_STOKES_B && ib < 0) ib = i;
    else if (k.form == F_STOKES_BT && it < 0) it = i;
    else return false;
    if (!fast_pattern(k, loops[i].args, loops[i].nargs)) return false;
  }
  const int n = loops[ia].n;
  if (n <= 0 || loops[ib].n != n || loops[it].n != n || loops[ib].iter != loops[ia].iter ||
      loops[it].iter != loops[ia].iter || loops[ia].kernel->nparams < 1)
    return false;
  const loam_arg_desc &A = loops[ia].args[0], &B = loops[ib].args[0], &T = loops[it].args[0], &X = loops[ia].args[1];
  for (int i : {ib, it}) {
    const loam_arg_desc& Xi = loops[i].args[1];
    if (Xi.data != X.data || Xi.map->values != X.map->values || Xi.map->arity != X.map->arity) return false;
  }
  const NodeMap RA = node_view(A.map), CA = node_view(A.col_map), RB = node_view(B.map), CB = node_view(B.col_map),
                RT = node_view(T.map), CT = node_view(T.col_map);
  auto same = [](const NodeMap& a, const NodeMap& b) {
    return a.v.v == b.v.v && a.v.arity == b.v.arity && a.v.target == b.v.target && a.dim == b.dim && a.v.n == b.v.n;
  };
  if (!same(RA, CA) || !same(RA, CB) || !same(RA, RT) || !same(RB, CT)) return false;
  if (RA.v.arity != 6 || RA.dim != 2 || RB.v.arity != 3 || RB.dim != 1 || RA.v.n != n || RB.v.n != n) return false;
  const MapView xm{X.map->values, n, X.map->arity, X.map->target_size};
  if (xm.arity != 3 || X.map->source_size != n || RB.v.target != xm.target) return false;
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!aligned(X.data) || !aligned(A.data) || !aligned(B.data) || !aligned(T.data)) return false;
  if (A.data == B.data || A.data == T.data || B.data == T.data) return false;
  std::vector<uint64_t> key{(uint64_t)n};
  bool cacheable = true;
  for (const loam_arg_desc* a : {&A, &B, &T}) {
    for (uint64_t id : {a->map->id, a->col_map->id, a->sparsity->id}) {
      key.push_back(id);
      cacheable &= id != 0;
    }
  }
  key.push_back(X.map->id);
  cacheable &= X.map->id != 0;
  std::shared_ptr<ThFused> P;
  if (cacheable) {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    auto f = g_th_cache.find(key);
    if (f != g_th_cache.end()) P = f->second;
  }
  if (!P) {
    plan_tick("plan start", s);
    P = std::make_shared<ThFused>();
    bool ok = RB.v.v == xm.v || prefix_equal(RB.v.v, 3, xm.v, 3, 3, n, s);
    auto exact = [&](const loam_arg_desc& a, const NodeMap& R, const NodeMap& C) {
      const loam_sparsity_desc* sp = a.sparsity;
      return pattern_provenance_exact(a) ||
             pattern_is_maps_pattern(R.v, C.v, R.dim, C.dim, sp->row_ptr, sp->col_idx, sp->nnz, s);
    };
    ok = ok && exact(A, RA, CA) && exact(B, RB, CB) && exact(T, RT, CT);
    plan_tick("thtile: checks", s);
    if (ok) {
      PairPlan pp;
      build_pairs(RA.v.v, n, 6, RA.v.target, pp, s);
      ThtileSpec ts;
      ts.spoke_items = env_int("LOAM_GPU_TH_SPOKES", ts.spoke_items);
      ts.edge_items = env_int("LOAM_GPU_TH_EDGES", ts.edge_items);
      ok = build_thtile(P->plan, ts, n, RA.v.target, xm.target, RA.v.v, xm.v, pp, A.sparsity->row_ptr, A.sparsity->nnz,
                        B.sparsity->row_ptr, B.sparsity->nnz, T.sparsity->row_ptr, T.sparsity->nnz, s);
      plan_tick("thtile", s);
    }
    if (!ok) P->plan = ThtilePlan{};
    P->ok = ok;
    LG_CUDA(cudaStreamSynchronize(s)); // plan data complete before a PDL kernel reads it
    if (cacheable) {
      std::lock_guard<std::mutex> g(g_cache_mutex);
      g_th_cache[key] = P;
    }
  }
  if (!P->ok) return false;
  const int acc = ((A.flags & LOAM_ARG_ZERO) ? 0 : 1) | ((B.flags & LOAM_ARG_ZERO) ? 0 : 2) |
                  ((T.flags & LOAM_ARG_ZERO) ? 0 : 4);
  launch_thtile(P->plan, X.data, A.data, B.data, T.data, loops[ia].kernel->params[0], acc, s);
  return true;
}

void execute_blocks(const LoopDesc* loops, int nloops, cudaStream_t s) {
  require(nloops >= 0 && (nloops == 0 || loops != nullptr), LOAM_ERR(InvalidArgument), "block loops without a list");
  // every loop is validated before anything is written (parloop.hpp:193 per loop)
  for (int i = 0; i < nloops; ++i) validate(loops[i].kernel, loops[i].n, loops[i].iter, loops[i].args, loops[i].nargs);
  if (try_taylor_hood(loops, nloops, s)) return;
  for (int i = 0; i < nloops; ++i) execute(loops[i].kernel, loops[i].n, loops[i].iter, loops[i].args, loops[i].nargs, s);
}

void wave_step(const loam_kernel_desc* kd, int n, uint64_t iter, const loam_arg_desc* args, int nargs,
               const double* p_in, const double* phi_in, double* p_out, double* phi_out, const double* pc,
               const uint8_t* bc, double half_dt, double* state, cudaStream_t s) {
  require(kd != nullptr, LOAM_ERR(InvalidArgument), "parloop without kernel");
  const Entry& k = lookup(kd->name);
  validate_args(k, n, iter, args, nargs);
  require(k.form == F_STIFFNESS_ACTION && k.gd == 2 && k.nrn == 3 && !k.bilinear && nargs == 3,
          LOAM_ERR(UnsupportedForm), "wave step: the action must be stiffness_action_p1_tri");
  require(strategy() == 0 && fast_pattern(k, args, nargs), LOAM_ERR(UnsupportedForm),
          "wave step: needs the auto strategy's vertex-star plan");
  std::shared_ptr<FastPlan> P;
  g_plan_probe = &P;
  try {
    run_fast(k, n, args, nargs, FormParams{{0, 0, 0, 0}}, s);
  } catch (...) {
    g_plan_probe = nullptr;
    throw;
  }
  g_plan_probe = nullptr;
  require(P && P->use_star, LOAM_ERR(UnsupportedForm), "wave step: the mesh has no vertex-star plan");
  StarArgs t{};
  t.star = P->star.get();
  t.nrows = args[0].set_size;
  t.coords = args[1].data;
  t.coeff = nullptr;
  t.out = nullptr;
  WaveFields w{p_in, phi_in, p_out, phi_out, pc, bc, half_dt, state};
  if (t.nrows == 0) return;
  k_wave_step<FormT<F_STIFFNESS_ACTION, 2, 1>><<<ceil_div(t.nrows, 256), 256, 0, s>>>(t, w);
  count_launch();
  LG_LAUNCH_CHECK();
}

void plan_cache_clear() {
  std::lock_guard<std::mutex> g(g_cache_mutex);
  g_fast_cache.clear();
  g_color_cache.clear();
  g_th_cache.clear();
}

void plan_cache_release(uint64_t id) {
  // key layouts: fast plans = 7 shape words, then object ids; colourings =
  // {iteration set id, n, map ids...}
  auto holds = [id](const std::vector<uint64_t>& k, size_t from, size_t skip) {
    for (size_t i = from; i < k.size(); ++i)
      if (i != skip && k[i] == id) return true;
    return false;
  };
  std::vector<std::shared_ptr<FastPlan>> dead_fast;
  std::vector<std::shared_ptr<ColorCacheEntry>> dead_color;
  {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    for (auto it = g_fast_cache.begin(); it != g_fast_cache.end();) {
      if (holds(it->first, 7, (size_t)-1)) {
        dead_fast.push_back(std::move(it->second));
        it = g_fast_cache.erase(it);
      } else {
        ++it;
      }
    }
    for (auto it = g_color_cache.begin(); it != g_color_cache.end();) {
      if (holds(it->first, 0, 1)) {
        dead_color.push_back(std::move(it->second));
        it = g_color_cache.erase(it);
      } else {
        ++it;
      }
    }
  }
  std::vector<std::shared_ptr<ThFused>> dead_th;
  {
    std::lock_guard<std::mutex> g(g_cache_mutex);
    for (auto it = g_th_cache.begin(); it != g_th_cache.end();) {
      if (holds(it->first, 1, (size_t)-1)) {
        dead_th.push_back(std::move(it->second));
        it = g_th_cache.erase(it);
      } else {
        ++it;
      }
    }
  }
  if (!dead_fast.empty() || !dead_color.empty() || !dead_th.empty())
    LG_CUDA(cudaDeviceSynchronize()); // queued launches may use them
}

namespace {
__global__ void k_map_check(const int32_t* __restrict__ v, int64_t n, int target, unsigned long long* bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int x = v[t];
  if (x < 0 || x >= target) atomicCAS(bad, 0ull, (1ull << 63) | (uint32_t)x);
}
} // namespace

void map_check(const loam_map_desc* m, cudaStream_t s) { // topology.hpp:45-48
  require(m->arity > 0, LOAM_ERR(InvalidArgument), "Map arity must be positive");
  const int64_t total = (int64_t)m->source_size * m->arity;
  DevBuf<unsigned long long> bad(1, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), s));
  if (total) {
    k_map_check<<<ceil_div(total, kTPB), kTPB, 0, s>>>(m->values, total, m->target_size, bad.get());
    count_launch();
    LG_LAUNCH_CHECK();
  }
  unsigned long long h = 0;
  LG_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (h >> 63)
    fail(LOAM_ERR(IndexOutOfRange), "map: map entry " + std::to_string((int)(uint32_t)h) +
                                        " outside target set of size " + std::to_string(m->target_size));
}

void color_iteration(int n, const loam_map_desc* maps, int nmaps, int32_t* colors, int32_t* ncolors,
                     cudaStream_t s) {
  std::vector<MapView> mv;
  for (int i = 0; i < nmaps; ++i) {
    require(maps[i].source_size == n, LOAM_ERR(SourceMismatch),
            "conflict map source differs from iteration set");
    bool dup = false;
    for (int j = 0; j < i; ++j) dup |= maps[j].values == maps[i].values && maps[j].arity == maps[i].arity;
    if (!dup) mv.push_back(MapView{maps[i].values, n, maps[i].arity, maps[i].target_size});
  }
  ColorPlan cp;
  if (mv.empty()) { // direct loop: everything colour 0 (test_topology.cpp:64-67)
    LG_CUDA(cudaMemsetAsync(colors, 0, sizeof(int32_t) * n, s));
    *ncolors = n > 0 ? 1 : 0;
    return;
  }
  color_dev(n, mv, cp, s);
  if (n) LG_CUDA(cudaMemcpyAsync(colors, cp.colors.get(), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  *ncolors = cp.ncolors;
}

} // namespace loam_gpu
