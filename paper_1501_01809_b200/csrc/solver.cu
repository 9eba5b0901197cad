// solver.cu -- the consumers of the assembled matrix on sm_100a:
// CSR SpMV, nested 2x2 block SpMV and preconditioned CG.
//
// Reference: data.hpp:236-250 (mat_spmv), solver.hpp:21-58 (BlockMat,
// block_spmv), solver.hpp:60-207 (jacobi_inverse_diagonal, cg_iterate,
// cg_solve).
//
// * SpMV folds every row sequentially in column order with a separate
//   multiply and add (__dmul_rn / __dadd_rn: no FMA contraction), exactly as
//   the reference's `acc += vals[k] * x[col]`, so y is bitwise equal to the
//   reference.  One thread per row; a nested operator folds block 0 then
//   block 1 of its row (solver.hpp:42-53).
// * CG keeps the reference's control flow -- breakdown test on p'Ap, the
//   recurrence norm test re-verified with the true residual, Jacobi scaling,
//   maxit -- but runs it on the device: every kernel of an iteration is gated
//   by flags in a device-resident state (done / recheck), so the host
//   launches batches of iterations and synchronises only once per batch.
//   Vector updates keep the reference's separate multiply and add; dot
//   products are two-pass reductions in a fixed order (deterministic, not
//   the reference's sequential order: results agree to rounding).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "solver.cuh"

namespace loam_gpu {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxVecBlocks = 4 * 148;

// A nested 2x2 operator on the device; a plain Mat is block (0, 0) alone.
struct Op {
  const int64_t* rp[2][2];
  const int32_t* ci[2][2];
  const double* v[2][2];
  int rs[2], cs[2];
};

enum Gate : int { kAlways = 0, kNotDone = 1, kRecheck = 2 };

struct CgState {
  double rz, pq, alpha, beta, rnorm, target, atol;
  int it, done, recheck, status, fail_it, converged, reason;
};

__device__ __forceinline__ bool gated_off(const CgState* st, int gate) {
  if (gate == kAlways || st == nullptr) return false;
  if (gate == kNotDone) return st->done != 0;
  return st->done != 0 || st->recheck == 0;
}

// Block reduction in a fixed order (warp shuffles, then warp 0 over the
// per-warp sums): deterministic for a given launch shape.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double part[kThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) part[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < kThreads / 32 ? part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  return s; // valid in thread 0
}

// y = A x (+ optional partial of dot(w, y) per block)
__global__ void __launch_bounds__(kThreads) k_spmv(const __grid_constant__ Op op, const double* __restrict__ x,
                                                   double* __restrict__ y, const double* __restrict__ w,
                                                   double* partials, const CgState* st, int gate) {
  if (gated_off(st, gate)) return;
  const int n = op.rs[0] + op.rs[1];
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (row < n) {
    const int bi = row < op.rs[0] ? 0 : 1;
    const int r = bi == 0 ? row : row - op.rs[0];
    int col_off = 0;
#pragma unroll
    for (int bj = 0; bj < 2; ++bj) {
      if (op.rp[bi][bj]) {
        const int64_t k1 = __ldg(op.rp[bi][bj] + r + 1);
        const int32_t* ci = op.ci[bi][bj];
        const double* v = op.v[bi][bj];
        for (int64_t k = __ldg(op.rp[bi][bj] + r); k < k1; ++k)
          acc = __dadd_rn(acc, __dmul_rn(__ldg(v + k), __ldg(x + col_off + __ldg(ci + k))));
      }
      col_off += op.cs[bj];
    }
    y[row] = acc;
  }
  if (partials) {
    const double s = block_sum(row < n ? __dmul_rn(w[row], acc) : 0.0);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

// Plain CSR with long rows (C4: 45 entries per dof row): the CTA's 256 rows
// own one contiguous entry range, which is staged through shared memory in
// coalesced chunks; each thread still folds its own row sequentially in
// column order, so y stays bitwise equal to the reference.
constexpr int kChunk = 2048; // entries per staged chunk (24 KB)
__global__ void __launch_bounds__(kThreads) k_spmv_staged(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                          const double* __restrict__ v, int n,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          const double* __restrict__ w, double* partials,
                                                          const CgState* st, int gate) {
  if (gated_off(st, gate)) return;
  __shared__ double sv[kChunk];
  __shared__ int32_t sc[kChunk];
  const int r0 = blockIdx.x * blockDim.x, row = r0 + threadIdx.x;
  const int r1 = min(n, r0 + (int)blockDim.x);
  const int64_t e0 = __ldg(rp + r0), e1 = __ldg(rp + r1);
  int64_t k = row < n ? __ldg(rp + row) : e1;
  const int64_t kend = row < n ? __ldg(rp + row + 1) : e1;
  double acc = 0.0;
  for (int64_t c0 = e0; c0 < e1; c0 += kChunk) {
    const int len = (int)(e1 - c0 < kChunk ? e1 - c0 : kChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
      sv[t] = __ldg(v + c0 + t);
      sc[t] = __ldg(ci + c0 + t);
    }
    __syncthreads();
    const int64_t stop = kend < c0 + len ? kend : c0 + len;
    for (; k < stop; ++k) acc = __dadd_rn(acc, __dmul_rn(sv[k - c0], __ldg(x + sc[k - c0])));
  }
  if (row < n) y[row] = acc;
  if (partials) {
    const double s = block_sum(row < n ? __dmul_rn(w[row], acc) : 0.0);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                  int64_t n, double* partials) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

enum Step : int { kInitRn, kBnorm, kInitRz, kPq, kRn, kTrue, kRz };

// Sum the partials in a fixed order and apply one scalar step of cg_iterate.
__global__ void __launch_bounds__(kThreads) k_finish(const double* partials, int nparts, CgState* st, int step,
                                                     int gate, double rtol) {
  if (gated_off(st, gate)) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s = __dadd_rn(s, partials[i]);
  s = block_sum(s);
  if (threadIdx.x != 0) return;
  switch (step) {
  case kInitRn: st->rnorm = sqrt(s); break;
  case kBnorm: st->target = fmax(rtol * sqrt(s), st->atol); break;
  case kInitRz: st->rz = s; break;
  case kPq: // solver.hpp:140-143
    st->pq = s;
    if (!(s > 0.0)) {
      st->status = 1;
      st->fail_it = st->it + 1;
      st->done = 1;
    } else {
      st->alpha = st->rz / s;
    }
    break;
  case kRn: // solver.hpp:146-148
    st->it += 1;
    st->rnorm = sqrt(s);
    st->recheck = st->rnorm <= st->target ? 1 : 0;
    break;
  case kTrue: // solver.hpp:149-160
    st->rnorm = sqrt(s);
    st->recheck = 0;
    if (st->rnorm <= st->target) {
      st->done = 1;
      st->converged = 1;
      st->reason = st->rnorm <= st->atol ? 1 : 0;
    }
    break;
  case kRz: { // solver.hpp:162-166
    const double rz_next = s;
    st->beta = rz_next / st->rz;
    st->rz = rz_next;
  } break;
  }
}

// x += alpha p; r -= alpha q; partial r.r
__global__ void __launch_bounds__(kThreads) k_axpy2(double* __restrict__ x, double* __restrict__ r,
                                                    const double* __restrict__ p, const double* __restrict__ q,
                                                    int64_t n, const CgState* st, double* partials) {
  if (st->done) return;
  const double a = st->alpha;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(a, q[i]));
    r[i] = ri;
    s = __dadd_rn(s, __dmul_rn(ri, ri));
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// r = b - q; partial r.r
__global__ void __launch_bounds__(kThreads) k_residual(double* __restrict__ r, const double* __restrict__ b,
                                                       const double* __restrict__ q, int64_t n, const CgState* st,
                                                       int gate, double* partials) {
  if (gated_off(st, gate)) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = __dsub_rn(b[i], q[i]);
    r[i] = ri;
    s = __dadd_rn(s, __dmul_rn(ri, ri));
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// z = inv_diag * r (or r); partial r.z; optionally p = z
__global__ void __launch_bounds__(kThreads) k_precond(double* __restrict__ z, const double* __restrict__ r,
                                                      const double* __restrict__ inv, double* __restrict__ p,
                                                      int64_t n, const CgState* st, int gate, double* partials) {
  if (gated_off(st, gate)) return;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = inv ? __dmul_rn(inv[i], r[i]) : r[i];
    z[i] = zi;
    if (p) p[i] = zi;
    s = __dadd_rn(s, __dmul_rn(r[i], zi));
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// p = z + beta p
__global__ void __launch_bounds__(kThreads) k_pupdate(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                                      const CgState* st) {
  if (st->done) return;
  const double b = st->beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(b, p[i]));
}

// Jacobi: inv[off + r] = 1 / A(r, r) (Mat::at: 0 when (r, r) is not in the
// pattern); the first row with a non-positive diagonal is reported
// (solver.hpp:64-76).
__global__ void k_inv_diag(const int64_t* rp, const int32_t* ci, const double* v, int n, double* inv, int* bad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t lo = rp[r], hi = rp[r + 1];
  double d = 0.0;
  while (lo < hi) { // columns are sorted (build_sparsity)
    const int64_t mid = (lo + hi) >> 1;
    const int c = ci[mid];
    if (c == r) {
      d = v[mid];
      break;
    }
    if (c < r) lo = mid + 1;
    else hi = mid;
  }
  if (!(d > 0.0)) atomicMin(bad, r);
  inv[r] = 1.0 / d;
}

int vec_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads), kMaxVecBlocks)); }

Op make_op(const BlockOperator& B) {
  Op op{};
  for (int i = 0; i < 2; ++i) {
    op.rs[i] = B.row_sizes[i];
    op.cs[i] = B.col_sizes[i];
    for (int j = 0; j < 2; ++j) {
      const loam_sparsity_desc* sp = B.sparsity[i][j];
      if (!sp) continue;
      op.rp[i][j] = sp->row_ptr;
      op.ci[i][j] = sp->col_idx;
      op.v[i][j] = B.values[i][j];
    }
  }
  return op;
}

void launch_spmv(const Op& op, const double* x, double* y, const double* w, double* partials, const CgState* st,
                 int gate, cudaStream_t s, int64_t nnz_hint = 0) {
  const int n = op.rs[0] + op.rs[1];
  if (n == 0) return;
  const bool plain = op.rs[1] == 0 && !op.rp[0][1] && !op.rp[1][0] && !op.rp[1][1];
  if (plain && nnz_hint > (int64_t)16 * n) // long rows: coalesced staging
    k_spmv_staged<<<ceil_div(n, kThreads), kThreads, 0, s>>>(op.rp[0][0], op.ci[0][0], op.v[0][0], n, x, y, w,
                                                               partials, st, gate);
  else
    k_spmv<<<ceil_div(n, kThreads), kThreads, 0, s>>>(op, x, y, w, partials, st, gate);
  count_launch();
  LG_LAUNCH_CHECK();
}

void check_layout(const BlockOperator& B) {
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      if (const loam_sparsity_desc* sp = B.sparsity[i][j])
        require(sp->nrows == B.row_sizes[i] && sp->ncols == B.col_sizes[j], LOAM_ERR(DimensionMismatch),
                "block shape inconsistent with layout");
}

int64_t nnz_of(const BlockOperator& B) {
  int64_t z = 0;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      if (B.sparsity[i][j]) z += B.sparsity[i][j]->nnz;
  return z;
}

} // namespace

BlockOperator single_block(const loam_sparsity_desc* sp, const double* values) {
  BlockOperator B{};
  B.sparsity[0][0] = sp;
  B.values[0][0] = values;
  B.row_sizes[0] = sp->nrows;
  B.col_sizes[0] = sp->ncols;
  return B;
}

void spmv(const BlockOperator& B, const double* x, int64_t x_len, double* y, bool nested, cudaStream_t s) {
  if (nested) {
    require(x_len == (int64_t)B.col_sizes[0] + B.col_sizes[1], LOAM_ERR(DimensionMismatch),
            "block spmv operand length != total column count");
    check_layout(B);
  } else {
    require(x_len == B.col_sizes[0], LOAM_ERR(DimensionMismatch), "spmv operand length != matrix column count");
  }
  launch_spmv(make_op(B), x, y, nullptr, nullptr, nullptr, kAlways, s, nnz_of(B));
}

namespace {
// CG runs on a private non-blocking stream (graph capture is not allowed on
// the legacy default stream), ordered after / before the caller's stream.
cudaStream_t solver_stream() {
  static cudaStream_t cs = [] {
    cudaStream_t t;
    LG_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    return t;
  }();
  return cs;
}
struct StreamJoin {
  cudaStream_t user, own;
  cudaEvent_t ev;
  StreamJoin(cudaStream_t u) : user(u), own(solver_stream()) {
    LG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    LG_CUDA(cudaEventRecord(ev, user));
    LG_CUDA(cudaStreamWaitEvent(own, ev, 0));
  }
  ~StreamJoin() {
    cudaEventRecord(ev, own);
    cudaStreamWaitEvent(user, ev, 0);
    cudaEventDestroy(ev);
  }
};
} // namespace

loam_solve_report cg_solve(const BlockOperator& B, const double* b, int64_t b_len, double* x, double rtol,
                           double atol, int maxit, bool jacobi, bool nested, cudaStream_t user_stream) {
  StreamJoin join(user_stream);
  const cudaStream_t s = join.own;
  const int64_t n = (int64_t)B.row_sizes[0] + B.row_sizes[1];
  if (nested) {
    require(n == (int64_t)B.col_sizes[0] + B.col_sizes[1], LOAM_ERR(DimensionMismatch), "cg needs a square operator");
    require(b_len == n, LOAM_ERR(DimensionMismatch), "rhs length != operator size");
    check_layout(B);
  } else {
    require(B.row_sizes[0] == B.col_sizes[0], LOAM_ERR(DimensionMismatch), "cg needs a square matrix");
    require(b_len == n, LOAM_ERR(DimensionMismatch), "rhs length != matrix size");
  }
  const Op op = make_op(B);
  const int vb = vec_blocks(n), sb = std::max(1, ceil_div(n, kThreads));
  DevBuf<double> r(n, s), z(n, s), p(n, s), q(n, s), partials(std::max(vb, sb) + 1, s), inv;
  DevBuf<CgState> st(1, s);
  CgState h{};
  h.atol = atol;
  LG_CUDA(cudaMemcpyAsync(st.get(), &h, sizeof(h), cudaMemcpyHostToDevice, s));
  const double* invp = nullptr;
  if (jacobi) { // solver.hpp:64-76, 190-201
    inv.alloc(n, s);
    DevBuf<int> bad(1, s);
    const int big = INT32_MAX;
    LG_CUDA(cudaMemcpyAsync(bad.get(), &big, sizeof(int), cudaMemcpyHostToDevice, s));
    int64_t off = 0;
    for (int i = 0; i < (nested ? 2 : 1); ++i) {
      const loam_sparsity_desc* sp = B.sparsity[i][i];
      require(sp != nullptr, LOAM_ERR(IndefiniteBreakdown), "jacobi needs the diagonal blocks");
      require(sp->nrows == sp->ncols, LOAM_ERR(DimensionMismatch), "jacobi needs a square matrix");
      if (sp->nrows) {
        k_inv_diag<<<ceil_div(sp->nrows, kThreads), kThreads, 0, s>>>(sp->row_ptr, sp->col_idx, B.values[i][i],
                                                                       sp->nrows, inv.get() + off, bad.get());
        count_launch();
        LG_LAUNCH_CHECK();
      }
      int hb = INT32_MAX;
      LG_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
      require(hb == INT32_MAX, LOAM_ERR(IndefiniteBreakdown),
              "non-positive diagonal entry at row " + std::to_string(hb) + "; matrix is not SPD");
      off += sp->nrows;
    }
    invp = inv.get();
  }
  auto dot_finish = [&](int nparts, int step, int gate) {
    k_finish<<<1, kThreads, 0, s>>>(partials.get(), nparts, st.get(), step, gate, rtol);
    count_launch();
    LG_LAUNCH_CHECK();
  };
  // prologue (solver.hpp:101-132): r = b - A x0, target, early exit, z, p, rz
  const int64_t nnz = nnz_of(B);
  launch_spmv(op, x, q.get(), nullptr, nullptr, nullptr, kAlways, s, nnz);
  k_residual<<<vb, kThreads, 0, s>>>(r.get(), b, q.get(), n, nullptr, kAlways, partials.get());
  count_launch();
  dot_finish(vb, kInitRn, kAlways);
  k_dot<<<vb, kThreads, 0, s>>>(b, b, n, partials.get());
  count_launch();
  dot_finish(vb, kBnorm, kAlways);
  LG_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  loam_solve_report rep{};
  if (h.rnorm <= h.target) {
    rep.converged = 1;
    rep.final_residual_norm = h.rnorm;
    rep.reason = h.rnorm <= atol ? 1 : 0;
    return rep;
  }
  k_precond<<<vb, kThreads, 0, s>>>(z.get(), r.get(), invp, p.get(), n, nullptr, kAlways, partials.get());
  count_launch();
  dot_finish(vb, kInitRz, kAlways);
  // iterations (solver.hpp:134-167) in batches; every kernel is gated, so a
  // batch may run past convergence / breakdown without effect.  A full batch
  // is captured once into a CUDA graph and replayed (10 launches per
  // iteration would otherwise be launch-bound on small systems).
  auto enqueue = [&](int iters) {
    for (int t = 0; t < iters; ++t) {
      launch_spmv(op, p.get(), q.get(), p.get(), partials.get(), st.get(), kNotDone, s, nnz);
      dot_finish(sb, kPq, kNotDone);
      k_axpy2<<<vb, kThreads, 0, s>>>(x, r.get(), p.get(), q.get(), n, st.get(), partials.get());
      count_launch();
      dot_finish(vb, kRn, kNotDone);
      launch_spmv(op, x, q.get(), nullptr, nullptr, st.get(), kRecheck, s, nnz);
      k_residual<<<vb, kThreads, 0, s>>>(r.get(), b, q.get(), n, st.get(), kRecheck, partials.get());
      count_launch();
      dot_finish(vb, kTrue, kRecheck);
      k_precond<<<vb, kThreads, 0, s>>>(z.get(), r.get(), invp, nullptr, n, st.get(), kNotDone, partials.get());
      count_launch();
      dot_finish(vb, kRz, kNotDone);
      k_pupdate<<<vb, kThreads, 0, s>>>(p.get(), z.get(), n, st.get());
      count_launch();
      LG_LAUNCH_CHECK();
    }
  };
  constexpr int kBatch = 16;
  cudaGraphExec_t exec = nullptr;
  int launched = 0;
  while (launched < maxit) {
    const int nb = std::min(kBatch, maxit - launched);
    if (nb == kBatch && maxit >= 2 * kBatch) {
      if (!exec) {
        cudaGraph_t g;
        LG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        enqueue(kBatch);
        LG_CUDA(cudaStreamEndCapture(s, &g));
        LG_CUDA(cudaGraphInstantiate(&exec, g, 0));
        LG_CUDA(cudaGraphDestroy(g));
      }
      LG_CUDA(cudaGraphLaunch(exec, s));
    } else {
      enqueue(nb);
    }
    launched += nb;
    LG_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    if (h.done) break;
  }
  if (exec) cudaGraphExecDestroy(exec);
  require(h.status == 0, LOAM_ERR(IndefiniteBreakdown),
          "p'Ap <= 0 after " + std::to_string(h.fail_it) + " iterations; matrix is not SPD");
  rep.iterations = h.it;
  rep.final_residual_norm = h.rnorm;
  rep.converged = h.converged;
  rep.reason = h.converged ? h.reason : 2;
  return rep;
}

} // namespace loam_gpu
