// fem.cu -- the device operations around the assembly loop:
// Dirichlet rows on a device CSR, bc.apply on a node Dat, pointwise
// expressions over node Dats, and norms.
//
// Reference:
//   * apply_dirichlet / apply_dirichlet_rows  fem/assemble.hpp:54-81
//     -- zero row r inside its sparsity, diagonal 1, rhs[r] = bc value;
//        MissingDiagonal "diagonal (r, r) outside sparsity" otherwise;
//   * DirichletBC::apply                      fem/bc.hpp:21-26
//   * pointwise(out, op, expr)                fem/assemble.hpp:150-319
//     -- out (=|+=|-=) expr at every node and component, expr a tree of
//        constants, fields and + - * / and negation, evaluated in double
//        with one rounding per operation;
//   * inf_norm                                bench.hpp (wave loop).
// Every result is bitwise equal to the reference: the expression program is
// interpreted with __dadd_rn / __dmul_rn / __ddiv_rn (no FMA contraction) in
// the reference's evaluation order; out + (-v) is written as out - v, which
// IEEE arithmetic makes identical.  The Dirichlet entry points check every
// diagonal BEFORE mutating anything (the reference stops at the first missing
// diagonal after modifying the earlier rows).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "fem.cuh"

namespace loam_gpu {
namespace {

constexpr int kThreads = 256;

// One warp per bc node: position of the diagonal inside row r (-1 if absent).
__global__ void k_find_diag(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ nodes, int nn, int64_t* __restrict__ diag,
                            unsigned long long* __restrict__ first_bad) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nn) return;
  const int r = nodes[w];
  const int64_t b = rp[r], e = rp[r + 1];
  int64_t hit = -1;
  for (int64_t k = b + lane; k < e; k += 32)
    if (ci[k] == r) hit = k;
  for (int o = 16; o; o >>= 1) hit = max(hit, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)hit, o));
  if (lane == 0) {
    diag[w] = hit;
    if (hit < 0) atomicMin(first_bad, (unsigned long long)w);
  }
}

__global__ void k_dirichlet(const int64_t* __restrict__ rp, const int32_t* __restrict__ nodes, int nn,
                            const int64_t* __restrict__ diag, double* __restrict__ values, double* __restrict__ rhs,
                            const double* __restrict__ node_values, double constant) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nn) return;
  const int r = nodes[w];
  const int64_t b = rp[r], e = rp[r + 1], d = diag[w];
  for (int64_t k = b + lane; k < e; k += 32) values[k] = k == d ? 1.0 : 0.0;
  if (lane == 0 && rhs) rhs[r] = node_values ? node_values[r] : constant;
}

__global__ void k_bc_apply(double* __restrict__ dat, const int32_t* __restrict__ nodes, int nn,
                           const double* __restrict__ node_values, double constant,
                           const double* __restrict__ constant_dev) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const int r = nodes[i];
  dat[r] = node_values ? node_values[r] : (constant_dev ? *constant_dev : constant);
}

// bench::run_wave's clock (bench.hpp:222-300) on device state
// {t, bc value, |p|, first-period max, blow-up step, steps}
__global__ void k_wave_clock(double* s, double dt, double first_period, int phase) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (phase == 0) {
    s[1] = sin(10.0 * M_PI * s[0]);
    s[2] = 0.0; // |p| of this step: written by the reduction, or max-folded by the fused step
    return;
  }
  s[0] += dt;
  s[5] += 1.0;
  const double pn = s[2];
  if (s[0] <= first_period) s[3] = fmax(s[3], pn);
  if (s[4] == 0.0 && s[3] > 0.0 && pn > 1e3 * s[3]) s[4] = s[5];
}

// ---- pointwise: postfix program in shared memory, register stack ---------
constexpr int kMaxProgram = 64, kMaxFields = 16;

struct PwLaunch {
  double* out;
  const double* fields[kMaxFields];
  int64_t n;
  int op;   // 0 assign, 1 add, 2 sub
  int nprog;
  loam_pw_instr prog[kMaxProgram];
};

__device__ __forceinline__ double pw_eval(const PwLaunch& L, const loam_pw_instr* prog, int64_t i) {
  double st[kMaxPwDepth];
  int sp = 0;
  for (int q = 0; q < L.nprog; ++q) {
    const loam_pw_instr in = prog[q];
    switch (in.op) {
    case LOAM_PW_CONST: st[sp++] = in.value; break;
    case LOAM_PW_FIELD: st[sp++] = in.field < 0 ? L.out[i] : L.fields[in.field][i]; break;
    case LOAM_PW_NEG: st[sp - 1] = -st[sp - 1]; break;
    default: {
      const double b = st[--sp], a = st[sp - 1];
      double v;
      if (in.op == LOAM_PW_ADD) v = __dadd_rn(a, b);
      else if (in.op == LOAM_PW_SUB) v = __dsub_rn(a, b);
      else if (in.op == LOAM_PW_MUL) v = __dmul_rn(a, b);
      else v = __ddiv_rn(a, b);
      st[sp - 1] = v;
    }
    }
  }
  return st[0];
}

__global__ void __launch_bounds__(kThreads) k_pointwise(const __grid_constant__ PwLaunch L) {
  __shared__ loam_pw_instr prog[kMaxProgram];
  for (int q = threadIdx.x; q < L.nprog; q += blockDim.x) prog[q] = L.prog[q];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = pw_eval(L, prog, i);
    if (L.op == 0) L.out[i] = v;
    else if (L.op == 1) L.out[i] = __dadd_rn(L.out[i], v);
    else L.out[i] = __dsub_rn(L.out[i], v);
  }
}

// ---- reductions: fixed-shape two-pass (deterministic) ---------------------
__device__ __forceinline__ double red_op(int kind, double a, double b) {
  switch (kind) {
  case LOAM_REDUCE_SUM: return a + b;
  case LOAM_REDUCE_MIN: return fmin(a, b);
  default: return fmax(a, b); // MAX and MAX_ABS (inputs already |x|)
  }
}
__device__ __forceinline__ double red_identity(int kind) {
  return kind == LOAM_REDUCE_SUM ? 0.0 : kind == LOAM_REDUCE_MIN ? INFINITY : (kind == LOAM_REDUCE_MAX ? -INFINITY : 0.0);
}

constexpr int kRedBlocks = 4 * 148;

__global__ void __launch_bounds__(kThreads) k_reduce1(const double* __restrict__ x, int64_t n, int kind,
                                                      double* __restrict__ part) {
  double v = red_identity(kind);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = kind == LOAM_REDUCE_MAX_ABS ? fabs(x[i]) : x[i];
    v = red_op(kind, v, xi);
  }
  __shared__ double s[kThreads / 32];
  for (int o = 16; o; o >>= 1) v = red_op(kind, v, __shfl_down_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = s[0];
    for (int w = 1; w < kThreads / 32; ++w) t = red_op(kind, t, s[w]);
    part[blockIdx.x] = t;
  }
}

__global__ void k_reduce2(const double* __restrict__ part, int np, int kind, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = red_identity(kind);
    for (int b = 0; b < np; ++b) t = red_op(kind, t, part[b]);
    *out = t;
  }
}

} // namespace

void apply_dirichlet(const loam_sparsity_desc* sp, double* values, double* rhs, const int32_t* nodes, int nn,
                     const double* node_values, double constant, cudaStream_t s) {
  require(sp != nullptr && values != nullptr, LOAM_ERR(InvalidArgument), "apply_dirichlet without a matrix");
  require(sp->nrows == sp->ncols, LOAM_ERR(ShapeMismatch), "matrix is not square on the bc space");
  require(nn >= 0 && (nn == 0 || nodes != nullptr), LOAM_ERR(InvalidArgument), "bc node list is null");
  if (nn == 0) return;
  // bc nodes must be rows of the matrix (the reference indexes row_offsets()[r])
  std::vector<int32_t> h(nn);
  LG_CUDA(cudaMemcpyAsync(h.data(), nodes, sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  for (int r : h)
    require(r >= 0 && r < sp->nrows, LOAM_ERR(IndexOutOfRange),
            "bc node " + std::to_string(r) + " outside the matrix rows");
  DevBuf<int64_t> diag(nn, s);
  DevBuf<unsigned long long> bad(1, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long), s));
  const int blocks = ceil_div((int64_t)nn * 32, kThreads);
  k_find_diag<<<blocks, kThreads, 0, s>>>(sp->row_ptr, sp->col_idx, nodes, nn, diag.get(), bad.get());
  count_launch();
  LG_LAUNCH_CHECK();
  unsigned long long hb = 0;
  LG_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (hb != ~0ull) {
    const int r = h[hb];
    fail(LOAM_ERR(MissingDiagonal),
         "diagonal (" + std::to_string(r) + ", " + std::to_string(r) + ") outside sparsity");
  }
  k_dirichlet<<<blocks, kThreads, 0, s>>>(sp->row_ptr, nodes, nn, diag.get(), values, rhs, node_values, constant);
  count_launch();
  LG_LAUNCH_CHECK();
}

void bc_apply(double* dat, int set_size, const int32_t* nodes, int nn, const double* node_values, double constant,
              cudaStream_t s, const double* constant_dev) {
  require(nn >= 0 && (nn == 0 || (nodes != nullptr && dat != nullptr)), LOAM_ERR(InvalidArgument),
          "bc apply without data or nodes");
  (void)set_size;
  if (nn == 0) return;
  k_bc_apply<<<ceil_div(nn, kThreads), kThreads, 0, s>>>(dat, nodes, nn, node_values, constant, constant_dev);
  count_launch();
  LG_LAUNCH_CHECK();
}

int pw_check(const loam_pw_instr* prog, int nprog, int nfields) {
  require(prog != nullptr && nprog > 0 && nprog <= kMaxProgram, LOAM_ERR(InvalidArgument),
          "pointwise program must hold 1.." + std::to_string(kMaxProgram) + " instructions");
  int depth = 0, maxd = 0;
  for (int q = 0; q < nprog; ++q) {
    const loam_pw_instr& in = prog[q];
    switch (in.op) {
    case LOAM_PW_CONST: ++depth; break;
    case LOAM_PW_FIELD:
      require(in.field >= -1 && in.field < nfields, LOAM_ERR(InvalidArgument), "pointwise field index out of range");
      ++depth;
      break;
    case LOAM_PW_NEG: require(depth >= 1, LOAM_ERR(InvalidArgument), "pointwise stack underflow"); break;
    case LOAM_PW_ADD: case LOAM_PW_SUB: case LOAM_PW_MUL: case LOAM_PW_DIV:
      require(depth >= 2, LOAM_ERR(InvalidArgument), "pointwise stack underflow");
      --depth;
      break;
    default: fail(LOAM_ERR(InvalidArgument), "unknown pointwise opcode " + std::to_string(in.op));
    }
    maxd = std::max(maxd, depth);
  }
  require(depth == 1, LOAM_ERR(InvalidArgument), "pointwise program must leave exactly one value");
  require(maxd <= kMaxPwDepth, LOAM_ERR(InvalidArgument), "pointwise expression too deep");
  return maxd;
}

void pointwise(double* out, int64_t n, int op, const loam_pw_instr* prog, int nprog, const double* const* fields,
               int nfields, cudaStream_t s) {
  require(out != nullptr || n == 0, LOAM_ERR(InvalidArgument), "pointwise without output");
  require(op >= 0 && op <= 2, LOAM_ERR(InvalidArgument), "pointwise op must be assign, add or sub");
  require(nfields >= 0 && nfields <= kMaxFields, LOAM_ERR(InvalidArgument), "too many pointwise fields");
  pw_check(prog, nprog, nfields);
  if (n == 0) return;
  PwLaunch L{};
  L.out = out;
  L.n = n;
  L.op = op;
  L.nprog = nprog;
  for (int k = 0; k < nfields; ++k) {
    require(fields[k] != nullptr, LOAM_ERR(InvalidArgument), "pointwise field is null");
    L.fields[k] = fields[k];
  }
  for (int q = 0; q < nprog; ++q) L.prog[q] = prog[q];
  const int grid = (int)std::min<int64_t>(ceil_div(n, kThreads), 8 * 148);
  k_pointwise<<<grid, kThreads, 0, s>>>(L);
  count_launch();
  LG_LAUNCH_CHECK();
}

void reduce(const double* x, int64_t n, int kind, double* result_dev, cudaStream_t s) {
  require(kind >= LOAM_REDUCE_SUM && kind <= LOAM_REDUCE_MAX_ABS, LOAM_ERR(InvalidArgument), "unknown reduction");
  require(x != nullptr || n == 0, LOAM_ERR(InvalidArgument), "reduce without data");
  DevBuf<double> part(kRedBlocks, s);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kRedBlocks, ceil_div(n, kThreads)));
  k_reduce1<<<nb, kThreads, 0, s>>>(x, n, kind, part.get());
  k_reduce2<<<1, 32, 0, s>>>(part.get(), nb, kind, result_dev);
  count_launch(2);
  LG_LAUNCH_CHECK();
}

void wave_clock(double* state, double dt, double first_period, int phase, cudaStream_t s) {
  require(state != nullptr && (phase == 0 || phase == 1), LOAM_ERR(InvalidArgument), "wave clock: bad arguments");
  k_wave_clock<<<1, 32, 0, s>>>(state, dt, first_period, phase);
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
