// solver.cuh -- host interface of solver.cu (SpMV, block SpMV, CG).
#pragma once
#include "common.cuh"

namespace loam_gpu {

// Nested 2x2 operator (solver.hpp:21-28); a null sparsity is a zero block.
struct BlockOperator {
  const loam_sparsity_desc* sparsity[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  const double* values[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int row_sizes[2] = {0, 0};
  int col_sizes[2] = {0, 0};
};

BlockOperator single_block(const loam_sparsity_desc* sp, const double* values);

// y = A x; nested selects block_spmv's checks and messages.
void spmv(const BlockOperator& op, const double* x, int64_t x_len, double* y, bool nested, cudaStream_t s);

loam_solve_report cg_solve(const BlockOperator& op, const double* b, int64_t b_len, double* x, double rtol,
                           double atol, int maxit, bool jacobi, bool nested, cudaStream_t s);

} // namespace loam_gpu
