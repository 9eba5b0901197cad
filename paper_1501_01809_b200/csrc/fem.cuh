// fem.cuh -- host interface of fem.cu (Dirichlet rows, bc.apply, pointwise, norms).
#pragma once
#include "common.cuh"

namespace loam_gpu {

constexpr int kMaxPwDepth = 16;

// apply_dirichlet (fem/assemble.hpp:54-66); rhs == nullptr: apply_dirichlet_rows (:69-79).
// node_values == nullptr: the constant (DirichletBC::value_at, fem/bc.hpp:17-19).
void apply_dirichlet(const loam_sparsity_desc* sp, double* values, double* rhs, const int32_t* nodes, int nn,
                     const double* node_values, double constant, cudaStream_t s);
// DirichletBC::apply (fem/bc.hpp:21-26)
// constant_dev (optional): the constant read from device memory (graph capture)
void bc_apply(double* dat, int set_size, const int32_t* nodes, int nn, const double* node_values, double constant,
              cudaStream_t s, const double* constant_dev = nullptr);
// bench::run_wave's clock on device state (include/loam_gpu.h loam_gpu_wave_clock)
void wave_clock(double* state, double dt, double first_period, int phase, cudaStream_t s);
// pointwise (fem/assemble.hpp:252-314) over n = set_size * dim values; returns the stack depth
int pw_check(const loam_pw_instr* prog, int nprog, int nfields);
void pointwise(double* out, int64_t n, int op, const loam_pw_instr* prog, int nprog, const double* const* fields,
               int nfields, cudaStream_t s);
// fixed-shape reduction into *result_dev
void reduce(const double* x, int64_t n, int kind, double* result_dev, cudaStream_t s);

} // namespace loam_gpu
