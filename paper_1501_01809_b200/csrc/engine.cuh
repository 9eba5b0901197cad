// engine.cuh -- host interface of the par_loop engine (engine.cu).
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace loam_gpu {

struct Options {
  int inc_strategy = 0;   // 0 auto, 1 atomics, 2 owner-computes, 3 colouring
  int check_sparsity = 1;
  int locality = 1;
  int test_kernels = 0;   // expose the reference test-suite kernels (add_one, ...)
  int deterministic = 0;  // bitwise-reproducible scatter paths only
};
Options& options();

struct KernelInfo {
  std::string name;
  std::vector<std::string> param_names;
  std::vector<std::vector<int>> extents;
};
const KernelInfo* find_kernel(const std::string& name);
const std::string& kernel_names();

void validate(const loam_kernel_desc* k, int n, uint64_t iter_id, const loam_arg_desc* args,
              int nargs);
void execute(const loam_kernel_desc* k, int n, uint64_t iter_id, const loam_arg_desc* args,
             int nargs, cudaStream_t s);
// fem::assemble_blocks (fem/assemble.hpp:439-448): the loops of a nested block
// matrix in one call; the Taylor-Hood triple runs as one launch (thtile.cuh).
struct LoopDesc {
  const loam_kernel_desc* kernel;
  int n;
  uint64_t iter;
  const loam_arg_desc* args;
  int nargs;
};
void execute_blocks(const LoopDesc* loops, int nloops, cudaStream_t s);
void plan_cache_clear();
// evict every cached plan keyed by an object id (Map / Sparsity destroyed)
void plan_cache_release(uint64_t id);
// bench::run_wave's step (bench.hpp:267-289) fused into the vertex-star
// stiffness action of `args` (b INC, X READ, phi READ; engine.cu k_wave_step).
void wave_step(const loam_kernel_desc* k, int n, uint64_t iter_id, const loam_arg_desc* args, int nargs,
               const double* p_in, const double* phi_in, double* p_out, double* phi_out, const double* pc,
               const uint8_t* bc, double half_dt, double* state, cudaStream_t s);

// Services.
void map_check(const loam_map_desc* m, cudaStream_t s);
void color_iteration(int n, const loam_map_desc* maps, int nmaps, int32_t* colors,
                     int32_t* ncolors, cudaStream_t s);

} // namespace loam_gpu
