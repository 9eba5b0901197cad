// test_kernels.cuh -- device versions of the element kernels the reference's
// own test suite builds as ASTs, registered by the same names so parity tests
// can issue the identical par_loops:
//   test_parloop.cpp:19-42   double_direct, add_one, ones_block
//   test_parloop.cpp:182-200 fill;  :202-237 sum, maxval;  :261-269 weighted_scatter
//   test_parloop.cpp:294-297 sumcells;  :357-373 bump
//   acceptance.cpp:126-236   dw, drw, dinc, gw, iinc, iincv, gsum, gmm
// Each functor reads/writes only its staged buffers (parloop.hpp:253-285).
#pragma once

namespace loam_gpu {
namespace testk {

struct DoubleDirect { // A[0] = 2*B[0]
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] = 2.0 * p[1][0]; }
};
struct AddOne { // V[i] += 1
  static constexpr int STAGE = 3;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int i = 0; i < 3; ++i) p[0][i] += 1.0;
  }
};
struct OnesBlock { // A[i][j] += 1
  static constexpr int STAGE = 9;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int k = 0; k < 9; ++k) p[0][k] += 1.0;
  }
};
struct WeightedScatter { // V[i] += (i+1) * X[0]
  static constexpr int STAGE = 4;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int i = 0; i < 3; ++i) p[0][i] += (i + 1.0) * p[1][0];
  }
};
struct Bump { // V[i] = V[i] + 1
  static constexpr int STAGE = 3;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int i = 0; i < 3; ++i) p[0][i] = p[0][i] + 1.0;
  }
};
struct Fill { // V[i] = 1  (V{2})
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int i = 0; i < 2; ++i) p[0][i] = 1.0;
  }
};
struct Sum { // G[0] += X[0]
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] += p[1][0]; }
};
struct MaxVal { // G[0] = X[0]
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] = p[1][0]; }
};
struct SumCells { // G[0] += X[0]*X[0]
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] += p[1][0] * p[1][0]; }
};
struct Dw { // A = 3 B
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] = 3.0 * p[1][0]; }
};
struct Drw { // A = A + 0.5 B
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] = p[0][0] + 0.5 * p[1][0]; }
};
struct Dinc { // A += B*B
  static constexpr int STAGE = 2;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] += p[1][0] * p[1][0]; }
};
struct Gw { // A = V0 + V1 + V2
  static constexpr int STAGE = 4;
  __device__ static void run(double* const* p, const FormParams&) {
    p[0][0] = p[1][0] + p[1][1] + p[1][2];
  }
};
struct Iincv { // V[i][0] += C ; V[i][1] += 2C   (V{3,2})
  static constexpr int STAGE = 7;
  __device__ static void run(double* const* p, const FormParams&) {
    for (int i = 0; i < 3; ++i) {
      p[0][i * 2 + 0] += p[1][0];
      p[0][i * 2 + 1] += 2.0 * p[1][0];
    }
  }
};
struct Gsum { // G += B * S
  static constexpr int STAGE = 3;
  __device__ static void run(double* const* p, const FormParams&) { p[0][0] += p[1][0] * p[2][0]; }
};
struct Gmm { // LO = B ; HI = B
  static constexpr int STAGE = 3;
  __device__ static void run(double* const* p, const FormParams&) {
    p[0][0] = p[2][0];
    p[1][0] = p[2][0];
  }
};

} // namespace testk
} // namespace loam_gpu
