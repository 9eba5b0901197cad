// dmma_probe.cu -- is there FP64 tensor-core (DMMA) throughput on a B200 beyond
// the FP64 CUDA-core (DFMA) pipe?  Design data for DESIGN.md section 5 (the
// north star asks that FP64 tensor cores be used "only where it really is" a
// contraction, evidenced by counters): DFMA alone, DMMA alone (m8n8k4 and
// m16n8k8), and both issued together from the same warps / from different warps
// of one SM.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kIters = 4096;
constexpr int kChains = 8; // independent accumulators per thread

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1688(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// NF DFMAs and NM DMMAs (m8n8k4) per loop iteration, compile-time (no predication);
// NM < 0: |NM| m16n8k8 DMMAs
template <int NF, int NM>
__global__ void __launch_bounds__(256) probe(double* out, double seed) {
  const int tid = threadIdx.x + blockIdx.x * blockDim.x;
  double x = seed + tid * 1e-9, y = 1.0 - 1e-9 * tid;
  double f[kChains], c0[kChains], c1[kChains];
  double c4[kChains / 2][4];
#pragma unroll
  for (int k = 0; k < kChains; ++k) {
    f[k] = k;
    c0[k] = k;
    c1[k] = -k;
  }
#pragma unroll
  for (int k = 0; k < kChains / 2; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) c4[k][q] = k + q;
  const double a4[4] = {x, y, x + 1, y - 1}, b2[2] = {y, x};
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k % kChains] = fma(f[k % kChains], x, y);
    if constexpr (NM > 0) {
#pragma unroll
      for (int k = 0; k < NM; ++k) dmma884(c0[k % kChains], c1[k % kChains], x, y);
    } else if constexpr (NM < 0) {
#pragma unroll
      for (int k = 0; k < -NM; ++k) dmma1688(c4[k % (kChains / 2)], a4, b2);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += f[k] + c0[k] + c1[k];
#pragma unroll
  for (int k = 0; k < kChains / 2; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c4[k][q];
  if (s == 12345.678) out[tid] = s;
}

template <int NF, int NM>
int run(const char* name, double* out, int blocks, int threads) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0));
    probe<NF, NM><<<blocks, threads>>>(out, 0.5);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0 && ms < best) best = ms;
  }
  const double warps = double(blocks) * threads / 32;
  // flops per warp instruction: DFMA 64, m8n8k4 512, m16n8k8 2048
  const double fma_fl = warps * kIters * NF * 64.0;
  const double mma_fl = warps * kIters * (NM > 0 ? NM * 512.0 : -NM * 2048.0);
  printf("%-44s %8.3f ms  DFMA %6.2f TFLOP/s  DMMA %6.2f TFLOP/s  total %6.2f\n", name, best, fma_fl / best / 1e9,
         mma_fl / best / 1e9, (fma_fl + mma_fl) / best / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount, blocks = sms * 8, threads = 256;
  double* out;
  CK(cudaMalloc(&out, sizeof(double) * blocks * threads));
  printf("# %s, %d SMs; %d blocks x %d threads (64 warps / SM), %d iterations, %d independent chains per thread\n", p.name,
         sms, blocks, threads, kIters, kChains);
  printf("# per iteration: NF DFMA + NM DMMA warp instructions; if the two shared no hardware, a mixed row would take\n");
  printf("# the max of its parts' times, if they share the FP64 units, the sum\n");
  if (run<64, 0>("64 DFMA", out, blocks, threads)) return 1;
  if (run<0, 8>("8 DMMA m8n8k4", out, blocks, threads)) return 1;
  if (run<0, -2>("2 DMMA m16n8k8", out, blocks, threads)) return 1;
  if (run<64, 8>("64 DFMA + 8 DMMA m8n8k4 (equal flops)", out, blocks, threads)) return 1;
  if (run<32, 8>("32 DFMA + 8 DMMA m8n8k4", out, blocks, threads)) return 1;
  if (run<64, 4>("64 DFMA + 4 DMMA m8n8k4", out, blocks, threads)) return 1;
  if (run<64, -2>("64 DFMA + 2 DMMA m16n8k8 (equal flops)", out, blocks, threads)) return 1;
  return 0;
}
