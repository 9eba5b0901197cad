// Design-data microbenchmarks for the par_loop scatter strategy (not product code).
//   1. fp64 RED (atomicAdd, result unused) throughput: random / locality-sorted
//      addresses into arrays of 2 MB (L2), 59 MB (L2) and 1 GB (HBM).
//   2. DFMA throughput.
//   3. read-only, write-only and copy HBM bandwidth.
//   4. empty-kernel launch cost, back-to-back and inside a CUDA graph.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void red_random(double* a, uint64_t n, int per_thread, uint64_t seed, int locality) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int k = 0; k < per_thread; ++k) {
    uint64_t idx;
    if (locality) {  // sorted-ish: neighbouring threads hit nearby addresses (stride ~ 3 entries)
      uint64_t base = (t * 3 + (mix(t * 131 + k + seed) % 8)) ;
      idx = base % n;
    } else {
      idx = mix(t * 977 + k + seed) % n;
    }
    atomicAdd(a + idx, 1.0);
  }
}

__global__ void dfma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.5, d = 0.25, e = 0.125, f = 0.0625, g = 0.03, h = 0.01;
  for (int i = 0; i < iters; ++i) {
    a = fma(a, b, c); d = fma(d, b, e); f = fma(f, b, g); h = fma(h, b, c);
    c = fma(c, b, a); e = fma(e, b, d); g = fma(g, b, f); b = fma(b, 1.0, 1e-30);
  }
  if (a + c + d + e + f + g + h == 1234.5) out[0] = a;
}

__global__ void read_kernel(const double2* __restrict__ a, uint64_t n, double* out) {
  double s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i); s += v.x + v.y;
  }
  if (s == 1234.5) out[0] = s;
}
__global__ void write_kernel(double2* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_double2(0.0, 0.0);
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void empty_kernel() {}
__global__ void flush_kernel(double* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) a[i] += 1.0;
}

int main() {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  double* flush; uint64_t nflush = (512ull << 20) / 8;
  CK(cudaMalloc(&flush, nflush * 8));
  auto do_flush = [&]() { flush_kernel<<<148 * 8, 512>>>(flush, nflush); };

  // ---- 1. fp64 RED throughput
  for (uint64_t bytes : {2ull << 20, 59ull << 20, 1ull << 30}) {
    uint64_t n = bytes / 8;
    double* a; CK(cudaMalloc(&a, bytes)); CK(cudaMemset(a, 0, bytes));
    for (int loc = 0; loc < 2; ++loc) {
      int threads = 148 * 2048, per = 32;
      red_random<<<threads / 256, 256>>>(a, n, per, 1, loc);
      CK(cudaDeviceSynchronize());
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        do_flush();
        CK(cudaEventRecord(e0));
        red_random<<<threads / 256, 256>>>(a, n, per, rep + 7, loc);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      double ops = (double)threads * per;
      printf("RED.F64 array=%6.1f MB locality=%d : %.1f Gatom/s (%.3f ms for %.1f M)\n", bytes / 1048576.0, loc, ops / best / 1e6, best, ops / 1e6);
    }
    CK(cudaFree(a));
  }

  // ---- 2. DFMA
  {
    double* out; CK(cudaMalloc(&out, 8));
    int iters = 4096, blocks = 148 * 8, tpb = 256;
    dfma_kernel<<<blocks, tpb>>>(out, iters); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); dfma_kernel<<<blocks, tpb>>>(out, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
  }

  // ---- 3. bandwidth
  {
    uint64_t bytes = 2ull << 30; uint64_t n2 = bytes / 16;
    double2 *a, *b; double* out;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 0, bytes));
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      read_kernel<<<g, 512>>>(a, n2, out);
      CK(cudaEventRecord(e0)); read_kernel<<<g, 512>>>(a, n2, out); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); printf("read  grid=%d: %.0f GB/s\n", g, bytes / ms / 1e6);
      CK(cudaEventRecord(e0)); write_kernel<<<g, 512>>>(b, n2); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); printf("write grid=%d: %.0f GB/s\n", g, bytes / ms / 1e6);
      CK(cudaEventRecord(e0)); copy_kernel<<<g, 512>>>(a, b, n2); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); printf("copy  grid=%d: %.0f GB/s (r+w)\n", g, 2 * bytes / ms / 1e6);
    }
    CK(cudaEventRecord(e0)); CK(cudaMemsetAsync(b, 0, bytes)); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1)); printf("cudaMemset 2GB: %.0f GB/s\n", bytes / ms / 1e6);
    uint64_t small = 59ull << 20;
    do_flush();
    CK(cudaEventRecord(e0)); CK(cudaMemsetAsync(b, 0, small)); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1)); printf("cudaMemset 59MB: %.2f us\n", ms * 1e3);
    CK(cudaFree(a)); CK(cudaFree(b));
  }

  // ---- 4. launch cost
  {
    for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32>>>();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); for (int i = 0; i < 1000; ++i) empty_kernel<<<148, 128>>>(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1)); printf("empty launch back-to-back: %.2f us\n", ms);
    cudaStream_t s; CK(cudaStreamCreate(&s));
    cudaGraph_t gph; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 100; ++i) empty_kernel<<<148, 128, 0, s>>>();
    CK(cudaStreamEndCapture(s, &gph)); CK(cudaGraphInstantiate(&ge, gph, 0));
    CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s)); for (int i = 0; i < 10; ++i) CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1)); printf("empty launch in graph: %.2f us\n", ms * 1e3 / 1000);
    CK(cudaEventRecord(e0, s)); empty_kernel<<<148, 128, 0, s>>>(); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1)); printf("single empty kernel event-to-event: %.2f us\n", ms * 1e3);
  }
  return 0;
}
