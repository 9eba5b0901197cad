// mesh.cu -- mesh-side builders on the device.
//
// * P2 node numbering (fem/space.hpp:48-72): vertices keep their ids, the
//   unique edges {min, max} are numbered lexicographically from nv (std::set
//   order = sorted 64-bit keys min << 32 | max), and a cell row is its
//   vertices followed by its edges -- triangles in the reference's order
//   (1,2),(0,2),(0,1) (space.hpp:66-71), tetrahedra in the extension order
//   (2,3),(1,3),(1,2),(0,3),(0,2),(0,1) shared with elements.cuh.  Edge keys
//   are radix-sorted and de-duplicated (CUB), every cell edge finds its id by
//   binary search in the sorted unique list: bit-exact with the reference.
// * Exterior facets (mesh.hpp:48-89 derive_exterior_facets): facet keys are
//   the sorted facet vertices (local facet f = the cell's vertices without
//   vertex f, mesh.hpp:36-42), radix-sorted with their (cell, f) code; a key
//   seen once is exterior, more than twice is NonManifold; the exterior
//   facets are emitted in (cell, local facet) discovery order -- the
//   reference's order -- with their sorted vertices and (cell, f).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <string>

#include "mesh.cuh"

namespace loam_gpu {
namespace {

constexpr int kThreads = 256;

template <class F>
void cub_run(F f, cudaStream_t s) {
  size_t bytes = 0;
  LG_CUDA(f(nullptr, bytes));
  DevBuf<uint8_t> tmp(bytes ? bytes : 1, s);
  LG_CUDA(f(tmp.get(), bytes));
}

__host__ __device__ constexpr int edge_a(int gd, int k) {
  return gd == 2 ? (k == 0 ? 1 : 0) : (k == 0 ? 2 : (k == 1 || k == 2) ? 1 : 0);
}
__host__ __device__ constexpr int edge_b(int gd, int k) {
  return gd == 2 ? (k == 2 ? 1 : 2) : ((k == 0 || k == 1 || k == 3) ? 3 : (k == 2 || k == 4) ? 2 : 1);
}

__device__ __forceinline__ unsigned long long edge_key(int a, int b) {
  const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
  return ((unsigned long long)lo << 32) | hi;
}

__global__ void k_edge_keys(const int32_t* __restrict__ cv, int ncells, int gd, unsigned long long* __restrict__ keys) {
  const int ne = gd == 2 ? 3 : 6, nv = gd + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ncells * ne) return;
  const int64_t c = i / ne;
  const int k = (int)(i - c * ne);
  keys[i] = edge_key(cv[c * nv + edge_a(gd, k)], cv[c * nv + edge_b(gd, k)]);
}

__global__ void k_p2_rows(const int32_t* __restrict__ cv, int ncells, int gd, int nverts,
                          const unsigned long long* __restrict__ uniq, int nuniq, int32_t* __restrict__ cn) {
  const int ne = gd == 2 ? 3 : 6, nv = gd + 1, nn = nv + ne;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  for (int v = 0; v < nv; ++v) cn[c * nn + v] = cv[c * nv + v];
  for (int k = 0; k < ne; ++k) {
    const unsigned long long key = edge_key(cv[c * nv + edge_a(gd, k)], cv[c * nv + edge_b(gd, k)]);
    int lo = 0, hi = nuniq; // lower_bound
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (uniq[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    cn[c * nn + nv + k] = nverts + lo;
  }
}

// facet key: sorted vertices packed (2D: 32-bit halves; 3D: 21 bits each)
__global__ void k_facet_keys(const int32_t* __restrict__ cv, int ncells, int gd, unsigned long long* __restrict__ keys,
                             int32_t* __restrict__ codes) {
  const int nf = gd + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ncells * nf) return;
  const int64_t c = i / nf;
  const int f = (int)(i - c * nf);
  int v[3], m = 0;
  for (int lv = 0; lv <= gd; ++lv)
    if (lv != f) v[m++] = cv[c * nf + lv];
  // sort the gd facet vertices
  for (int a = 0; a < gd; ++a)
    for (int b = a + 1; b < gd; ++b)
      if (v[b] < v[a]) {
        const int t = v[a];
        v[a] = v[b];
        v[b] = t;
      }
  keys[i] = gd == 2 ? (((unsigned long long)v[0] << 32) | (unsigned)v[1])
                    : (((unsigned long long)v[0] << 42) | ((unsigned long long)v[1] << 21) | (unsigned long long)v[2]);
  codes[i] = (int32_t)i;
}

// per sorted position: run length of its key (1 = exterior); flags by code
__global__ void k_facet_flags(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ codes, int64_t n,
                              uint8_t* __restrict__ exterior, int* __restrict__ nonmanifold) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  const bool first = i == 0 || keys[i - 1] != k;
  if (!first) return;
  int64_t e = i + 1;
  while (e < n && keys[e] == k) ++e;
  if (e - i > 2) atomicMin(nonmanifold, codes[i]);
  if (e - i == 1) exterior[codes[i]] = 1;
}

__global__ void k_facet_out(const int32_t* __restrict__ cv, const int32_t* __restrict__ sel, int nsel, int gd,
                            int32_t* __restrict__ fverts, int32_t* __restrict__ fcell) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsel) return;
  const int nf = gd + 1, code = sel[i], c = code / nf, f = code - c * nf;
  int v[3], m = 0;
  for (int lv = 0; lv <= gd; ++lv)
    if (lv != f) v[m++] = cv[(int64_t)c * nf + lv];
  for (int a = 0; a < gd; ++a)
    for (int b = a + 1; b < gd; ++b)
      if (v[b] < v[a]) {
        const int t = v[a];
        v[a] = v[b];
        v[b] = t;
      }
  for (int a = 0; a < gd; ++a) fverts[(int64_t)i * gd + a] = v[a];
  fcell[2 * i] = c;
  fcell[2 * i + 1] = f;
}

__global__ void k_iota(int32_t* __restrict__ x, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}

} // namespace

int p2_cell_node_map_dev(const int32_t* cv, int ncells, int nverts, int gd, int32_t* cn, cudaStream_t s) {
  require(gd == 2 || gd == 3, LOAM_ERR(InvalidArgument), "P2 numbering needs a triangle or tetrahedron mesh");
  require(ncells >= 0 && nverts >= 0, LOAM_ERR(InvalidArgument), "negative mesh size");
  const int ne = gd == 2 ? 3 : 6;
  const int64_t nk = (int64_t)ncells * ne;
  require(nk < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "edge key count exceeds 2^31");
  if (ncells == 0) return nverts;
  DevBuf<unsigned long long> keys(nk, s), sorted(nk, s), uniq(nk, s);
  k_edge_keys<<<ceil_div(nk, kThreads), kThreads, 0, s>>>(cv, ncells, gd, keys.get());
  count_launch();
  LG_LAUNCH_CHECK();
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, keys.get(), sorted.get(), (int)nk, 0, 64, s);
  }, s);
  DevBuf<int> nsel(1, s);
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted.get(), uniq.get(), nsel.get(), (int)nk, s);
  }, s);
  int nu = 0;
  LG_CUDA(cudaMemcpyAsync(&nu, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  require((int64_t)nverts + nu < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "P2 node count exceeds 2^31");
  k_p2_rows<<<ceil_div(ncells, kThreads), kThreads, 0, s>>>(cv, ncells, gd, nverts, uniq.get(), nu, cn);
  count_launch();
  LG_LAUNCH_CHECK();
  return nverts + nu;
}

int exterior_facets_dev(const int32_t* cv, int ncells, int nverts, int gd, int32_t** fverts, int32_t** fcell,
                        cudaStream_t s) {
  require(gd == 2 || gd == 3, LOAM_ERR(InvalidArgument), "exterior facets need a triangle or tetrahedron mesh");
  require(gd == 2 || nverts <= (1 << 21), LOAM_ERR(InvalidArgument),
          "tetrahedral facet keys pack 21-bit vertex ids (at most 2^21 vertices)");
  const int nf = gd + 1;
  const int64_t n = (int64_t)ncells * nf;
  require(n < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "facet count exceeds 2^31");
  *fverts = nullptr;
  *fcell = nullptr;
  if (ncells == 0) return 0;
  DevBuf<unsigned long long> keys(n, s), skeys(n, s);
  DevBuf<int32_t> codes(n, s), scodes(n, s), sel(n, s);
  DevBuf<uint8_t> ext(n, s);
  DevBuf<int> bad(1, s), nsel(1, s);
  LG_CUDA(cudaMemsetAsync(ext.get(), 0, n, s));
  LG_CUDA(cudaMemsetAsync(bad.get(), 0x7f, sizeof(int), s));
  k_facet_keys<<<ceil_div(n, kThreads), kThreads, 0, s>>>(cv, ncells, gd, keys.get(), codes.get());
  count_launch();
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, keys.get(), skeys.get(), codes.get(), scodes.get(), (int)n, 0, 64, s);
  }, s);
  k_facet_flags<<<ceil_div(n, kThreads), kThreads, 0, s>>>(skeys.get(), scodes.get(), n, ext.get(), bad.get());
  k_iota<<<ceil_div(n, kThreads), kThreads, 0, s>>>(codes.get(), n);
  count_launch(2);
  LG_LAUNCH_CHECK();
  int hbad = 0;
  LG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  require(hbad == 0x7f7f7f7f, LOAM_ERR(NonManifold), "facet shared by more than two cells");
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, codes.get(), ext.get(), sel.get(), nsel.get(), (int)n, s);
  }, s);
  int ns = 0;
  LG_CUDA(cudaMemcpyAsync(&ns, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  LG_CUDA(cudaMalloc(reinterpret_cast<void**>(fverts), sizeof(int32_t) * std::max<int64_t>(1, (int64_t)ns * gd)));
  LG_CUDA(cudaMalloc(reinterpret_cast<void**>(fcell), sizeof(int32_t) * std::max<int64_t>(1, 2 * (int64_t)ns)));
  if (ns) {
    k_facet_out<<<ceil_div(ns, kThreads), kThreads, 0, s>>>(cv, sel.get(), ns, gd, *fverts, *fcell);
    count_launch();
    LG_LAUNCH_CHECK();
  }
  LG_CUDA(cudaStreamSynchronize(s));
  return ns;
}

} // namespace loam_gpu
