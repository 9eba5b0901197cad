// order.cu -- vertex renumbering on the device: reverse
// Cuthill-McKee (topology.hpp:127-178), the mesh vertex adjacency
// (mesh.hpp:350-362) and the consistent renumbering of coordinates and the
// cell->vertex map (mesh.hpp:364-386).
//
// RCM is a sequential BFS in the reference: a queue, every dequeued vertex
// appends its unvisited neighbours sorted by (degree, index).  The order it
// produces is level-synchronous in disguise: the vertices of BFS level L+1
// appear grouped by their FIRST discoverer -- the level-L vertex with the
// smallest queue position among their level-L neighbours (every level-L
// vertex is dequeued, in position order, before any level-L+1 vertex) -- and
// inside one discoverer by (degree, index).  So one level is
//   expand:  every frontier vertex u (queue position p) atomicMin's p into
//            parent[v] of each unvisited neighbour v; the first touch of v
//            appends it to the candidate list;
//   sort:    one 64-bit radix sort of parent << 32 | rank(v), rank = v's
//            position in the global (degree, index) order (sorted once);
//   emit:    the sorted candidates are the next queue segment, marked visited.
// Seeds follow the reference's next_seed (minimum degree, lowest index among
// the unvisited): a monotone cursor over the (degree, index) order.  Degree-0
// vertices are singleton components at the head of that order and are
// emitted in one step.  The result is bit-identical to the reference,
// including the reference's degree = adjacency-list length (self entries and
// duplicates count, as in the reference).  Input validation follows the
// reference's scan order: the first entry (u, v) in CSR order that is out of
// range (IndexOutOfRange) or has no back entry (AsymmetricAdjacency) is
// reported.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>
#include <string>

#include "mesh.cuh"
#include "plan.cuh"

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

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 16)); }

// First bad entry in CSR order, packed entry << 2 | kind (1 = out of range, 2 = asymmetric).
__global__ void k_rcm_validate(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               unsigned long long* __restrict__ first_bad) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
      const int v = ci[k];
      unsigned kind = 0;
      if (v < 0 || v >= n) {
        kind = 1;
      } else {
        kind = 2;
        for (int64_t q = rp[v]; q < rp[v + 1]; ++q)
          if (ci[q] == u) { kind = 0; break; }
      }
      if (kind) {
        atomicMin(first_bad, ((unsigned long long)k << 2) | kind);
        break;  // later entries of this row cannot come first
      }
    }
  }
}

// key = degree << 32 | index, the reference's next_seed / neighbour order.
__global__ void k_rcm_degkeys(int n, const int64_t* __restrict__ rp, unsigned long long* __restrict__ keys) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    keys[u] = ((unsigned long long)(rp[u + 1] - rp[u]) << 32) | (unsigned)u;
}

__global__ void k_rcm_rank(int n, const unsigned long long* __restrict__ sorted, int32_t* __restrict__ byrank,
                           int32_t* __restrict__ rank, int* __restrict__ nzero) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = (int)(unsigned)sorted[i];
    byrank[i] = v;
    rank[v] = i;
    const bool z = (sorted[i] >> 32) == 0;
    if (z && (i == n - 1 || (sorted[i + 1] >> 32) != 0)) *nzero = i + 1;
  }
}

// Degree-0 vertices: order[i] = byrank[i], visited.
__global__ void k_rcm_isolated(int nz, const int32_t* __restrict__ byrank, int32_t* __restrict__ order,
                               uint8_t* __restrict__ visited) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nz; i += gridDim.x * blockDim.x) {
    order[i] = byrank[i];
    visited[byrank[i]] = 1;
  }
}

// Smallest cursor position >= lo (within [lo, hi)) whose vertex is unvisited.
__global__ void k_rcm_seed(int lo, int hi, const int32_t* __restrict__ byrank, const uint8_t* __restrict__ visited,
                           int* __restrict__ found) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
    if (!visited[byrank[i]]) { atomicMin(found, i); return; }
}

__global__ void k_rcm_start(int pos, const int32_t* __restrict__ byrank, const int* __restrict__ found,
                            int32_t* __restrict__ order, uint8_t* __restrict__ visited) {
  const int v = byrank[*found];
  order[pos] = v;
  visited[v] = 1;
}

// One warp per frontier vertex: neighbours strided over the lanes.
__global__ void k_rcm_expand(int base, int m, const int32_t* __restrict__ order, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, const uint8_t* __restrict__ visited,
                             int32_t* __restrict__ parent, int32_t* __restrict__ touched,
                             int32_t* __restrict__ cand, int* __restrict__ ncand) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < m; w += warps) {
    const int p = base + w, u = order[p];
    for (int64_t k = rp[u] + lane; k < rp[u + 1]; k += 32) {
      const int v = ci[k];
      if (visited[v]) continue;
      atomicMin(&parent[v], p);
      if (atomicExch(&touched[v], 1) == 0) cand[atomicAdd(ncand, 1)] = v;
    }
  }
}

__global__ void k_rcm_keys(int m, const int32_t* __restrict__ cand, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ rank, unsigned long long* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int v = cand[i];
    keys[i] = ((unsigned long long)(unsigned)parent[v] << 32) | (unsigned)rank[v];
  }
}

__global__ void k_rcm_emit(int base, int m, const unsigned long long* __restrict__ keys,
                           const int32_t* __restrict__ byrank, int32_t* __restrict__ order,
                           uint8_t* __restrict__ visited) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int v = byrank[(unsigned)keys[i]];
    order[base + i] = v;
    visited[v] = 1;
  }
}

// Consecutive BFS levels in ONE block while a level's candidates fit a
// shared-memory sort (kLevelCap keys): expand -> keys -> bitonic sort -> emit
// per level with block barriers instead of ~8 launches and a host read.
// Reads of data other threads of this launch wrote go around L1 (ld.cg).
// Stops when the component is exhausted (cur[2] = 0) or a level overflows
// the cap (cur[3] = its candidate count: cand / parent / touched are set,
// the host sorts and emits that level).  cur = {pos, base, m, overflow}.
constexpr int kLevelCap = 4096, kLevelThreads = 1024;

__global__ void __launch_bounds__(kLevelThreads) k_rcm_levels(const int64_t* __restrict__ rp,
                                                              const int32_t* __restrict__ ci, int32_t* order,
                                                              uint8_t* visited, int32_t* parent, int32_t* touched,
                                                              int32_t* cand, const int32_t* __restrict__ rank,
                                                              const int32_t* __restrict__ byrank, int* cur) {
  __shared__ unsigned long long sk[kLevelCap];
  __shared__ int s_cnt;
  const int tid = threadIdx.x;
  int pos = cur[0], base = cur[1], m = cur[2];
  while (m > 0 && m <= kLevelCap / 2) { // wide frontiers go back to the grid-wide path
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int w = tid; w < m; w += kLevelThreads) { // a thread per frontier vertex: one latency chain per level
      const int p = base + w, u = __ldcg(order + p);
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        const int v = ci[k];
        if (__ldcg(visited + v)) continue;
        atomicMin(&parent[v], p);
        if (atomicExch(&touched[v], 1) == 0) cand[atomicAdd(&s_cnt, 1)] = v;
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt == 0 || cnt > kLevelCap) {
      if (tid == 0) {
        cur[0] = pos;
        cur[1] = base;
        cur[2] = cnt == 0 ? 0 : m;
        cur[3] = cnt;
      }
      return;
    }
    int P = 1;
    while (P < cnt) P <<= 1;
    for (int i = tid; i < P; i += kLevelThreads) {
      if (i < cnt) {
        const int v = __ldcg(cand + i);
        sk[i] = ((unsigned long long)(unsigned)__ldcg(parent + v) << 32) | (unsigned)rank[v];
      } else {
        sk[i] = ~0ull;
      }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < P; i += kLevelThreads) {
          const int x = i ^ j;
          if (x > i) {
            const unsigned long long a = sk[i], b = sk[x];
            if ((a > b) == ((i & k) == 0)) {
              sk[i] = b;
              sk[x] = a;
            }
          }
        }
        __syncthreads();
      }
    for (int i = tid; i < cnt; i += kLevelThreads) {
      const int v = byrank[(unsigned)sk[i]];
      order[pos + i] = v;
      visited[v] = 1;
    }
    __syncthreads();
    base = pos;
    m = cnt;
    pos += cnt;
  }
  if (tid == 0) { // exhausted (m == 0) or a wide frontier (m > cap / 2): no level pending
    cur[0] = pos;
    cur[1] = base;
    cur[2] = m;
    cur[3] = -1;
  }
}

__global__ void k_reverse(int n, const int32_t* __restrict__ in, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[n - 1 - i] = in[i];
}

int bits_for(unsigned x) {
  int b = 1;
  while (b < 32 && (x >> b)) ++b;
  return b;
}

// ---- vertex adjacency: the cell-vertex sparsity without its diagonal -------
__global__ void k_offdiag_count(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                int64_t* __restrict__ cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) c += ci[k] != r;
    cnt[r] = c;
    if (r == 0) cnt[n] = 0;
  }
}

__global__ void k_offdiag_fill(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const int64_t* __restrict__ orp, int32_t* __restrict__ oci) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int64_t o = orp[r];
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
      if (ci[k] != r) oci[o++] = ci[k];
  }
}

// ---- renumbering ----------------------------------------------------------
__global__ void k_inverse_perm(int n, const int32_t* __restrict__ perm, int32_t* __restrict__ new_of,
                               int* __restrict__ bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = perm[i];
    if (o < 0 || o >= n || atomicExch(&new_of[o], i) != -1) *bad = 1;
  }
}

__global__ void k_permute_coords(int n, int gd, const int32_t* __restrict__ perm, const double* __restrict__ src,
                                 double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n * gd;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / gd;
    dst[i] = src[(int64_t)perm[v] * gd + (i - v * gd)];
  }
}

__global__ void k_renumber_map(int64_t len, int n, const int32_t* __restrict__ new_of, const int32_t* __restrict__ cv,
                               int32_t* __restrict__ out, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = cv[i];
    if (v < 0 || v >= n) { *bad = 1; continue; }
    out[i] = new_of[v];
  }
}

} // namespace

__global__ void k_rcm_rowptr_check(int n, const int64_t* __restrict__ rp, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && rp[0] != 0) atomicOr(bad, 1);
  if (i < n && rp[i + 1] < rp[i]) atomicOr(bad, 1);
}

void rcm_order_dev(int n, const int64_t* rp, const int32_t* ci, int32_t* out, cudaStream_t s) {
  require(n >= 0, LOAM_ERR(InvalidArgument), "negative vertex count");
  if (n == 0) return;
  // the list structure first: row_ptr must start at 0 and never
  // decrease, or the validation below would read outside col_idx and fault
  {
    DevBuf<int> shape(1, s);
    LG_CUDA(cudaMemsetAsync(shape.get(), 0, sizeof(int), s));
    k_rcm_rowptr_check<<<grid_for(n), kThreads, 0, s>>>(n, rp, shape.get());
    count_launch();
    LG_CUDA(cudaGetLastError());
    int hshape = 0;
    LG_CUDA(cudaMemcpyAsync(&hshape, shape.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    require(hshape == 0, LOAM_ERR(InvalidArgument), "adjacency list count != n (row offsets not a CSR of n lists)");
  }
  DevBuf<unsigned long long> bad(1, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long), s));
  k_rcm_validate<<<grid_for(n), kThreads, 0, s>>>(n, rp, ci, bad.get());
  count_launch();
  LG_CUDA(cudaGetLastError());
  unsigned long long hbad = 0;
  LG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(hbad), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    const int64_t k = (int64_t)(hbad >> 2);
    if ((hbad & 3) == 1) throw Error(LOAM_ERR(IndexOutOfRange), "adjacency index out of range");
    int64_t u = 0;  // row of entry k, for the message
    std::vector<int64_t> hrp(n + 1);
    LG_CUDA(cudaMemcpy(hrp.data(), rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    while (u + 1 <= n && hrp[u + 1] <= k) ++u;
    int32_t v = 0;
    LG_CUDA(cudaMemcpy(&v, ci + k, sizeof(v), cudaMemcpyDeviceToHost));
    throw Error(LOAM_ERR(AsymmetricAdjacency),
                "edge " + std::to_string(u) + "-" + std::to_string(v) + " not symmetric");
  }

  // (degree, index) order and ranks.
  DevBuf<unsigned long long> keys(n, s), skeys(n, s);
  DevBuf<int32_t> byrank(n, s), rank(n, s), parent(n, s), touched(n, s), cand(n, s), order(n, s);
  DevBuf<uint8_t> visited(n, s);
  DevBuf<int> cnt(2, s);  // [0] candidate count / isolated count, [1] seed cursor
  k_rcm_degkeys<<<grid_for(n), kThreads, 0, s>>>(n, rp, keys.get());
  count_launch();
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, keys.get(), skeys.get(), n, 0, 64, s);
  }, s);
  LG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int) * 2, s));
  LG_CUDA(cudaMemsetAsync(visited.get(), 0, n, s));
  LG_CUDA(cudaMemsetAsync(touched.get(), 0, sizeof(int32_t) * n, s));
  LG_CUDA(cudaMemsetAsync(parent.get(), 0x7f, sizeof(int32_t) * n, s));
  k_rcm_rank<<<grid_for(n), kThreads, 0, s>>>(n, skeys.get(), byrank.get(), rank.get(), cnt.get());
  count_launch();
  int nz = 0;
  LG_CUDA(cudaMemcpyAsync(&nz, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (nz) {
    k_rcm_isolated<<<grid_for(nz), kThreads, 0, s>>>(nz, byrank.get(), order.get(), visited.get());
    count_launch();
  }

  const int rank_bits = bits_for((unsigned)n);
  size_t sort_bytes = 0;
  LG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, keys.get(), skeys.get(), n, 0, 64, s));
  DevBuf<uint8_t> sort_tmp(sort_bytes ? sort_bytes : 1, s);
  int pos = nz, cursor = nz;
  static const bool use_levels = !std::getenv("LOAM_GPU_RCM_NO_BLOCK");
  DevBuf<int> lcur(4, s);
  int hc[2];
  while (pos < n) {
    // next seed: the first unvisited vertex of the (degree, index) order
    int found = n;
    for (int lo = cursor; found == n && lo < n; lo += 4096) {
      const int hi = std::min(n, lo + 4096);
      LG_CUDA(cudaMemcpyAsync(cnt.get() + 1, &n, sizeof(int), cudaMemcpyHostToDevice, s));
      k_rcm_seed<<<grid_for(hi - lo), kThreads, 0, s>>>(lo, hi, byrank.get(), visited.get(), cnt.get() + 1);
      count_launch();
      LG_CUDA(cudaMemcpyAsync(&found, cnt.get() + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
    }
    require(found < n, LOAM_ERR(InvalidArgument), "rcm: no seed left before every vertex was placed");
    cursor = found + 1;
    k_rcm_start<<<1, 1, 0, s>>>(pos, byrank.get(), cnt.get() + 1, order.get(), visited.get());
    count_launch();
    int base = pos, m = 1;
    ++pos;
    while (m > 0) {
      if (use_levels && m <= kLevelCap / 2) { // as many levels as fit one block's sort, in one launch
        int hcur[4] = {pos, base, m, 0};
        LG_CUDA(cudaMemcpyAsync(lcur.get(), hcur, sizeof(hcur), cudaMemcpyHostToDevice, s));
        k_rcm_levels<<<1, kLevelThreads, 0, s>>>(rp, ci, order.get(), visited.get(), parent.get(), touched.get(),
                                                cand.get(), rank.get(), byrank.get(), lcur.get());
        count_launch();
        LG_CUDA(cudaMemcpyAsync(hcur, lcur.get(), sizeof(hcur), cudaMemcpyDeviceToHost, s));
        LG_CUDA(cudaStreamSynchronize(s));
        pos = hcur[0];
        base = hcur[1];
        m = hcur[2];
        if (m == 0) break;
        if (hcur[3] < 0) continue; // frontier too wide for the block: the grid-wide path takes the next level
        // this level overflowed the block sort: its candidates are listed
        const int mc = hcur[3];
        k_rcm_keys<<<grid_for(mc), kThreads, 0, s>>>(mc, cand.get(), parent.get(), rank.get(), keys.get());
        count_launch();
        size_t b = sort_bytes;
        LG_CUDA(cub::DeviceRadixSort::SortKeys(sort_tmp.get(), b, keys.get(), skeys.get(), mc, 0, 32 + rank_bits, s));
        k_rcm_emit<<<grid_for(mc), kThreads, 0, s>>>(pos, mc, skeys.get(), byrank.get(), order.get(), visited.get());
        count_launch();
        base = pos;
        m = mc;
        pos += mc;
        continue;
      }
      LG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int), s));
      k_rcm_expand<<<grid_for((int64_t)m * 32), kThreads, 0, s>>>(base, m, order.get(), rp, ci, visited.get(),
                                                                  parent.get(), touched.get(), cand.get(),
                                                                  cnt.get());
      count_launch();
      LG_CUDA(cudaMemcpyAsync(hc, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      LG_CUDA(cudaStreamSynchronize(s));
      const int mc = hc[0];
      if (mc == 0) break;
      k_rcm_keys<<<grid_for(mc), kThreads, 0, s>>>(mc, cand.get(), parent.get(), rank.get(), keys.get());
      count_launch();
      size_t b = sort_bytes;
      LG_CUDA(cub::DeviceRadixSort::SortKeys(sort_tmp.get(), b, keys.get(), skeys.get(), mc, 0, 32 + rank_bits, s));
      k_rcm_emit<<<grid_for(mc), kThreads, 0, s>>>(pos, mc, skeys.get(), byrank.get(), order.get(), visited.get());
      count_launch();
      base = pos;
      m = mc;
      pos += mc;
    }
  }
  k_reverse<<<grid_for(n), kThreads, 0, s>>>(n, order.get(), out);
  count_launch();
  LG_CUDA(cudaGetLastError());
  LG_CUDA(cudaStreamSynchronize(s));
}

int64_t vertex_adjacency_dev(const int32_t* cv, int ncells, int nverts, int gd, int64_t** rp_out, int32_t** ci_out,
                             cudaStream_t s) {
  MapView m{cv, ncells, gd + 1, nverts};
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  int64_t nnz = 0;
  build_sparsity_dev(m, m, 1, 1, &rp, &ci, &nnz, s);
  DevBuf<int64_t> cnt(nverts + 1, s);
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(rp_out), sizeof(int64_t) * (nverts + 1), s));
  if (nverts) {
    k_offdiag_count<<<grid_for(nverts), kThreads, 0, s>>>(nverts, rp, ci, cnt.get());
    count_launch();
  } else {
    LG_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int64_t), s));
  }
  cub_run([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt.get(), *rp_out, nverts + 1, s);
  }, s);
  int64_t total = 0;
  LG_CUDA(cudaMemcpyAsync(&total, *rp_out + nverts, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ci_out), sizeof(int32_t) * (total ? total : 1), s));
  if (nverts) {
    k_offdiag_fill<<<grid_for(nverts), kThreads, 0, s>>>(nverts, rp, ci, *rp_out, *ci_out);
    count_launch();
  }
  LG_CUDA(cudaGetLastError());
  LG_CUDA(cudaFreeAsync(rp, s));
  LG_CUDA(cudaFreeAsync(ci, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return total;
}

void renumber_vertices_dev(int nverts, int gd, const double* coords, int ncells, const int32_t* cv,
                           const int32_t* perm, double* coords_out, int32_t* cv_out, cudaStream_t s) {
  if (nverts == 0 && ncells == 0) return;
  DevBuf<int32_t> new_of(nverts ? nverts : 1, s);
  DevBuf<int> bad(2, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int) * 2, s));
  LG_CUDA(cudaMemsetAsync(new_of.get(), 0xff, sizeof(int32_t) * (nverts ? nverts : 1), s));
  if (nverts) {
    k_inverse_perm<<<grid_for(nverts), kThreads, 0, s>>>(nverts, perm, new_of.get(), bad.get());
    count_launch();
  }
  int hb[2];
  LG_CUDA(cudaMemcpyAsync(hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  require(hb[0] == 0, LOAM_ERR(InvalidArgument), "perm is not a permutation of the vertices");
  if (coords && coords_out && nverts) {
    k_permute_coords<<<grid_for((int64_t)nverts * gd), kThreads, 0, s>>>(nverts, gd, perm, coords, coords_out);
    count_launch();
  }
  const int64_t len = (int64_t)ncells * (gd + 1);
  if (len) {
    k_renumber_map<<<grid_for(len), kThreads, 0, s>>>(len, nverts, new_of.get(), cv, cv_out, bad.get() + 1);
    count_launch();
  }
  LG_CUDA(cudaMemcpyAsync(hb + 1, bad.get() + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  require(hb[1] == 0, LOAM_ERR(IndexOutOfRange), "cell vertex out of range");
}

} // namespace loam_gpu
