#include <atomic>
// plan.cu -- device-side plan construction (see plan.cuh).
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "plan.cuh"

namespace loam_gpu {

namespace {

constexpr int kTPB = 256;

template <class F>
void cub_call(F f, cudaStream_t s) {
  size_t bytes = 0;
  LG_CUDA(f(nullptr, bytes));
  DevBuf<uint8_t> tmp(bytes ? bytes : 1, s);
  LG_CUDA(f(tmp.get(), bytes));
}

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= maxval) ++b;
  return b;
}

__global__ void k_min_key(const int32_t* __restrict__ m, int n, int arity, int32_t* keys,
                          int32_t* iota) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int k = m[(int64_t)e * arity];
  for (int a = 1; a < arity; ++a) k = min(k, m[(int64_t)e * arity + a]);
  keys[e] = k;
  iota[e] = e;
}

__global__ void k_gather_rows(const int32_t* __restrict__ m, const int32_t* __restrict__ perm,
                              int n, int arity, int32_t* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * arity) return;
  int64_t p = t / arity;
  int a = (int)(t - p * arity);
  out[t] = m[(int64_t)perm[p] * arity + a];
}

__global__ void k_iota(int32_t* v, int64_t n) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) v[t] = (int32_t)t;
}

__global__ void k_count(const int32_t* __restrict__ keys, int64_t n, int32_t* counts) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) atomicAdd(counts + keys[t], 1);
}

// Blockedness of a dof-expanded pattern: for node row r, rows r*rd+d have the
// same length L = cd * Ln and col_idx[start + t*cd + c] = node_t*cd + c.
__global__ void k_check_blocked(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                int nrows_node, int rd, int cd, int* bad) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows_node) return;
  const int64_t s0 = rp[(int64_t)r * rd], l0 = rp[(int64_t)r * rd + 1] - s0;
  if (l0 % cd) { *bad = 1; return; }
  for (int d = 0; d < rd; ++d) {
    const int64_t s = rp[(int64_t)r * rd + d], l = rp[(int64_t)r * rd + d + 1] - s;
    if (l != l0) { *bad = 1; return; }
    for (int64_t t = 0; t < l; t += cd) {
      const int node = ci[s + t] / cd;
      if (ci[s + t] != node * cd) { *bad = 1; return; }
      for (int c = 1; c < cd; ++c)
        if (ci[s + t + c] != node * cd + c) { *bad = 1; return; }
    }
  }
}

__global__ void k_ranks(const int32_t* __restrict__ pairs, int64_t npairs, int nrn, int ncn,
                        const int32_t* __restrict__ srows, const int32_t* __restrict__ scols,
                        const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int rd,
                        int cd, uint8_t* ranks, unsigned long long* err) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  const int32_t k = pairs[p];
  const int s = k / nrn;
  const int r = srows[k];
  const int64_t start = rp[(int64_t)r * rd];
  const int len = (int)((rp[(int64_t)r * rd + 1] - start) / cd);
  for (int j = 0; j < ncn; ++j) {
    const int c = scols[(int64_t)s * ncn + j];
    int lo = 0, hi = len;
    while (lo < hi) { // lower_bound over node columns (data.hpp:129-136)
      int mid = (lo + hi) >> 1;
      if (ci[start + (int64_t)mid * cd] / cd < c) lo = mid + 1;
      else hi = mid;
    }
    if (lo == len || ci[start + (int64_t)lo * cd] / cd != c) {
      // first offender: (dof row, dof col) as Mat::addto reports it
      atomicCAS(err, 0ull, (1ull << 63) | ((unsigned long long)(r * rd) << 32) | (unsigned)(c * cd));
      return;
    }
    if (lo > 255) {
      atomicCAS(err, 0ull, (1ull << 62));
      return;
    }
    ranks[p * ncn + j] = (uint8_t)lo;
  }
}

__global__ void k_node_starts(const int64_t* __restrict__ rp, int nrows_node, int rd, int64_t* out) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= nrows_node) out[r] = rp[(int64_t)r * rd];
}

// ---- sparsity
__global__ void k_emit_keys(const int32_t* __restrict__ rm, int ar_r, const int32_t* __restrict__ cm,
                            int ar_c, int n, unsigned long long* keys) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)ar_r * ar_c;
  if (t >= (int64_t)n * per) return;
  const int64_t e = t / per;
  const int rem = (int)(t - e * per);
  const int a = rem / ar_c, b = rem - a * ar_c;
  keys[t] = ((unsigned long long)(uint32_t)rm[e * ar_r + a] << 32) | (uint32_t)cm[e * ar_c + b];
}

__global__ void k_key_rows(const unsigned long long* __restrict__ keys, int64_t n, int32_t* counts) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) atomicAdd(counts + (int)(keys[t] >> 32), 1);
}

__global__ void k_expand_rowptr(const int64_t* __restrict__ node_off, int nrows_node, int rd, int cd,
                                int64_t* rp) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > (int64_t)nrows_node * rd) return;
  if (t == (int64_t)nrows_node * rd) { rp[t] = node_off[nrows_node] * rd * cd; return; }
  const int r = (int)(t / rd), d = (int)(t - (int64_t)r * rd);
  const int64_t len = node_off[r + 1] - node_off[r];
  rp[t] = node_off[r] * rd * cd + d * len * cd;
}

__global__ void k_fill_cols(const unsigned long long* __restrict__ ukeys, int64_t nu,
                            const int64_t* __restrict__ node_off, const int64_t* __restrict__ rp,
                            int rd, int cd, int32_t* ci) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nu) return;
  const unsigned long long k = ukeys[t];
  const int r = (int)(k >> 32), c = (int)(uint32_t)k;
  const int64_t pos = t - node_off[r];
  for (int d = 0; d < rd; ++d) {
    const int64_t base = rp[(int64_t)r * rd + d] + pos * cd;
    for (int x = 0; x < cd; ++x) ci[base + x] = c * cd + x;
  }
}

// ---- colouring (Jones-Plassmann, priority = ascending index == greedy order)
struct InvMap {
  const int32_t* ptr;  // [target+1]
  const int32_t* ent;  // pair codes f*arity+k incident to target, ascending f
  const int32_t* map;
  int arity;
};

constexpr int kMaxColorWords = 4; // 256 colours

template <int NM>
__global__ void k_jp_round(int n, InvMap m0, InvMap m1, InvMap m2, InvMap m3, int32_t* colors,
                           int* remaining, int* overflow) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  volatile int32_t* col = colors;
  if (col[e] >= 0) return;
  unsigned long long mask[kMaxColorWords] = {0, 0, 0, 0};
  const InvMap ms[4] = {m0, m1, m2, m3};
#pragma unroll
  for (int mi = 0; mi < NM; ++mi) {
    const InvMap& m = ms[mi];
    for (int k = 0; k < m.arity; ++k) {
      const int t = m.map[(int64_t)e * m.arity + k];
      for (int q = m.ptr[t]; q < m.ptr[t + 1]; ++q) {
        const int f = m.ent[q] / m.arity;
        if (f >= e) break; // only earlier entities constrain e (topology.hpp:152-159)
        const int c = col[f];
        if (c < 0) { atomicAdd(remaining, 1); return; } // not decided yet: next round
        mask[c >> 6] |= 1ull << (c & 63);
      }
    }
  }
  int c = 0;
  while (c < 64 * kMaxColorWords && (mask[c >> 6] >> (c & 63) & 1ull)) ++c;
  if (c >= 64 * kMaxColorWords) { *overflow = 1; return; }
  col[e] = c;
}

__global__ void k_node_pattern(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int nrows_node,
                               int rd, int cd, int64_t* nptr, int32_t* nadj) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nrows_node) return;
  const int64_t s0 = rp[(int64_t)r * rd];
  nptr[r] = s0 / ((int64_t)rd * cd);
  if (r == nrows_node) return;
  const int64_t len = (rp[(int64_t)r * rd + 1] - s0) / cd;
  const int64_t o = s0 / ((int64_t)rd * cd);
  for (int64_t k = 0; k < len; ++k) nadj[o + k] = ci[s0 + k * cd] / cd;
}

// Records of the neighbour-list plan (P1 forms): the cell is rotated so the
// owning row is local vertex 0, and the record packs the in-row ranks of the
// other vertices (i+1)%N .. (i+N-1)%N, `bits` each from bit 0.  The row's own
// rank is a per-row constant recomputed by the kernel.
template <class Rec>
__global__ void k_records(const int32_t* __restrict__ pairs, int64_t npairs, int nrn,
                          const int32_t* __restrict__ srows, const int32_t* __restrict__ pptr, int nrows_node,
                          const int64_t* __restrict__ nptr, const int32_t* __restrict__ nadj, int bits, Rec* recs,
                          unsigned long long* err) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows_node) return;
  const int64_t a0 = nptr[r];
  const int len = (int)(nptr[r + 1] - a0);
  if (len > (1 << bits)) { atomicCAS(err, 0ull, 1ull << 62); return; }
  for (int p = pptr[r]; p < pptr[r + 1]; ++p) {
    const int k = pairs[p];
    const int s = k / nrn, i = k - s * nrn;
    uint32_t rec = 0;
    for (int j = 0; j < nrn; ++j) {
      const int c = srows[(int64_t)s * nrn + (i + j) % nrn];
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nadj[a0 + mid] < c) lo = mid + 1;
        else hi = mid;
      }
      if (lo == len || nadj[a0 + lo] != c) {
        atomicCAS(err, 0ull, (1ull << 63) | ((unsigned long long)(uint32_t)r << 32) | (uint32_t)c);
        return;
      }
      if (j > 0) rec |= (uint32_t)lo << ((j - 1) * bits);
    }
    recs[p] = (Rec)rec;
  }
}

} // namespace

__global__ void k_i64_to_i32(const int64_t* __restrict__ a, int64_t n, int32_t* b) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) b[t] = (int32_t)a[t];
}

bool build_nbr(NbrPlan& np, const int32_t* sorted_rows, int ncells, int nrn, int nrows_node,
               const CsrView& csr, int tile_rows, int tile_seg, int tile_slots, int tile_runs,
               cudaStream_t s) {
  np.nrows_node = nrows_node;
  np.nrn = nrn;
  // ---- node-level pattern, as plan-owned int32 arrays padded by 16 bytes
  CsrView node = csr;
  int64_t* built_rp = nullptr;
  int32_t* built_ci = nullptr;
  if (!csr.row_ptr) { // Dat INC: the pattern of (map, map)
    MapView m{sorted_rows, ncells, nrn, nrows_node};
    int64_t nnz = 0;
    build_sparsity_dev(m, m, 1, 1, &built_rp, &built_ci, &nnz, s);
    node = CsrView{built_rp, built_ci, nrows_node, nrows_node, nnz, 1, 1};
  }
  np.rd = node.rd;
  np.cd = node.cd;
  const int64_t nn = node.nnz / ((int64_t)node.rd * node.cd);
  require(nn < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "node pattern exceeds 2^31 entries");
  np.nptr.alloc(nrows_node + 1 + 4, s);
  DevBuf<int32_t> nadj(nn + 4, s);
  LG_CUDA(cudaMemsetAsync(np.nptr.get(), 0, np.nptr.bytes(), s));
  LG_CUDA(cudaMemsetAsync(nadj.get(), 0, nadj.bytes(), s));
  if (node.rd == 1 && node.cd == 1) {
    k_i64_to_i32<<<ceil_div(nrows_node + 1, kTPB), kTPB, 0, s>>>(node.row_ptr, nrows_node + 1, np.nptr.get());
    count_launch();
    if (nn) LG_CUDA(cudaMemcpyAsync(nadj.get(), node.col_idx, sizeof(int32_t) * nn, cudaMemcpyDeviceToDevice, s));
  } else {
    DevBuf<int64_t> tmp(nrows_node + 1, s);
    k_node_pattern<<<ceil_div(nrows_node + 1, kTPB), kTPB, 0, s>>>(node.row_ptr, node.col_idx, nrows_node, node.rd,
                                                                   node.cd, tmp.get(), nadj.get());
    k_i64_to_i32<<<ceil_div(nrows_node + 1, kTPB), kTPB, 0, s>>>(tmp.get(), nrows_node + 1, np.nptr.get());
    count_launch(2);
  }
  LG_LAUNCH_CHECK();
  if (built_rp) {
    LG_CUDA(cudaFreeAsync(built_rp, s));
    LG_CUDA(cudaFreeAsync(built_ci, s));
  }
  // ---- pairs grouped by row, packed records
  plan_tick("nbr: node pattern", s);
  PairPlan pp;
  build_pairs(sorted_rows, ncells, nrn, nrows_node, pp, s);
  plan_tick("nbr: pairs", s);
  std::vector<int32_t> h(nrows_node + 1), hp(nrows_node + 1);
  LG_CUDA(cudaMemcpyAsync(h.data(), np.nptr.get(), sizeof(int32_t) * (nrows_node + 1), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaMemcpyAsync(hp.data(), pp.ptr.get(), sizeof(int32_t) * (nrows_node + 1), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  int64_t maxlen = 1;
  for (int r = 0; r < nrows_node; ++r) maxlen = std::max<int64_t>(maxlen, h[r + 1] - h[r]);
  np.bits = bits_for(maxlen - 1);
  np.max_len = (int)maxlen;
  const int rbits = (nrn - 1) * np.bits;
  if (rbits > 32) return false;
  np.rec_bytes = rbits <= 8 ? 1 : (rbits <= 16 ? 2 : 4);
  np.recs.alloc(pp.npairs * np.rec_bytes + 16, s);
  LG_CUDA(cudaMemsetAsync(np.recs.get(), 0, np.recs.bytes(), s));
  DevBuf<unsigned long long> err(1, s);
  LG_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(unsigned long long), s));
  DevBuf<int64_t> nptr64(nrows_node + 1, s);
  {
    std::vector<int64_t> h64(h.begin(), h.end());
    LG_CUDA(cudaMemcpyAsync(nptr64.get(), h64.data(), sizeof(int64_t) * (nrows_node + 1), cudaMemcpyHostToDevice, s));
    if (pp.npairs) {
      if (np.rec_bytes == 1)
        k_records<uint8_t><<<ceil_div(nrows_node, kTPB), kTPB, 0, s>>>(
            pp.pairs.get(), pp.npairs, nrn, sorted_rows, pp.ptr.get(), nrows_node, nptr64.get(), nadj.get(),
            np.bits, reinterpret_cast<uint8_t*>(np.recs.get()), err.get());
      else if (np.rec_bytes == 2)
        k_records<uint16_t><<<ceil_div(nrows_node, kTPB), kTPB, 0, s>>>(
            pp.pairs.get(), pp.npairs, nrn, sorted_rows, pp.ptr.get(), nrows_node, nptr64.get(), nadj.get(),
            np.bits, reinterpret_cast<uint16_t*>(np.recs.get()), err.get());
      else
        k_records<uint32_t><<<ceil_div(nrows_node, kTPB), kTPB, 0, s>>>(
            pp.pairs.get(), pp.npairs, nrn, sorted_rows, pp.ptr.get(), nrows_node, nptr64.get(), nadj.get(),
            np.bits, reinterpret_cast<uint32_t*>(np.recs.get()), err.get());
      count_launch();
      LG_LAUNCH_CHECK();
    }
    unsigned long long herr = 0;
    LG_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(herr), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    if (herr >> 63) {
      const int row = (int)((herr >> 32) & 0x7fffffff), col = (int)(uint32_t)herr;
      fail(LOAM_ERR(OutsideSparsity), "mat: entry (" + std::to_string(row * node.rd) + ", " +
                                          std::to_string(col * node.cd) + ") outside sparsity");
    }
    if (herr >> 62) return false;
  }
  plan_tick("nbr: records", s);
  np.pptr.alloc(nrows_node + 1 + 4, s);
  LG_CUDA(cudaMemsetAsync(np.pptr.get(), 0, np.pptr.bytes(), s));
  LG_CUDA(cudaMemcpyAsync(np.pptr.get(), pp.ptr.get(), sizeof(int32_t) * (nrows_node + 1), cudaMemcpyDeviceToDevice, s));
  // ---- CTA tiles with contiguous vertex windows
  std::vector<int32_t> hadj(nn);
  if (nn) LG_CUDA(cudaMemcpyAsync(hadj.data(), nadj.get(), sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  const int64_t w = (int64_t)node.rd * node.cd;
  const int nv = nrows_node; // P1: row nodes are the coordinate vertices
  constexpr int kGap = 8;    // merge runs separated by <= kGap unused vertices
  std::vector<uint16_t> hw(nn + 8, 0);
  std::vector<uint8_t> hs(nrows_node + 16, 0);
  // chunks of whole tile-row blocks tiled on all host cores (window slots and
  // self ranks written in place; tiles concatenated, run offsets shifted)
  struct TileChunk {
    bool ok = true, has_empty_row = false;
    std::vector<int32_t> tiles, runs;
    std::vector<std::pair<int, int>> tile_of_rows;
    int max_rows = 0, max_adj = 0, max_pairs = 0, max_seg = 0, max_slots = 0, max_runs = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nrows_node, tile_rows, [&](int t, int64_t cb0, int64_t cb1) {
  TileChunk& O = tch[t];
  std::vector<int32_t>& tiles = O.tiles;
  std::vector<int32_t>& runs = O.runs;
  std::vector<std::pair<int, int>>& tile_of_rows = O.tile_of_rows;
  bool& has_empty_row = O.has_empty_row;
  std::vector<int32_t> verts;
  std::vector<std::pair<int, int>> rr;
  auto make_runs = [&](int r0, int r1) { // runs of the tile's vertices; returns slot count
    verts.assign(hadj.begin() + h[r0], hadj.begin() + h[r1]);
    std::sort(verts.begin(), verts.end());
    verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
    rr.clear();
    int slots = 0;
    for (int v : verts) {
      const int lo = v & ~1, hi = std::min(nv, (v + 2) & ~1);
      if (!rr.empty() && lo <= rr.back().second + kGap) rr.back().second = std::max(rr.back().second, hi);
      else rr.emplace_back(lo, hi);
    }
    for (auto& x : rr) slots += x.second - x.first;
    return slots;
  };
  int r0 = (int)cb0;
  const int rend = (int)cb1;
  while (r0 < rend) {
    int r1 = std::min(rend, r0 + tile_rows);
    while (r1 > r0 + 1 && (int64_t)(h[r1] - h[r0]) * w > tile_seg) --r1;
    int slots = make_runs(r0, r1);
    while (r1 > r0 + 1 && (slots > tile_slots || (int)rr.size() > tile_runs)) {
      r1 = r0 + (r1 - r0) / 2;
      slots = make_runs(r0, r1);
    }
    if (slots > tile_slots || (int)rr.size() > tile_runs || (int64_t)(h[r1] - h[r0]) * w > tile_seg) {
      O.ok = false; // a single row does not fit: use the pair-list path
      return;
    }
    // window slots: run k occupies [base_k, base_k + hi - lo)
    std::vector<int> base(rr.size());
    int acc = 0;
    for (size_t k = 0; k < rr.size(); ++k) {
      base[k] = acc;
      acc += rr[k].second - rr[k].first;
    }
    for (int64_t a = h[r0]; a < h[r1]; ++a) {
      const int v = hadj[a];
      size_t k = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
      hw[a] = (uint16_t)(base[k] + v - rr[k].first);
    }
    tile_of_rows.push_back({r0, r1});
    for (int r = r0; r < r1; ++r) {
      int q = 0;
      while (h[r] + q < h[r + 1] && hadj[h[r] + q] != r) ++q;
      // a row node no cell of the loop touches (a sub-mesh loop) has an empty
      // pattern row and no pairs: its owner writes nothing but its zero
      require(h[r] + q < h[r + 1] || (h[r] == h[r + 1] && hp[r] == hp[r + 1]), LOAM_ERR(InvalidArgument),
              "row node missing from its own pattern row");
      if (h[r] == h[r + 1]) has_empty_row = true;
      hs[r] = (uint8_t)q;
    }
    tiles.insert(tiles.end(), {r0, r1, h[r0], h[r1], hp[r0], hp[r1], (int)runs.size() / 2, (int)rr.size()});
    for (auto& x : rr) runs.insert(runs.end(), {x.first, x.second});
    O.max_rows = std::max(O.max_rows, r1 - r0);
    O.max_adj = std::max(O.max_adj, h[r1] - h[r0]);
    O.max_pairs = std::max(O.max_pairs, hp[r1] - hp[r0]);
    O.max_seg = std::max<int>(O.max_seg, (int)((h[r1] - h[r0]) * w));
    O.max_slots = std::max(O.max_slots, slots);
    O.max_runs = std::max(O.max_runs, (int)rr.size());
    r0 = r1;
  }
  });
  std::vector<int32_t> tiles, runs;
  std::vector<std::pair<int, int>> tile_of_rows;
  bool has_empty_row = false;
  for (int t = 0; t < ntch; ++t) {
    TileChunk& O = tch[t];
    if (!O.ok) return false;
    const int rshift = (int)(runs.size() / 2);
    for (size_t q = 0; q < O.tiles.size(); q += 8) O.tiles[q + 6] += rshift;
    tiles.insert(tiles.end(), O.tiles.begin(), O.tiles.end());
    runs.insert(runs.end(), O.runs.begin(), O.runs.end());
    tile_of_rows.insert(tile_of_rows.end(), O.tile_of_rows.begin(), O.tile_of_rows.end());
    has_empty_row = has_empty_row || O.has_empty_row;
    np.max_rows = std::max(np.max_rows, O.max_rows);
    np.max_adj = std::max(np.max_adj, O.max_adj);
    np.max_pairs = std::max(np.max_pairs, O.max_pairs);
    np.max_seg = std::max(np.max_seg, O.max_seg);
    np.max_slots = std::max(np.max_slots, O.max_slots);
    np.max_runs = std::max(np.max_runs, O.max_runs);
  }
  tch.clear();
  plan_tick("nbr: host tiles", s);
  np.ntiles = (int)tiles.size() / 8;
  np.tiles.alloc(tiles.size() ? tiles.size() : 8, s);
  np.runs.alloc(runs.size() ? runs.size() : 2, s);
  np.widx.alloc(hw.size(), s);
  np.selfr.alloc(hs.size(), s);
  // ---- ring mode for P1 triangles (nrn == 3): chain each row's cells along the
  // vertex ring / fan so a kernel fetches one new vertex per cell and completes
  // every off-diagonal entry after two consecutive cells (no read-modify-write)
  np.ring = false;
  if (nrn == 3 && maxlen <= 8 && np.max_slots <= 4095 && pp.npairs && !has_empty_row) {
    std::vector<int32_t> hpairs(pp.npairs), hrows((size_t)ncells * nrn);
    // pp.ptr was moved into np.pptr above; pair codes are still in pp.pairs
    LG_CUDA(cudaMemcpyAsync(hpairs.data(), pp.pairs.get(), sizeof(int32_t) * pp.npairs, cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaMemcpyAsync(hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size(), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> rptr(nrows_node + 1);
    for (int r = 0; r <= nrows_node; ++r) rptr[r] = hp[r] + r;
    std::vector<uint16_t> rrec((size_t)rptr[nrows_node] + 8, 0);
    std::vector<uint32_t> rinfo(nrows_node + 4, 0);
    // rows are independent: chunks of rows on all host cores
    std::atomic<bool> all_ok{true};
    parallel_chunks(nrows_node, 1, [&](int, int64_t rb0, int64_t rb1) {
      bool ok = true;
      std::vector<int> av, bv;
      std::vector<char> used;
      for (int r = (int)rb0; r < (int)rb1 && ok; ++r) {
        auto slot_of = [&](int v) { // window slot of vertex v in this row's tile
          for (int64_t a = h[r]; a < h[r + 1]; ++a)
            if (hadj[a] == v) return (int)hw[a];
          return -1;
        };
        auto rank_of = [&](int v) {
          for (int64_t a = h[r]; a < h[r + 1]; ++a)
            if (hadj[a] == v) return (int)(a - h[r]);
          return -1;
        };
        const int P = hp[r + 1] - hp[r];
        av.resize(P);
        bv.resize(P);
        for (int q = 0; q < P; ++q) {
          const int code = hpairs[hp[r] + q];
          const int c = code / 3, i = code - 3 * c;
          av[q] = hrows[(size_t)c * 3 + (i + 1) % 3];
          bv[q] = hrows[(size_t)c * 3 + (i + 2) % 3];
        }
        const int self_slot = slot_of(r), self_rank = rank_of(r);
        rinfo[r] = (uint32_t)self_slot | ((uint32_t)self_rank << 16);
        if (P == 0) {
          rrec[rptr[r]] = (uint16_t)((self_slot << 4) | self_rank);
          continue;
        }
        // degree of every neighbour in the star; open fans start at a degree-1 vertex
        int start = av[0], ones = 0;
        for (int q = 0; q < P && ok; ++q)
          for (int v : {av[q], bv[q]}) {
            int deg = 0;
            for (int u = 0; u < P; ++u) deg += (av[u] == v) + (bv[u] == v);
            if (deg > 2 || v == r) ok = false;
            if (deg == 1) { ++ones; start = v; }
          }
        if (!ok || (ones != 0 && ones != 2)) { ok = false; break; }
        used.assign(P, 0);
        int v = start;
        rrec[rptr[r]] = (uint16_t)((slot_of(v) << 4) | rank_of(v));
        for (int k = 0; k < P; ++k) {
          int q = 0;
          while (q < P && (used[q] || (av[q] != v && bv[q] != v))) ++q;
          if (q == P) { ok = false; break; } // star is not a single fan / ring
          used[q] = 1;
          v = av[q] == v ? bv[q] : av[q];
          rrec[rptr[r] + 1 + k] = (uint16_t)((slot_of(v) << 4) | rank_of(v));
        }
        if (ok && ones == 0 && v != start) ok = false; // a ring must close
      }
      if (!ok) all_ok = false;
    });
    (void)tile_of_rows;
    if (all_ok) {
      np.ring = true;
      np.rptr.alloc(rptr.size() + 4, s);
      np.rrecs.alloc(rrec.size(), s);
      np.rowinfo.alloc(rinfo.size(), s);
      LG_CUDA(cudaMemsetAsync(np.rptr.get(), 0, np.rptr.bytes(), s));
      LG_CUDA(cudaMemcpyAsync(np.rptr.get(), rptr.data(), sizeof(int32_t) * rptr.size(), cudaMemcpyHostToDevice, s));
      LG_CUDA(cudaMemcpyAsync(np.rrecs.get(), rrec.data(), sizeof(uint16_t) * rrec.size(), cudaMemcpyHostToDevice, s));
      LG_CUDA(cudaMemcpyAsync(np.rowinfo.get(), rinfo.data(), sizeof(uint32_t) * rinfo.size(), cudaMemcpyHostToDevice, s));
      // ring tiles: 16 ints -- the 8 tile fields (P0/P1 in ring-record units)
      // followed by the first kRingInlineRuns window runs, so a producer gets a
      // tile's meta and runs from one 64-byte line with no dependent load
      const size_t nt = tiles.size() / 8;
      std::vector<int32_t> rt(nt * 16, 0);
      for (size_t t = 0; t < nt; ++t) {
        for (int q = 0; q < 8; ++q) rt[16 * t + q] = tiles[8 * t + q];
        rt[16 * t + 4] = rptr[tiles[8 * t + 0]];
        rt[16 * t + 5] = rptr[tiles[8 * t + 1]];
        const int ro = tiles[8 * t + 6], rc = tiles[8 * t + 7];
        for (int q = 0; q < std::min(rc, kRingInlineRuns); ++q) {
          rt[16 * t + 8 + 2 * q] = runs[2 * (ro + q)];
          rt[16 * t + 9 + 2 * q] = runs[2 * (ro + q) + 1];
        }
      }
      np.rtiles.alloc(rt.size() ? rt.size() : 16, s);
      if (!rt.empty())
        LG_CUDA(cudaMemcpyAsync(np.rtiles.get(), rt.data(), sizeof(int32_t) * rt.size(), cudaMemcpyHostToDevice, s));
      np.max_pairs += np.max_rows; // ring records per tile: pairs + one head per row
    }
  }
  if (!tiles.empty())
    LG_CUDA(cudaMemcpyAsync(np.tiles.get(), tiles.data(), sizeof(int32_t) * tiles.size(), cudaMemcpyHostToDevice, s));
  if (!runs.empty())
    LG_CUDA(cudaMemcpyAsync(np.runs.get(), runs.data(), sizeof(int32_t) * runs.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(np.widx.get(), hw.data(), sizeof(uint16_t) * hw.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(np.selfr.get(), hs.data(), hs.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

// Local node permutation induced by a vertex permutation sigma (new vertex
// index of old vertex v is sigma[v]) on Lagrange P1 / P2 simplices; returns
// newpos[old local node].  P2 local edges follow elements.cuh / space.hpp.
namespace {
const int kTriEdge[3][2] = {{1, 2}, {0, 2}, {0, 1}};
const int kTetEdge[6][2] = {{2, 3}, {1, 3}, {1, 2}, {0, 3}, {0, 2}, {0, 1}};
} // namespace
void induced(int gd, int nloc, const int* sigma, int* newpos) {
  const int nv = gd + 1;
  for (int v = 0; v < nv && v < nloc; ++v) newpos[v] = sigma[v];
  if (nloc == nv) return;
  const int ne = gd == 2 ? 3 : 6;
  const int (*E)[2] = gd == 2 ? kTriEdge : kTetEdge;
  for (int e = 0; e < ne; ++e) {
    int a = sigma[E[e][0]], b = sigma[E[e][1]];
    if (a > b) std::swap(a, b);
    for (int f = 0; f < ne; ++f)
      if (E[f][0] == a && E[f][1] == b) newpos[nv + e] = nv + f;
  }
}
// Vertex permutation that makes row-space local node i canonical.
// Returns the canonical local index (0 or nv).
int canonical_sigma(int gd, int nrn, int i, int* sigma) {
  const int nv = gd + 1;
  if (i < nv) { // vertex i -> 0, the others keep their relative order
    int k = 1;
    for (int v = 0; v < nv; ++v) sigma[v] = v == i ? 0 : k++;
    return 0;
  }
  const int (*E)[2] = gd == 2 ? kTriEdge : kTetEdge;
  const int a = E[i - nv][0], b = E[i - nv][1];
  // edge (a,b) -> the first local edge: (1,2) on triangles, (2,3) on tets
  int k = 0;
  const int ta = gd == 2 ? 1 : 2, tb = gd == 2 ? 2 : 3;
  for (int v = 0; v < nv; ++v) sigma[v] = v == a ? ta : (v == b ? tb : k++);
  (void)nrn;
  return nv;
}

bool build_ptile(PTilePlan& out, const PTileSpec& sp, int ncells, int nrows_node, const int32_t* sorted_rows,
                 const int32_t* sorted_cols, const int32_t* sorted_x, int nverts, const int32_t* sorted_coeff,
                 int ncoeff_nodes, const PairPlan& pp, const CsrView& csr, cudaStream_t s) {
  const int gd = sp.gd, nv = gd + 1, nrn = sp.nrn, ncn = sp.ncn, ncf = sp.ncoeff;
  const int64_t np = pp.npairs;
  // ---- host copies
  auto hrows = host_array<int32_t>((size_t)ncells * nrn), hx = host_array<int32_t>((size_t)ncells * nv),
       hpairs = host_array<int32_t>(np), hp = host_array<int32_t>(nrows_node + 1);
  std::vector<int32_t> hcols, hcf;
  hvec<uint8_t> hrank;
  std::vector<int64_t> hn(nrows_node + 1, 0), rp;
  if (ncn) hrank.resize((size_t)np * ncn);
  if (ncf) hcf.resize((size_t)ncells * ncf);
  if (ncn) rp.resize((size_t)nrows_node * csr.rd + 1);
  parallel_d2h({{hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size()},
                {hx.data(), sorted_x, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * (size_t)np},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * (size_t)(nrows_node + 1)},
                {hrank.data(), pp.ranks.get(), hrank.size()},
                {hcf.data(), sorted_coeff, sizeof(int32_t) * hcf.size()},
                {rp.data(), csr.row_ptr, sizeof(int64_t) * rp.size()}},
               s);
  if (ncn) // node-level pattern offsets from the (blocked) CSR
    for (int r = 0; r <= nrows_node; ++r) hn[r] = rp[(size_t)r * csr.rd] / ((int64_t)csr.rd * csr.cd);
  (void)sorted_cols;
  const int W = sp.rd * sp.cd;
  // ---- record layout
  const int off_cf = 2 * nv, off_rk = off_cf + 2 * ncf, off_ci = off_rk + ncn;
  const int rb = (off_ci + 1 + 3) & ~3;
  out.rec_bytes = rb;
  out.nrows_node = nrows_node;
  // ---- tiles with coordinate / coefficient windows
  constexpr int kGap = 8;
  auto make_runs = [&](std::vector<int>& ids, int limit, std::vector<std::pair<int, int>>& rr) {
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    rr.clear();
    int slots = 0;
    for (int v : ids) {
      const int lo = v & ~1, hi = std::min(limit, (v + 2) & ~1);
      if (!rr.empty() && lo <= rr.back().second + kGap) rr.back().second = std::max(rr.back().second, hi);
      else rr.emplace_back(lo, hi);
    }
    for (auto& x : rr) slots += x.second - x.first;
    return slots;
  };
  std::vector<uint8_t> recs((size_t)np * rb + 64, 0);
  auto slot_in = [](const std::vector<std::pair<int, int>>& R, const std::vector<int>& base, int v) {
    size_t k = std::upper_bound(R.begin(), R.end(), std::make_pair(v, INT32_MAX)) - R.begin() - 1;
    return base[k] + v - R[k].first;
  };
  // chunks of whole tile-row blocks tiled on all host cores (records are
  // written in place; tiles concatenated with their run offsets shifted)
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs, cruns;
    int max_rows = 0, max_pairs = 0, max_seg = 0, max_slots = 0, max_cslots = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nrows_node, sp.tile_rows, [&](int t, int64_t cb0, int64_t cb1) {
  TileChunk& O = tch[t];
  std::vector<int32_t>& tiles = O.tiles;
  std::vector<int32_t>& runs = O.runs;
  std::vector<int32_t>& cruns = O.cruns;
  std::vector<int> vid, cid;
  std::vector<std::pair<int, int>> rr, cr;
  // generation stamps (calloc'd: only the pages a chunk touches map)
  struct Stamps {
    int* p;
    explicit Stamps(size_t n) : p(static_cast<int*>(std::calloc(n + 1, sizeof(int)))) {
      if (!p) throw std::bad_alloc();
    }
    ~Stamps() { std::free(p); }
  } cstamp(ncells), vstamp(nverts), fstamp(ncf ? ncoeff_nodes : 0);
  int gen = 0;
  int r0 = (int)cb0;
  const int rend = (int)cb1;
  while (r0 < rend) {
    int r1 = std::min(rend, r0 + sp.tile_rows);
    auto fits = [&](int a, int b, int& slots, int& cslots) {
      if (ncn && (hn[b] - hn[a]) * W > sp.tile_seg) return false;
      if (hp[b] - hp[a] > sp.tile_pairs) return false;
      ++gen;
      vid.clear();
      cid.clear();
      for (int p = hp[a]; p < hp[b]; ++p) { // distinct cells' distinct vertices / coefficient nodes
        const int c = hpairs[p] / nrn;
        if (cstamp.p[c] == gen) continue;
        cstamp.p[c] = gen;
        for (int v = 0; v < nv; ++v) {
          const int x = hx[(size_t)c * nv + v];
          if (vstamp.p[x] != gen) {
            vstamp.p[x] = gen;
            vid.push_back(x);
          }
        }
        for (int q = 0; q < ncf; ++q) {
          const int x = hcf[(size_t)c * ncf + q];
          if (fstamp.p[x] != gen) {
            fstamp.p[x] = gen;
            cid.push_back(x);
          }
        }
      }
      slots = make_runs(vid, nverts, rr);
      cslots = ncf ? make_runs(cid, ncoeff_nodes, cr) : 0;
      return slots <= sp.tile_slots && (int)rr.size() <= sp.tile_runs && cslots <= sp.tile_slots &&
             (int)cr.size() <= sp.tile_runs;
    };
    int slots = 0, cslots = 0;
    while (!fits(r0, r1, slots, cslots)) {
      if (r1 == r0 + 1) {
        O.ok = false;
        return;
      }
      r1 = r0 + (r1 - r0) / 2;
    }
    std::vector<int> base(rr.size()), cbase(cr.size());
    for (size_t k = 0, acc = 0; k < rr.size(); ++k) {
      base[k] = (int)acc;
      acc += rr[k].second - rr[k].first;
    }
    for (size_t k = 0, acc = 0; k < cr.size(); ++k) {
      cbase[k] = (int)acc;
      acc += cr[k].second - cr[k].first;
    }
    for (int r = r0; r < r1; ++r)
      for (int p = hp[r]; p < hp[r + 1]; ++p) {
        const int code = hpairs[p], c = code / nrn, i = code - c * nrn;
        int sigma[4], inv[4], rowpos[10], colpos[10];
        const int ci = canonical_sigma(gd, nrn, i, sigma);
        for (int v = 0; v < nv; ++v) inv[sigma[v]] = v;
        uint8_t* rec = &recs[(size_t)p * rb];
        for (int k = 0; k < nv; ++k) { // permuted vertex k = original vertex inv[k]
          const uint16_t sl = (uint16_t)slot_in(rr, base, hx[(size_t)c * nv + inv[k]]);
          memcpy(rec + 2 * k, &sl, 2);
        }
        if (ncf) {
          induced(gd, ncf, sigma, colpos);
          for (int q = 0; q < ncf; ++q) {
            const uint16_t sl = (uint16_t)slot_in(cr, cbase, hcf[(size_t)c * ncf + q]);
            memcpy(rec + off_cf + 2 * colpos[q], &sl, 2);
          }
        }
        if (ncn) {
          induced(gd, ncn, sigma, colpos);
          for (int j = 0; j < ncn; ++j) rec[off_rk + colpos[j]] = hrank[(size_t)p * ncn + j];
        }
        (void)rowpos;
        rec[off_ci] = (uint8_t)ci;
      }
    // thread group per row: the G lanes of a row take interleaved pairs, so a
    // tile of few long rows (P2 vertex rows: 24 cells) still fills the CTA
    int maxp = 0, G = 1;
    for (int r = r0; r < r1; ++r) maxp = std::max(maxp, hp[r + 1] - hp[r]);
    while (G < 8 && (r1 - r0) * G * 2 <= sp.tile_rows && G * 4 <= maxp) G *= 2;
    tiles.insert(tiles.end(), {r0, r1, (int)hn[r0], (int)hn[r1], hp[r0], hp[r1], (int)runs.size() / 2,
                               (int)rr.size(), (int)cruns.size() / 2, (int)cr.size(), G, 0});
    for (auto& x : rr) runs.insert(runs.end(), {x.first, x.second});
    for (auto& x : cr) cruns.insert(cruns.end(), {x.first, x.second});
    O.max_rows = std::max(O.max_rows, r1 - r0);
    O.max_pairs = std::max(O.max_pairs, hp[r1] - hp[r0]);
    O.max_seg = std::max<int>(O.max_seg, (int)((hn[r1] - hn[r0]) * W));
    O.max_slots = std::max(O.max_slots, slots);
    O.max_cslots = std::max(O.max_cslots, cslots);
    r0 = r1;
  }
  });
  std::vector<int32_t> tiles, runs, cruns;
  for (int t = 0; t < ntch; ++t) {
    TileChunk& O = tch[t];
    if (!O.ok) return false;
    const int rshift = (int)(runs.size() / 2), cshift = (int)(cruns.size() / 2);
    for (size_t q = 0; q < O.tiles.size(); q += 12) {
      O.tiles[q + 6] += rshift;
      O.tiles[q + 8] += cshift;
    }
    tiles.insert(tiles.end(), O.tiles.begin(), O.tiles.end());
    runs.insert(runs.end(), O.runs.begin(), O.runs.end());
    cruns.insert(cruns.end(), O.cruns.begin(), O.cruns.end());
    out.max_rows = std::max(out.max_rows, O.max_rows);
    out.max_pairs = std::max(out.max_pairs, O.max_pairs);
    out.max_seg = std::max(out.max_seg, O.max_seg);
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_cslots = std::max(out.max_cslots, O.max_cslots);
  }
  tch.clear();
  out.ntiles = (int)tiles.size() / 12;
  std::vector<int32_t> pp32(hp.begin(), hp.end()), nn32(hn.begin(), hn.end());
  pp32.resize(pp32.size() + 8, 0);
  nn32.resize(nn32.size() + 8, 0);
  out.pptr.alloc(pp32.size(), s);
  out.nptr.alloc(nn32.size(), s);
  out.recs.alloc(recs.size(), s);
  out.runs.alloc(runs.size() + 2, s);
  out.cruns.alloc(cruns.size() + 2, s);
  out.tiles.alloc(tiles.size() + 12, s);
  LG_CUDA(cudaMemcpyAsync(out.pptr.get(), pp32.data(), sizeof(int32_t) * pp32.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.nptr.get(), nn32.data(), sizeof(int32_t) * nn32.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.recs.get(), recs.data(), recs.size(), cudaMemcpyHostToDevice, s));
  if (!runs.empty())
    LG_CUDA(cudaMemcpyAsync(out.runs.get(), runs.data(), sizeof(int32_t) * runs.size(), cudaMemcpyHostToDevice, s));
  if (!cruns.empty())
    LG_CUDA(cudaMemcpyAsync(out.cruns.get(), cruns.data(), sizeof(int32_t) * cruns.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.tiles.get(), tiles.data(), sizeof(int32_t) * tiles.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

void build_locality(const MapView& key, LocalityPlan& out, cudaStream_t s) {
  const int n = key.n;
  out.n = n;
  DevBuf<int32_t> keys(n, s), iota(n, s), keys_out(n, s);
  out.perm.alloc(n, s);
  if (n == 0) return;
  k_min_key<<<ceil_div(n, kTPB), kTPB, 0, s>>>(key.v, n, key.arity, keys.get(), iota.get());
  count_launch();
  LG_LAUNCH_CHECK();
  const int endbit = bits_for(key.target);
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, keys.get(), keys_out.get(), iota.get(),
                                           out.perm.get(), n, 0, endbit, s);
  }, s);
}

void gather_rows(const MapView& m, const int32_t* perm, SortedMap& out, cudaStream_t s) {
  out.arity = m.arity;
  out.target = m.target;
  const int64_t total = (int64_t)m.n * m.arity;
  out.v.alloc(total, s);
  if (!total) return;
  k_gather_rows<<<ceil_div(total, kTPB), kTPB, 0, s>>>(m.v, perm, m.n, m.arity, out.v.get());
  count_launch();
  LG_LAUNCH_CHECK();
}

void build_pairs(const int32_t* sorted_rows, int ncells, int nrn, int nrows_node, PairPlan& out,
                 cudaStream_t s) {
  const int64_t np = (int64_t)ncells * nrn;
  require(np < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "pair list exceeds 2^31 entries");
  out.nrows_node = nrows_node;
  out.nrn = nrn;
  out.npairs = np;
  out.ptr.alloc(nrows_node + 1, s);
  out.pairs.alloc(np, s);
  DevBuf<int32_t> iota(np, s), keys_out(np, s), counts(nrows_node + 1, s);
  LG_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * (nrows_node + 1), s));
  if (np) {
    k_iota<<<ceil_div(np, kTPB), kTPB, 0, s>>>(iota.get(), np);
    k_count<<<ceil_div(np, kTPB), kTPB, 0, s>>>(sorted_rows, np, counts.get());
    count_launch(2);
    LG_LAUNCH_CHECK();
    const int endbit = bits_for(nrows_node);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, sorted_rows, keys_out.get(), iota.get(),
                                             out.pairs.get(), (int)np, 0, endbit, s);
    }, s);
  }
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, counts.get(), out.ptr.get(), nrows_node + 1, s);
  }, s);
}

__global__ void k_cell_major_ranks(const int32_t* pairs, int64_t np, int ncn, const uint8_t* ranks, uint8_t* out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int64_t code = pairs[p];
  for (int j = 0; j < ncn; ++j) out[code * ncn + j] = ranks[p * ncn + j];
}

void cell_major_ranks(const PairPlan& pp, DevBuf<uint8_t>& out, cudaStream_t s) {
  out.alloc((size_t)pp.npairs * pp.ncn + 16, s);
  if (!pp.npairs) return;
  k_cell_major_ranks<<<ceil_div(pp.npairs, kTPB), kTPB, 0, s>>>(pp.pairs.get(), pp.npairs, pp.ncn, pp.ranks.get(),
                                                                  out.get());
  count_launch();
  LG_LAUNCH_CHECK();
}

void build_ranks(PairPlan& pp, const int32_t* sorted_rows, const int32_t* sorted_cols, int ncn,
                 const CsrView& csr, cudaStream_t s) {
  pp.ncn = ncn;
  DevBuf<int> bad(1, s);
  LG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  if (csr.rd > 1 || csr.cd > 1) {
    k_check_blocked<<<ceil_div(pp.nrows_node, kTPB), kTPB, 0, s>>>(
        csr.row_ptr, csr.col_idx, pp.nrows_node, csr.rd, csr.cd, bad.get());
    count_launch();
    LG_LAUNCH_CHECK();
  }
  int hbad = 0;
  LG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  require(!hbad, LOAM_ERR(ShapeMismatch), "sparsity is not blocked by the maps' dof expansion");
  pp.ranks.alloc(pp.npairs * ncn, s);
  DevBuf<unsigned long long> err(1, s);
  LG_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(unsigned long long), s));
  if (pp.npairs) {
    k_ranks<<<ceil_div(pp.npairs, kTPB), kTPB, 0, s>>>(pp.pairs.get(), pp.npairs, pp.nrn, ncn,
                                                       sorted_rows, sorted_cols, csr.row_ptr,
                                                       csr.col_idx, csr.rd, csr.cd,
                                                       pp.ranks.get(), err.get());
    count_launch();
    LG_LAUNCH_CHECK();
  }
  unsigned long long herr = 0;
  LG_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(herr), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (herr >> 63) {
    const int row = (int)((herr >> 32) & 0x7fffffff), col = (int)(uint32_t)herr;
    fail(LOAM_ERR(OutsideSparsity), "mat: entry (" + std::to_string(row) + ", " +
                                        std::to_string(col) + ") outside sparsity");
  }
  require(!(herr >> 62), LOAM_ERR(InvalidArgument), "row with more than 256 column nodes");
}

void build_chunks(PairPlan& pp, const CsrView& csr, int smax, int max_rows, cudaStream_t s) {
  const int nr = pp.nrows_node;
  DevBuf<int64_t> starts(nr + 1, s);
  k_node_starts<<<ceil_div(nr + 1, kTPB), kTPB, 0, s>>>(csr.row_ptr, nr, csr.rd, starts.get());
  count_launch();
  LG_LAUNCH_CHECK();
  std::vector<int64_t> h(nr + 1);
  LG_CUDA(cudaMemcpyAsync(h.data(), starts.get(), sizeof(int64_t) * (nr + 1),
                          cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> chunks{0};
  int seg_max = 0;
  int r0 = 0;
  while (r0 < nr) {
    int r1 = r0 + 1;
    require(h[r1] - h[r0] <= smax, LOAM_ERR(InvalidArgument), "row segment exceeds shared memory");
    while (r1 < nr && r1 - r0 < max_rows && h[r1 + 1] - h[r0] <= smax) ++r1;
    seg_max = std::max<int>(seg_max, (int)(h[r1] - h[r0]));
    chunks.push_back(r1);
    r0 = r1;
  }
  pp.nchunks = (int)chunks.size() - 1;
  pp.seg_max = seg_max;
  pp.chunk_row.alloc(chunks.size(), s);
  LG_CUDA(cudaMemcpyAsync(pp.chunk_row.get(), chunks.data(), sizeof(int32_t) * chunks.size(),
                          cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s)); // host vector goes out of scope
}

// Row-owner sparsity build: one thread per row node merges the column nodes
// of the cells around it (the node -> cell inverse of the row map) into a
// sorted, duplicate-free list -- pass 1 counts, pass 2 (after the scan) writes
// the dof-expanded columns.  No 64-bit key per (cell, i, j) is materialised or
// sorted (the radix path below sorts ncells * arity_r * arity_c keys); rows
// with more than kRowCap distinct column nodes send the whole build there.
constexpr int kRowCap = 192;

template <bool FILL>
__global__ void __launch_bounds__(128) k_row_cols(const int32_t* __restrict__ ptr, const int32_t* __restrict__ pairs,
                                                  int ar_r, const int32_t* __restrict__ cm, int ar_c, int nr,
                                                  int32_t* __restrict__ counts, int* overflow,
                                                  const int64_t* __restrict__ rp, int rd, int cd,
                                                  int32_t* __restrict__ ci) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nr) return;
  int list[kRowCap];
  int len = 0;
  bool over = false;
  for (int p = ptr[r]; p < ptr[r + 1] && !over; ++p) {
    const int64_t c = pairs[p] / ar_r;
    for (int j = 0; j < ar_c; ++j) {
      const int x = __ldg(cm + c * ar_c + j);
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (list[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      if (lo < len && list[lo] == x) continue;
      if (len == kRowCap) {
        over = true;
        break;
      }
      for (int q = len; q > lo; --q) list[q] = list[q - 1];
      list[lo] = x;
      ++len;
    }
  }
  if constexpr (!FILL) {
    counts[r] = len;
    if (over) *overflow = 1;
  } else {
    for (int d = 0; d < rd; ++d) {
      int32_t* dst = ci + rp[(int64_t)r * rd + d];
      for (int i = 0; i < len; ++i)
        for (int x = 0; x < cd; ++x) dst[(int64_t)i * cd + x] = list[i] * cd + x;
    }
  }
}

// node -> cells inverse of a map by counting + atomic cursors (the order of a
// node's cells is arbitrary: k_row_cols sorts what it merges)
__global__ void k_inv_fill(const int32_t* __restrict__ m, int64_t np, int arity, const int32_t* __restrict__ ptr,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ cells) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np) return;
  const int r = m[t];
  cells[ptr[r] + atomicAdd(cursor + r, 1)] = (int32_t)t; // the pair code cell * arity + i, as build_pairs
}

bool build_sparsity_rows(const MapView& rows, const MapView& cols, int rd, int cd, int64_t** row_ptr,
                         int32_t** col_idx, int64_t* nnz, cudaStream_t s) {
  const int n = rows.n, nr = rows.target;
  if (n == 0 || nr == 0 || (int64_t)n * rows.arity >= (int64_t(1) << 31)) return false;
  const int64_t np = (int64_t)n * rows.arity;
  plan_tick("sparsity: start", s);
  DevBuf<int32_t> pptr(nr + 1, s), pcells(np, s), cursor(nr + 1, s);
  LG_CUDA(cudaMemsetAsync(cursor.get(), 0, sizeof(int32_t) * (nr + 1), s));
  k_count<<<ceil_div(np, kTPB), kTPB, 0, s>>>(rows.v, np, cursor.get());
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cursor.get(), pptr.get(), nr + 1, s);
  }, s);
  LG_CUDA(cudaMemsetAsync(cursor.get(), 0, sizeof(int32_t) * (nr + 1), s));
  k_inv_fill<<<ceil_div(np, kTPB), kTPB, 0, s>>>(rows.v, np, rows.arity, pptr.get(), cursor.get(), pcells.get());
  count_launch(2);
  LG_LAUNCH_CHECK();
  plan_tick("sparsity: node -> cell inverse", s);
  DevBuf<int32_t> counts(nr + 1, s);
  DevBuf<int64_t> node_off(nr + 1, s);
  DevBuf<int> over(1, s);
  LG_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * (nr + 1), s));
  LG_CUDA(cudaMemsetAsync(over.get(), 0, sizeof(int), s));
  k_row_cols<false><<<ceil_div(nr, 128), 128, 0, s>>>(pptr.get(), pcells.get(), rows.arity, cols.v, cols.arity, nr,
                                                      counts.get(), over.get(), nullptr, rd, cd, nullptr);
  count_launch();
  LG_LAUNCH_CHECK();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, counts.get(), node_off.get(), nr + 1, s);
  }, s);
  int hover = 0;
  int64_t nu = 0;
  LG_CUDA(cudaMemcpyAsync(&hover, over.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaMemcpyAsync(&nu, node_off.get() + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  plan_tick("sparsity: row counts + scan", s);
  if (hover) return false;
  const int64_t nrows = (int64_t)nr * rd;
  const int64_t total = nu * rd * cd;
  require(total < (int64_t(1) << 40), LOAM_ERR(InvalidArgument), "sparsity too large");
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(row_ptr), sizeof(int64_t) * (nrows + 1), s));
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(col_idx), sizeof(int32_t) * (total ? total : 1), s));
  k_expand_rowptr<<<ceil_div(nrows + 1, kTPB), kTPB, 0, s>>>(node_off.get(), nr, rd, cd, *row_ptr);
  k_row_cols<true><<<ceil_div(nr, 128), 128, 0, s>>>(pptr.get(), pcells.get(), rows.arity, cols.v, cols.arity, nr,
                                                     nullptr, nullptr, *row_ptr, rd, cd, *col_idx);
  count_launch(2);
  LG_LAUNCH_CHECK();
  plan_tick("sparsity: columns", s);
  *nnz = total;
  return true;
}

void build_sparsity_dev(const MapView& rows, const MapView& cols, int rd, int cd,
                        int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, cudaStream_t s) {
  require(rows.n == cols.n, LOAM_ERR(SourceMismatch),
          "row and column maps must share their source set");
  const int n = rows.n;
  static const bool sort_only = std::getenv("LOAM_GPU_SPARSITY_SORT") != nullptr; // developer: the radix path
  if (!sort_only && build_sparsity_rows(rows, cols, rd, cd, row_ptr, col_idx, nnz, s)) return;
  const int64_t nk = (int64_t)n * rows.arity * cols.arity;
  require(nk < (int64_t(1) << 31), LOAM_ERR(InvalidArgument), "sparsity key count exceeds 2^31");
  DevBuf<unsigned long long> keys(nk, s), sorted(nk, s);
  if (nk) {
    k_emit_keys<<<ceil_div(nk, kTPB), kTPB, 0, s>>>(rows.v, rows.arity, cols.v, cols.arity, n,
                                                    keys.get());
    count_launch();
    LG_LAUNCH_CHECK();
    const int endbit = 32 + bits_for(rows.target);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, keys.get(), sorted.get(), (int)nk, 0, endbit, s);
    }, s);
  }
  DevBuf<int> nsel(1, s);
  LG_CUDA(cudaMemsetAsync(nsel.get(), 0, sizeof(int), s));
  if (nk)
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.get(), keys.get(), nsel.get(), (int)nk, s);
    }, s);
  int nu = 0;
  LG_CUDA(cudaMemcpyAsync(&nu, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  const int nr = rows.target;
  DevBuf<int32_t> counts(nr + 1, s);
  DevBuf<int64_t> node_off(nr + 1, s);
  LG_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * (nr + 1), s));
  if (nu) {
    k_key_rows<<<ceil_div(nu, kTPB), kTPB, 0, s>>>(keys.get(), nu, counts.get());
    count_launch();
    LG_LAUNCH_CHECK();
  }
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, counts.get(), node_off.get(), nr + 1, s);
  }, s);
  const int64_t nrows = (int64_t)nr * rd;
  const int64_t total = (int64_t)nu * rd * cd;
  require(total < (int64_t(1) << 40), LOAM_ERR(InvalidArgument), "sparsity too large");
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(row_ptr), sizeof(int64_t) * (nrows + 1), s));
  LG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(col_idx), sizeof(int32_t) * (total ? total : 1), s));
  k_expand_rowptr<<<ceil_div(nrows + 1, kTPB), kTPB, 0, s>>>(node_off.get(), nr, rd, cd, *row_ptr);
  count_launch();
  if (nu) {
    k_fill_cols<<<ceil_div(nu, kTPB), kTPB, 0, s>>>(keys.get(), nu, node_off.get(), *row_ptr, rd, cd,
                                                    *col_idx);
    count_launch();
  }
  LG_LAUNCH_CHECK();
  *nnz = total;
}

void color_dev(int n, const std::vector<MapView>& maps, ColorPlan& out, cudaStream_t s) {
  require(maps.size() <= 4, LOAM_ERR(InvalidArgument), "at most 4 distinct conflict maps");
  out.colors.alloc(n, s);
  if (n == 0) { out.ncolors = 0; out.offsets = {0}; return; }
  LG_CUDA(cudaMemsetAsync(out.colors.get(), 0xff, sizeof(int32_t) * n, s));
  // inverse maps (target -> ascending entities)
  std::vector<DevBuf<int32_t>> ptrs(maps.size()), ents(maps.size());
  InvMap inv[4] = {};
  for (size_t mi = 0; mi < maps.size(); ++mi) {
    const MapView& m = maps[mi];
    PairPlan pp; // target -> pair codes e*arity+k, ascending e within a target
    build_pairs(m.v, m.n, m.arity, m.target, pp, s);
    ptrs[mi] = std::move(pp.ptr);
    ents[mi] = std::move(pp.pairs);
    inv[mi] = InvMap{ptrs[mi].get(), ents[mi].get(), m.v, m.arity};
  }
  DevBuf<int> remaining(1, s), overflow(1, s);
  LG_CUDA(cudaMemsetAsync(overflow.get(), 0, sizeof(int), s));
  int rounds = 0;
  for (;;) {
    LG_CUDA(cudaMemsetAsync(remaining.get(), 0, sizeof(int), s));
    const int g = ceil_div(n, kTPB);
    switch (maps.size()) {
    case 0: k_jp_round<0><<<g, kTPB, 0, s>>>(n, inv[0], inv[1], inv[2], inv[3], out.colors.get(), remaining.get(), overflow.get()); break;
    case 1: k_jp_round<1><<<g, kTPB, 0, s>>>(n, inv[0], inv[1], inv[2], inv[3], out.colors.get(), remaining.get(), overflow.get()); break;
    case 2: k_jp_round<2><<<g, kTPB, 0, s>>>(n, inv[0], inv[1], inv[2], inv[3], out.colors.get(), remaining.get(), overflow.get()); break;
    case 3: k_jp_round<3><<<g, kTPB, 0, s>>>(n, inv[0], inv[1], inv[2], inv[3], out.colors.get(), remaining.get(), overflow.get()); break;
    default: k_jp_round<4><<<g, kTPB, 0, s>>>(n, inv[0], inv[1], inv[2], inv[3], out.colors.get(), remaining.get(), overflow.get()); break;
    }
    count_launch();
    LG_LAUNCH_CHECK();
    ++rounds;
    int hrem = 0, hov = 0;
    LG_CUDA(cudaMemcpyAsync(&hrem, remaining.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaMemcpyAsync(&hov, overflow.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    require(!hov, LOAM_ERR(InvalidArgument), "more than 256 colours");
    if (hrem == 0) break;
  }
  // entities sorted by (colour, index) and colour offsets
  DevBuf<int32_t> iota(n, s), ckeys(n, s), counts(257, s);
  out.order.alloc(n, s);
  k_iota<<<ceil_div(n, kTPB), kTPB, 0, s>>>(iota.get(), n);
  LG_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int32_t) * 257, s));
  k_count<<<ceil_div(n, kTPB), kTPB, 0, s>>>(out.colors.get(), n, counts.get());
  count_launch(2);
  LG_LAUNCH_CHECK();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, out.colors.get(), ckeys.get(), iota.get(),
                                           out.order.get(), n, 0, 9, s);
  }, s);
  std::vector<int32_t> hc(257);
  LG_CUDA(cudaMemcpyAsync(hc.data(), counts.get(), sizeof(int32_t) * 257, cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  out.ncolors = 0;
  for (int c = 0; c < 256; ++c)
    if (hc[c]) out.ncolors = c + 1;
  out.offsets.assign(out.ncolors + 1, 0);
  for (int c = 0; c < out.ncolors; ++c) out.offsets[c + 1] = out.offsets[c] + hc[c];
}


// ===========================================================================
// Ring plan on the device (the C2 headline's first-call cost).  Same tiles,
// window runs, slots and chain records as build_nbr's host ring mode for
// tiles of a fixed row count; any tile or row the fast path cannot handle
// (a window range over kRdBits, too many runs or slots, a non-manifold star,
// a row without pairs) sets a flag and the caller falls back to build_nbr.
// ===========================================================================
namespace {

constexpr int kRdThreads = 256;      // one CTA per tile, one thread per row
constexpr int kRdBits = 16384;       // window range bitmap (vertex pairs)
constexpr int kRdMaxRuns = 32;       // runs per tile (fixed stride in the runs array)
constexpr int kRdMaxAdj = 8 * kRdThreads;

struct RingDevArgs {
  const int32_t* rows;    // sorted cell rows [ncells x 3]
  const int32_t* nptr;    // node pattern offsets
  const int32_t* nadj;    // node pattern columns
  const int32_t* pptr;    // pair offsets per row
  const int32_t* pairs;   // cell * 3 + i
  int nrows, tile_rows, ntiles, tile_slots;
  int32_t* rtiles;        // [ntiles x 16]
  int32_t* runs;          // [ntiles x kRdMaxRuns x 2]
  int32_t* rptr;          // [nrows + 1]
  uint16_t* rrecs;
  uint32_t* rowinfo;
  int* stat;              // [0] fail flag, [1..] maxima: rows, adj, recs, slots, runs, len
};

__global__ void __launch_bounds__(kRdThreads) k_ring_plan(const RingDevArgs a) {
  __shared__ uint32_t bits[kRdBits / 32];
  __shared__ int run_lo[kRdMaxRuns], run_hi[kRdMaxRuns], run_base[kRdMaxRuns];
  __shared__ int nruns, vmin_s, vmax_s, fail_s, slots_s;
  __shared__ uint16_t eslot[kRdMaxAdj];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int r0 = t * a.tile_rows, r1 = min(a.nrows, r0 + a.tile_rows);
  const int a0 = a.nptr[r0], a1 = a.nptr[r1];
  if (tid == 0) {
    vmin_s = INT_MAX;
    vmax_s = -1;
    fail_s = (a1 - a0 > kRdMaxAdj) ? 1 : 0;
  }
  for (int q = tid; q < kRdBits / 32; q += kRdThreads) bits[q] = 0u;
  __syncthreads();
  int lmin = INT_MAX, lmax = -1;
  for (int e = a0 + tid; e < a1; e += kRdThreads) {
    const int v = a.nadj[e];
    lmin = min(lmin, v);
    lmax = max(lmax, v);
  }
  atomicMin(&vmin_s, lmin);
  atomicMax(&vmax_s, lmax);
  __syncthreads();
  const int base = vmin_s & ~1;
  if (tid == 0 && (vmax_s < 0 || (vmax_s - base) / 2 >= kRdBits)) fail_s = 1;
  __syncthreads();
  if (fail_s) {
    if (tid == 0) atomicExch(a.stat, 1);
    return;
  }
  for (int e = a0 + tid; e < a1; e += kRdThreads) {
    const int p = (a.nadj[e] - base) >> 1; // the even-aligned vertex pair of the id
    atomicOr(&bits[p >> 5], 1u << (p & 31));
  }
  __syncthreads();
  // runs, in id order, merged across gaps of <= 8 vertices (4 pairs):
  // build_nbr's make_runs on the sorted unique ids
  if (tid == 0) {
    const int npairs = (vmax_s - base) / 2 + 1;
    int n = 0, slots = 0, lo = -1, hi = -1;
    for (int p = 0; p < npairs; ++p) {
      if (!((bits[p >> 5] >> (p & 31)) & 1u)) continue;
      const int vlo = base + 2 * p, vhi = min(a.nrows, vlo + 2);
      if (lo >= 0 && vlo <= hi + 8) {
        hi = max(hi, vhi);
      } else {
        if (lo >= 0) {
          if (n == kRdMaxRuns) { fail_s = 1; break; }
          run_lo[n] = lo; run_hi[n] = hi; run_base[n] = slots; slots += hi - lo; ++n;
        }
        lo = vlo;
        hi = vhi;
      }
    }
    if (!fail_s && lo >= 0) {
      if (n == kRdMaxRuns) fail_s = 1;
      else { run_lo[n] = lo; run_hi[n] = hi; run_base[n] = slots; slots += hi - lo; ++n; }
    }
    if (slots > a.tile_slots) fail_s = 1;
    nruns = n;
    slots_s = slots;
  }
  __syncthreads();
  if (fail_s) {
    if (tid == 0) atomicExch(a.stat, 1);
    return;
  }
  // window slot of every pattern entry of the tile
  for (int e = a0 + tid; e < a1; e += kRdThreads) {
    const int v = a.nadj[e];
    int k = 0;
    while (k + 1 < nruns && run_lo[k + 1] <= v) ++k;
    eslot[e - a0] = (uint16_t)(run_base[k] + v - run_lo[k]);
  }
  __syncthreads();
  // one thread per row: the star's chain (the host's ring / fan order)
  const int r = r0 + tid;
  bool ok = true;
  if (r < r1) {
    const int na0 = a.nptr[r], L = a.nptr[r + 1] - na0;
    const int P = a.pptr[r + 1] - a.pptr[r];
    const int rp = a.pptr[r] + r;
    a.rptr[r] = rp;
    if (r + 1 == a.nrows) a.rptr[r + 1] = a.pptr[r + 1] + r + 1;
    auto rank_of = [&](int v) {
      for (int q = 0; q < L; ++q)
        if (a.nadj[na0 + q] == v) return q;
      return -1;
    };
    auto rec = [&](int v, int& out) {
      const int q = rank_of(v);
      if (q < 0 || q > 7) return false;
      out = (eslot[na0 + q - a0] << 4) | q;
      return true;
    };
    int av[8], bv[8];
    if (L > 8 || P > 7 || P == 0) ok = false;
    for (int q = 0; q < P && ok; ++q) {
      const int code = a.pairs[a.pptr[r] + q];
      const int c = code / 3, i = code - 3 * c;
      av[q] = a.rows[(int64_t)c * 3 + (i + 1) % 3];
      bv[q] = a.rows[(int64_t)c * 3 + (i + 2) % 3];
    }
    int self = -1, start = 0, ones = 0;
    if (ok) ok = rec(r, self);
    if (ok) {
      a.rowinfo[r] = (uint32_t)(self >> 4) | ((uint32_t)(self & 15) << 16);
      start = av[0];
      for (int q = 0; q < P && ok; ++q)
        for (int u2 = 0; u2 < 2; ++u2) {
          const int v = u2 ? bv[q] : av[q];
          int deg = 0;
          for (int u = 0; u < P; ++u) deg += (av[u] == v) + (bv[u] == v);
          if (deg > 2 || v == r) ok = false;
          if (deg == 1) { ++ones; start = v; }
        }
      if (ones != 0 && ones != 2) ok = false;
    }
    if (ok) {
      unsigned used = 0u;
      int v = start, x = 0;
      ok = rec(v, x);
      if (ok) a.rrecs[rp] = (uint16_t)x;
      for (int k = 0; k < P && ok; ++k) {
        int q = 0;
        while (q < P && (((used >> q) & 1u) || (av[q] != v && bv[q] != v))) ++q;
        if (q == P) { ok = false; break; }
        used |= 1u << q;
        v = av[q] == v ? bv[q] : av[q];
        ok = rec(v, x);
        if (ok) a.rrecs[rp + 1 + k] = (uint16_t)x;
      }
      if (ok && ones == 0 && v != start) ok = false; // a ring must close
    }
    if (!ok) atomicExch(a.stat, 1);
    atomicMax(a.stat + 6, L);
  }
  if (tid == 0) {
    int32_t* rt = a.rtiles + 16 * t;
    rt[0] = r0; rt[1] = r1; rt[2] = a0; rt[3] = a1;
    rt[4] = a.pptr[r0] + r0; rt[5] = a.pptr[r1] + r1;
    rt[6] = t * kRdMaxRuns; rt[7] = nruns;
    for (int q = 0; q < kRingInlineRuns; ++q) {
      rt[8 + 2 * q] = q < nruns ? run_lo[q] : 0;
      rt[9 + 2 * q] = q < nruns ? run_hi[q] : 0;
    }
    for (int q = 0; q < nruns; ++q) {
      a.runs[2 * (t * kRdMaxRuns + q)] = run_lo[q];
      a.runs[2 * (t * kRdMaxRuns + q) + 1] = run_hi[q];
    }
    atomicMax(a.stat + 1, r1 - r0);
    atomicMax(a.stat + 2, a1 - a0);
    atomicMax(a.stat + 3, rt[5] - rt[4]);
    atomicMax(a.stat + 4, slots_s);
    atomicMax(a.stat + 5, nruns);
  }
}

} // namespace

bool build_ring_dev(NbrPlan& np, const int32_t* sorted_rows, int ncells, int nrows_node, const CsrView& csr,
                    int tile_rows, int tile_seg, int tile_slots, cudaStream_t s) {
  if (csr.rd != 1 || csr.cd != 1 || !csr.row_ptr || nrows_node == 0 || tile_rows > kRdThreads ||
      csr.nnz >= (int64_t(1) << 31) || (int64_t)tile_rows * 8 > tile_seg)
    return false;
  np.nrows_node = nrows_node;
  np.nrn = 3;
  np.rd = np.cd = 1;
  const int64_t nn = csr.nnz;
  np.nptr.alloc(nrows_node + 1 + 4, s);
  LG_CUDA(cudaMemsetAsync(np.nptr.get(), 0, np.nptr.bytes(), s));
  k_i64_to_i32<<<ceil_div(nrows_node + 1, kTPB), kTPB, 0, s>>>(csr.row_ptr, nrows_node + 1, np.nptr.get());
  count_launch();
  PairPlan pp;
  build_pairs(sorted_rows, ncells, 3, nrows_node, pp, s);
  const int ntiles = ceil_div(nrows_node, tile_rows);
  const int64_t nrec = pp.npairs + nrows_node;
  np.rptr.alloc(nrows_node + 1 + 4, s);
  np.rrecs.alloc(nrec + 8, s);
  np.rowinfo.alloc(nrows_node + 4, s);
  np.rtiles.alloc((size_t)ntiles * 16, s);
  np.runs.alloc((size_t)ntiles * kRdMaxRuns * 2 + 2, s);
  LG_CUDA(cudaMemsetAsync(np.rptr.get(), 0, np.rptr.bytes(), s));
  LG_CUDA(cudaMemsetAsync(np.rrecs.get(), 0, np.rrecs.bytes(), s));
  DevBuf<int> stat(8, s);
  LG_CUDA(cudaMemsetAsync(stat.get(), 0, stat.bytes(), s));
  RingDevArgs a{sorted_rows, np.nptr.get(), csr.col_idx, pp.ptr.get(), pp.pairs.get(), nrows_node, tile_rows, ntiles,
                std::min(tile_slots, 4095), np.rtiles.get(), np.runs.get(), np.rptr.get(), np.rrecs.get(),
                np.rowinfo.get(), stat.get()};
  k_ring_plan<<<ntiles, kRdThreads, 0, s>>>(a);
  count_launch();
  LG_LAUNCH_CHECK();
  int h[8];
  LG_CUDA(cudaMemcpyAsync(h, stat.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  if (h[0]) return false;
  np.ring = true;
  np.ntiles = ntiles;
  np.max_rows = h[1];
  np.max_adj = h[2];
  np.max_pairs = h[3]; // ring records per tile (pairs + one head per row)
  np.max_slots = h[4];
  np.max_runs = h[5];
  np.max_len = h[6];
  np.max_seg = h[2];
  (void)nn;
  return true;
}

} // namespace loam_gpu
