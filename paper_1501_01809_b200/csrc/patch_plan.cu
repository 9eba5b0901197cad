// patch_plan.cu -- host construction of the cell-patch plan (patch.cuh).
//
// Built once per loop shape and cached with the other plans (the reference
// caches its colouring the same way, parloop.hpp:153-168).  The maps are
// copied to the host, the plan is built with a few passes plus a per-patch
// sort (threaded), and uploaded.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "patch.cuh"
#include "plan.cuh"

namespace loam_gpu {

namespace {

template <class Fn>
void parallel_for(int n, Fn fn) {
  const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 32));
  if (n < 64 || nt == 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (;;) {
        const int b = next.fetch_add(16);
        if (b >= n) break;
        for (int i = b; i < std::min(n, b + 16); ++i) fn(i);
      }
    });
  for (auto& x : th) x.join();
}

uint64_t spread_bits(uint64_t x, int dims) { // interleave the low bits of x with stride `dims`
  uint64_t r = 0;
  const int nb = dims == 2 ? 31 : 21;
  for (int b = 0; b < nb; ++b) r |= ((x >> b) & 1ull) << (b * dims);
  return r;
}

__global__ void k_count_ne(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                           unsigned long long* bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (; i < n; i += stride) c += a[i] != b[i];
  if (c) atomicAdd(bad, c);
}

__global__ void k_count_ne64(const int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t n,
                             unsigned long long* bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (; i < n; i += stride) c += a[i] != b[i];
  if (c) atomicAdd(bad, c);
}

} // namespace

bool pattern_is_map_pattern(const int32_t* m, int n, int arity, int target, int rd, int cd,
                            const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz, cudaStream_t s) {
  const MapView mv{m, n, arity, target};
  return pattern_is_maps_pattern(mv, mv, rd, cd, row_ptr, col_idx, nnz, s);
}

bool pattern_is_maps_pattern(const MapView& rows, const MapView& cols, int rd, int cd, const int64_t* row_ptr,
                             const int32_t* col_idx, int64_t nnz, cudaStream_t s) {
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  int64_t bn = 0;
  const int target = rows.target;
  build_sparsity_dev(rows, cols, rd, cd, &rp, &ci, &bn, s);
  bool same = bn == nnz;
  if (same) {
    DevBuf<unsigned long long> bad(1, s);
    LG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), s));
    const int64_t nr = (int64_t)target * rd + 1;
    k_count_ne64<<<kNumSMs * 4, 256, 0, s>>>(rp, row_ptr, nr, bad.get());
    if (nnz) k_count_ne<<<kNumSMs * 4, 256, 0, s>>>(ci, col_idx, nnz, bad.get());
    count_launch(nnz ? 2 : 1);
    LG_LAUNCH_CHECK();
    unsigned long long h = 0;
    LG_CUDA(cudaMemcpyAsync(&h, bad.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
    same = h == 0;
  }
  if (rp) LG_CUDA(cudaFreeAsync(rp, s));
  if (ci) LG_CUDA(cudaFreeAsync(ci, s));
  return same;
}

// Cell-owned patches (no halo, Dats): patch p = cells [p*S, (p+1)*S) of the
// order; its window holds every node of its cells, flagged (bit 31) when the
// node also belongs to a cell of another patch (the kernel adds those with a
// global fp64 RED, the others are written once).
bool build_cell_patches(PatchPlan& out, const PatchSpec& sp, int n, int nnodes, const std::vector<int32_t>& hr,
                        const std::vector<int32_t>& order, const std::vector<int32_t>& incid, cudaStream_t s) {
  const int nrn = sp.nrn, S = std::max(1, sp.max_cells);
  const int np = (n + S - 1) / S;
  std::vector<std::vector<int32_t>> wins(np);
  std::vector<int64_t> roff(np + 1, 0);
  for (int p = 0; p < np; ++p) roff[p + 1] = roff[p] + (((int64_t)(std::min(n, (p + 1) * S) - p * S) * nrn + 7) & ~int64_t(7));
  std::vector<uint16_t> recs(roff[np] + 8, 0);
  std::vector<int> bad(np, 0);
  std::vector<std::vector<int32_t>> cnts(np);
  parallel_for(np, [&](int p) {
    const int c0 = p * S, c1 = std::min(n, c0 + S);
    std::vector<int32_t> all;
    all.reserve((size_t)(c1 - c0) * nrn);
    for (int q = c0; q < c1; ++q)
      for (int i = 0; i < nrn; ++i) all.push_back(hr[(size_t)order[q] * nrn + i]);
    std::vector<int32_t> w(all);
    std::sort(w.begin(), w.end());
    std::vector<int32_t> cnt;
    std::vector<int32_t>& u = wins[p];
    for (size_t a = 0; a < w.size();) {
      size_t b = a;
      while (b < w.size() && w[b] == w[a]) ++b;
      u.push_back(w[a]);
      cnt.push_back((int32_t)(b - a));
      a = b;
    }
    if (u.size() > 32767) {
      bad[p] = 1;
      return;
    }
    uint16_t* rp_ = &recs[roff[p]];
    for (int q = c0; q < c1; ++q)
      for (int i = 0; i < nrn; ++i) {
        const int node = hr[(size_t)order[q] * nrn + i];
        rp_[(size_t)(q - c0) * nrn + i] = (uint16_t)(std::lower_bound(u.begin(), u.end(), node) - u.begin());
      }
    for (size_t k = 0; k < u.size(); ++k)
      if (cnt[k] != incid[u[k]]) u[k] |= (int32_t)0x80000000u; // shared with another patch
    cnts[p] = std::move(cnt);
  });
  for (int p = 0; p < np; ++p)
    if (bad[p]) return false;
  std::vector<int4> hdr(2 * (size_t)np);
  std::vector<int32_t> win;
  std::vector<uint16_t> nptr; // per patch: incidence offsets of its window nodes (nwin + 1)
  out = PatchPlan{};
  out.npatches = np;
  out.nrn = nrn;
  out.halo = false;
  int64_t nb = 0;
  for (int p = 0; p < np; ++p) {
    while (win.size() & 3) win.push_back(0);
    while (nptr.size() & 7) nptr.push_back(0);
    const int nc = std::min(n, (p + 1) * S) - p * S;
    hdr[2 * p] = make_int4((int)win.size(), (int)wins[p].size(), (int)roff[p], nc);
    hdr[2 * p + 1] = make_int4((int)nptr.size(), 0, 0, 0);
    int run = 0;
    for (int32_t c : cnts[p]) {
      nptr.push_back((uint16_t)run);
      run += c;
    }
    nptr.push_back((uint16_t)run);
    if (run > 65535) return false;
    for (int32_t x : wins[p]) nb += x < 0;
    win.insert(win.end(), wins[p].begin(), wins[p].end());
    out.max_win = std::max(out.max_win, (int)wins[p].size());
    out.max_cells = std::max(out.max_cells, nc);
  }
  out.tile_cells = n;
  out.boundary = nb;
  win.resize(win.size() + 8, 0);
  nptr.resize(nptr.size() + 16, 0);
  out.hdr.alloc(hdr.size(), s);
  out.win.alloc(win.size(), s);
  out.recs.alloc(recs.size(), s);
  out.own.alloc(nptr.size(), s);
  LG_CUDA(cudaMemcpyAsync(out.own.get(), nptr.data(), sizeof(uint16_t) * nptr.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.hdr.get(), hdr.data(), sizeof(int4) * hdr.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.win.get(), win.data(), sizeof(int32_t) * win.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.recs.get(), recs.data(), sizeof(uint16_t) * recs.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

bool build_patch(PatchPlan& out, const PatchSpec& sp, int ncells, int nnodes, const int32_t* rows,
                 const int32_t* xmap, int xstride, const double* coords, const int64_t* row_ptr,
                 cudaStream_t s) {
  const int gd = sp.gd, nv = gd + 1, nrn = sp.nrn, n = ncells;
  if (n <= 0 || nnodes <= 0 || nrn < nv) return false;
  // ---- host copies
  std::vector<int32_t> hr((size_t)n * nrn), hx((size_t)n * xstride);
  LG_CUDA(cudaMemcpyAsync(hr.data(), rows, sizeof(int32_t) * hr.size(), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaMemcpyAsync(hx.data(), xmap, sizeof(int32_t) * hx.size(), cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> rp;
  if (sp.bilinear) {
    rp.resize((size_t)nnodes * sp.rd + 1);
    LG_CUDA(cudaMemcpyAsync(rp.data(), row_ptr, sizeof(int64_t) * rp.size(), cudaMemcpyDeviceToHost, s));
  }
  LG_CUDA(cudaStreamSynchronize(s));
  // the coordinate map must be the vertex prefix of the row map (P1: equal;
  // P2: vertices first, space.hpp:41-46), so vertex coordinates are found
  // through the window slots of the first gd+1 row nodes
  int nverts = 0;
  for (int e = 0; e < n; ++e)
    for (int v = 0; v < nv; ++v) {
      const int x = hx[(size_t)e * xstride + v];
      if (x != hr[(size_t)e * nrn + v]) return false;
      nverts = std::max(nverts, x + 1);
    }
  std::vector<double> hc((size_t)nverts * gd);
  LG_CUDA(cudaMemcpyAsync(hc.data(), coords, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  // ---- Morton order of the cell centroids
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int v = 0; v < nverts; ++v)
    for (int a = 0; a < gd; ++a) {
      lo[a] = std::min(lo[a], hc[(size_t)v * gd + a]);
      hi[a] = std::max(hi[a], hc[(size_t)v * gd + a]);
    }
  const double qmax = gd == 2 ? 2147483647.0 : 2097151.0;
  std::vector<std::pair<uint64_t, int>> key(n);
  parallel_for((n + 4095) / 4096, [&](int b) {
    for (int e = b * 4096; e < std::min(n, (b + 1) * 4096); ++e) {
      uint64_t code = 0;
      for (int a = 0; a < gd; ++a) {
        double c = 0;
        for (int v = 0; v < nv; ++v) c += hc[(size_t)hr[(size_t)e * nrn + v] * gd + a];
        c /= nv;
        const double ext = hi[a] - lo[a];
        double t = ext > 0 ? (c - lo[a]) / ext : 0.0;
        t = std::min(1.0, std::max(0.0, t));
        code |= spread_bits((uint64_t)(t * qmax), gd) << a;
      }
      key[e] = {code, e};
    }
  });
  std::sort(key.begin(), key.end());
  std::vector<int32_t> order(n), pos(n);
  for (int p = 0; p < n; ++p) {
    order[p] = key[p].second;
    pos[key[p].second] = p;
  }
  std::vector<std::pair<uint64_t, int>>().swap(key);
  // ---- row ownership: the first cell (in the order) containing the node
  std::vector<int32_t> minpos(nnodes, n);
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < nrn; ++i) {
      int32_t& m = minpos[hr[(size_t)e * nrn + i]];
      m = std::min(m, pos[e]);
    }
  std::vector<int64_t> cost(nnodes, 1);
  if (sp.bilinear)
    for (int r = 0; r < nnodes; ++r) cost[r] = rp[(size_t)(r + 1) * sp.rd] - rp[(size_t)r * sp.rd];
  if (sp.bilinear) // in-row ranks are kept in 8 bits (patch_kernels.cuh)
    for (int r = 0; r < nnodes; ++r)
      if (cost[r] / ((int64_t)sp.rd * sp.cd) > 255) return false;
  std::vector<int64_t> poscost(n, 0);
  std::vector<int32_t> incid(nnodes, 0); // incident cells per node (= pairs)
  for (int r = 0; r < nnodes; ++r)
    if (minpos[r] < n) poscost[minpos[r]] += cost[r];
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < nrn; ++i) ++incid[hr[(size_t)e * nrn + i]];
  if (!sp.halo) return build_cell_patches(out, sp, n, nnodes, hr, order, incid, s);
  // ---- greedy patches over the order; shrink the budget until the tile
  // cells (own + halo) of every patch fit
  int64_t budget = std::max<int64_t>(sp.budget, 1);
  std::vector<int32_t> pstart, ppatch(n), owner(nnodes);
  std::vector<int64_t> coff;
  std::vector<int32_t> tcells;
  for (int attempt = 0;; ++attempt) {
    pstart.clear();
    int64_t acc = 0;
    for (int p = 0; p < n; ++p) {
      if (p == 0 || (acc + poscost[p] > budget && acc > 0)) {
        pstart.push_back(p);
        acc = 0;
      }
      acc += poscost[p];
      ppatch[p] = (int)pstart.size() - 1;
    }
    const int np = (int)pstart.size();
    for (int r = 0; r < nnodes; ++r) owner[r] = minpos[r] < n ? ppatch[minpos[r]] : -1;
    // tile cells per patch, in order position (own cells and halo interleaved)
    coff.assign(np + 1, 0);
    auto each_patch_of = [&](int e, auto&& f) {
      int seen[16], ns = 0;
      for (int i = 0; i < nrn; ++i) {
        const int p = owner[hr[(size_t)e * nrn + i]];
        bool dup = false;
        for (int k = 0; k < ns; ++k) dup |= seen[k] == p;
        if (!dup) {
          seen[ns++] = p;
          f(p);
        }
      }
    };
    for (int q = 0; q < n; ++q) each_patch_of(order[q], [&](int p) { ++coff[p + 1]; });
    int64_t maxc = 0;
    for (int p = 0; p < np; ++p) {
      maxc = std::max(maxc, coff[p + 1]);
      coff[p + 1] += coff[p];
    }
    if (maxc > sp.max_cells && budget > 1 && attempt < 12) {
      budget = std::max<int64_t>(1, budget * 3 / 4);
      continue;
    }
    if (maxc > sp.max_cells) return false;
    tcells.assign(coff[np], 0);
    std::vector<int64_t> fill(coff.begin(), coff.end() - 1);
    for (int q = 0; q < n; ++q) {
      const int e = order[q];
      each_patch_of(e, [&](int p) { tcells[fill[p]++] = e; });
    }
    break;
  }
  const int np = (int)pstart.size();
  // ---- owned rows per patch (ascending node id)
  std::vector<int64_t> ooff(np + 1, 0);
  int64_t untouched = 0;
  for (int r = 0; r < nnodes; ++r) {
    if (owner[r] >= 0) ++ooff[owner[r] + 1];
    else ++untouched;
  }
  for (int p = 0; p < np; ++p) ooff[p + 1] += ooff[p];
  std::vector<int32_t> onode(ooff[np]);
  {
    std::vector<int64_t> f(ooff.begin(), ooff.end() - 1);
    for (int r = 0; r < nnodes; ++r)
      if (owner[r] >= 0) onode[f[owner[r]]++] = r;
  }
  // ---- per-patch offsets: windows 16-byte aligned (4 ids), records 16-byte
  // aligned (8 slots), so the kernel stages both with 16-byte vector loads
  std::vector<int64_t> roff(np + 1, 0);
  for (int p = 0; p < np; ++p) roff[p + 1] = roff[p] + (((coff[p + 1] - coff[p]) * nrn + 7) & ~int64_t(7));
  // ---- windows, slot records, owned slots (per patch, threaded)
  std::vector<std::vector<int32_t>> wins(np);
  std::vector<uint16_t> recs(roff[np] + 8, 0);
  std::vector<uint16_t> own(ooff[np]);
  std::vector<int> bad(np, 0);
  parallel_for(np, [&](int p) {
    std::vector<int32_t>& w = wins[p];
    w.reserve((size_t)(coff[p + 1] - coff[p]) * nrn);
    for (int64_t t = coff[p]; t < coff[p + 1]; ++t)
      for (int i = 0; i < nrn; ++i) w.push_back(hr[(size_t)tcells[t] * nrn + i]);
    std::sort(w.begin(), w.end());
    w.erase(std::unique(w.begin(), w.end()), w.end());
    if (w.size() > 32767) { // slots and owned-row indices are 16-bit
      bad[p] = 1;
      return;
    }
    auto slot = [&](int node) { return (uint16_t)(std::lower_bound(w.begin(), w.end(), node) - w.begin()); };
    uint16_t* rp_ = &recs[roff[p]];
    for (int64_t t = coff[p]; t < coff[p + 1]; ++t)
      for (int i = 0; i < nrn; ++i) rp_[(t - coff[p]) * nrn + i] = slot(hr[(size_t)tcells[t] * nrn + i]);
    for (int64_t k = ooff[p]; k < ooff[p + 1]; ++k) own[k] = slot(onode[k]);
  });
  for (int p = 0; p < np; ++p)
    if (bad[p]) return false;
  // ---- headers, owned-row CSR offsets (Mats) and maxima
  std::vector<int4> hdr(2 * (size_t)np);
  std::vector<int32_t> win;
  std::vector<int64_t> orp;
  std::vector<int32_t> oseg;
  if (sp.bilinear) {
    orp.resize(ooff[np]);
    oseg.resize(ooff[np] + np);
  }
  out = PatchPlan{};
  out.npatches = np;
  out.nrn = nrn;
  for (int p = 0; p < np; ++p) {
    int64_t pairs = 0, seg = 0;
    for (int64_t k = ooff[p]; k < ooff[p + 1]; ++k) {
      pairs += incid[onode[k]];
      if (sp.bilinear) {
        orp[k] = rp[(size_t)onode[k] * sp.rd];
        oseg[k + p] = (int32_t)seg;
      }
      seg += cost[onode[k]];
    }
    if (sp.bilinear) oseg[ooff[p + 1] + p] = (int32_t)seg; // end of the patch's segment
    while (win.size() & 3) win.push_back(0);
    hdr[2 * p] = make_int4((int)win.size(), (int)wins[p].size(), (int)roff[p], (int)(coff[p + 1] - coff[p]));
    hdr[2 * p + 1] = make_int4((int)ooff[p], (int)(ooff[p + 1] - ooff[p]), (int)pairs, (int)seg);
    win.insert(win.end(), wins[p].begin(), wins[p].end());
    out.max_win = std::max(out.max_win, (int)wins[p].size());
    out.max_cells = std::max<int>(out.max_cells, (int)(coff[p + 1] - coff[p]));
    out.max_own = std::max<int>(out.max_own, (int)(ooff[p + 1] - ooff[p]));
    out.max_pairs = std::max<int>(out.max_pairs, (int)pairs);
    out.max_seg = std::max(out.max_seg, seg);
  }
  out.tile_cells = coff[np];
  out.own_rows = ooff[np];
  out.untouched = untouched;
  if (win.size() >= (size_t)INT32_MAX || roff[np] >= INT32_MAX || out.max_seg >= INT32_MAX) return false;
  win.resize(win.size() + 8, 0);
  out.hdr.alloc(hdr.size(), s);
  out.win.alloc(win.size(), s);
  out.recs.alloc(recs.size(), s);
  out.own.alloc(own.size() + 8, s);
  LG_CUDA(cudaMemcpyAsync(out.hdr.get(), hdr.data(), sizeof(int4) * hdr.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.win.get(), win.data(), sizeof(int32_t) * win.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.recs.get(), recs.data(), sizeof(uint16_t) * recs.size(), cudaMemcpyHostToDevice, s));
  LG_CUDA(cudaMemcpyAsync(out.own.get(), own.data(), sizeof(uint16_t) * own.size(), cudaMemcpyHostToDevice, s));
  if (sp.bilinear) {
    out.orp.alloc(orp.size() + 1, s);
    out.oseg.alloc(oseg.size() + 1, s);
    LG_CUDA(cudaMemcpyAsync(out.orp.get(), orp.data(), sizeof(int64_t) * orp.size(), cudaMemcpyHostToDevice, s));
    LG_CUDA(cudaMemcpyAsync(out.oseg.get(), oseg.data(), sizeof(int32_t) * oseg.size(), cudaMemcpyHostToDevice, s));
  }
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

} // namespace loam_gpu
