// wtile.cu -- link-walk tiles for scalar P2 matrices on tetrahedra (see wtile.cuh).
//
// Reference path replaced: assemble_matrix (fem/assemble.hpp:85-104) ->
// execute (parloop.hpp:191-384) with the P2 mass / stiffness / helmholtz
// element kernels (restated in elements.cuh FormT<FORM, 3, 2>), Mat::addto
// (data.hpp:205-222) on the pattern of build_sparsity(map, map) (data.hpp:149-179).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "linkwalk.cuh"
#include "stage.cuh"
#include "wtile.cuh"

namespace loam_gpu {

namespace {

inline int up16(int x) { return (x + 15) & ~15; }

constexpr int kWtConsumers = 128; // consumer threads per CTA = edge rows per tile at most
constexpr int kMaxLink = 12;      // cells around one edge
// local edge of a vertex pair (Simplex<3>: (2,3),(1,3),(1,2),(0,3),(0,2),(0,1))
const int kEk[4][4] = {{-1, 5, 4, 3}, {5, -1, 2, 1}, {4, 2, -1, 0}, {3, 1, 0, -1}};

} // namespace

bool build_wtile(WtilePlan& out, const WtileSpec& sp, int ncells, int nnodes, int nverts, const int32_t* rows,
                 const int32_t* xmap, const PairPlan& pp, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                 cudaStream_t s) {
  constexpr int NT = kWtConsumers;
  if (pp.nrn != 10 || ncells == 0 || nnz >= (int64_t(1) << 31) || nverts >= nnodes || nverts <= 0) return false;
  if (pp.npairs != (int64_t)ncells * 10) return false;
  const int tile_rows = std::min(sp.tile_rows, NT), max_link = std::min(sp.max_link, kMaxLink);
  auto hv = host_array<int32_t>((size_t)ncells * 10), hx = host_array<int32_t>((size_t)ncells * 4),
       hpairs = host_array<int32_t>((size_t)pp.npairs), hp = host_array<int32_t>(nnodes + 1);
  auto hrp = host_array<int64_t>((size_t)nnodes + 1);
  parallel_d2h({{hv.data(), rows, sizeof(int32_t) * hv.size()},
                {hx.data(), xmap, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * hpairs.size()},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * hp.size()},
                {hrp.data(), row_ptr, sizeof(int64_t) * hrp.size()}},
               s);
  // the vertex rows' columns: the transposed entries are stored at their positions
  const int64_t nvc = hrp[nverts];
  if (nvc <= 0 || nvc > nnz) return false;
  auto hci = host_array<int32_t>((size_t)nvc);
  parallel_d2h({{hci.data(), col_idx, sizeof(int32_t) * (size_t)nvc}}, s);
  plan_tick("wtile: D2H", s);
  {
    std::vector<char> bad(plan_threads(), 0);
    parallel_chunks(ncells, 1, [&](int t, int64_t c0, int64_t c1) {
      for (int64_t c = c0; c < c1; ++c) {
        const int32_t* r = &hv[(size_t)c * 10];
        const int32_t* x = &hx[(size_t)c * 4];
        bool ok = true;
        for (int j = 0; j < 4; ++j) {
          ok = ok && r[j] == x[j] && x[j] >= 0 && x[j] < nverts;
          for (int q = 0; q < j; ++q) ok = ok && x[q] != x[j];
        }
        for (int j = 4; j < 10; ++j) ok = ok && r[j] >= nverts;
        if (!ok) bad[t] = 1;
      }
    });
    for (char b : bad)
      if (b) return false;
  }
  // position of column x in vertex row u (or -1)
  auto vpos = [&](int u, int x) -> int64_t {
    const int32_t* b = &hci[hrp[u]];
    const int32_t* e = &hci[hrp[u + 1]];
    const int32_t* f = std::lower_bound(b, e, x);
    return (f != e && *f == x) ? (int64_t)(f - &hci[0]) : -1;
  };
  std::vector<int32_t> dpos(nverts);
  {
    std::vector<char> bad(plan_threads(), 0);
    parallel_chunks(nverts, 1, [&](int t, int64_t v0, int64_t v1) {
      for (int64_t v = v0; v < v1; ++v) {
        const int64_t p = vpos((int)v, (int)v);
        if (p < 0) bad[t] = 1;
        dpos[v] = (int32_t)p;
      }
    });
    for (char b : bad)
      if (b) return false;
  }
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs;
    std::vector<uint8_t> blob;
    int max_seg = 0, max_slots = 0, max_blob = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int nedges = nnodes - nverts;
  std::vector<int32_t> ev(sp.det ? nedges : 0), ew(sp.det ? nedges : 0); // deterministic mode: the rows' endpoints
  const int ntch = parallel_chunks(nedges, 1, [&](int t, int64_t cb0, int64_t cb1) {
    TileChunk& O = tch[t];
    struct Stamps {
      int* p;
      explicit Stamps(size_t n) : p(static_cast<int*>(std::calloc(n + 1, sizeof(int)))) {
        if (!p) throw std::bad_alloc();
      }
      ~Stamps() { std::free(p); }
    } vstamp(nverts);
    int gen = 0;
    auto fail = [&] { O.ok = false; };
    std::vector<int> vid, seq, cols;
    std::vector<std::pair<int, int>> rr;
    std::vector<int> base;
    LinkWalk lw;
    struct Item {
      uint32_t hdr, own;
      int nce, nlv;
      int xs[2 + kMaxLink + 1];                // coordinate ids v, w, p_0 .. p_nce
      uint8_t rk[3 + 3 * (kMaxLink + 1) + kMaxLink]; // v, w, e | per link vertex p, (v,p), (w,p) | per cell (p,q)
      int32_t pos[6 + kMaxLink + 1];           // (v,e) (w,e) (v,w) (w,v) (v,v) (w,w) | (p_j, e)
    };
    std::vector<Item> items;
    const int e_begin = nverts + (int)cb0, e_end = nverts + (int)cb1;
    int e0 = e_begin;
    auto rank_in = [](const std::vector<int>& sorted, int x) {
      return (int)(std::lower_bound(sorted.begin(), sorted.end(), x) - sorted.begin());
    };
    auto emit = [&](int n0, int n1) {
      ++gen;
      vid.clear();
      int maxce = 0, maxlv = 0;
      for (const Item& it : items) {
        maxce = std::max(maxce, it.nce);
        maxlv = std::max(maxlv, it.nlv);
        for (int q = 0; q < 3 + it.nce; ++q) {
          const int x = it.xs[q];
          if (vstamp.p[x] != gen) {
            vstamp.p[x] = gen;
            vid.push_back(x);
          }
        }
      }
      const int slots = link_runs(vid, nverts, rr);
      if (slots > sp.tile_slots || (int)rr.size() > sp.tile_runs || slots >= 0xffff) return false;
      base.resize(rr.size());
      for (size_t q = 0, acc = 0; q < rr.size(); ++q) {
        base[q] = (int)acc;
        acc += rr[q].second - rr[q].first;
      }
      auto slot_in = [&](int v) {
        size_t q = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
        return base[q] + v - rr[q].first;
      };
      // blocks of equal link lengths share warps (a warp's loop runs to its longest link)
      std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.nce > b.nce; });
      const int nitems = (int)items.size();
      const int ns = 3 + maxce, nr = 3 + 3 * maxlv + maxce, np = 6 + maxlv;
      const int off_s = 8 * NT, off_r = off_s + up16(2 * NT * ns), off_p = off_r + up16(NT * nr),
                bytes = off_p + 4 * NT * np;
      const size_t b0 = O.blob.size();
      O.blob.resize(b0 + bytes, 0);
      uint8_t* bp = O.blob.data() + b0;
      for (int i = 0; i < nitems; ++i) {
        const Item& it = items[i];
        memcpy(bp + 4 * i, &it.hdr, 4);
        memcpy(bp + 4 * NT + 4 * i, &it.own, 4);
        for (int q = 0; q < 3 + it.nce; ++q) {
          const uint16_t sl = (uint16_t)slot_in(it.xs[q]);
          memcpy(bp + off_s + 2 * (q * NT + i), &sl, 2);
        }
        for (int q = 0; q < 3; ++q) bp[off_r + q * NT + i] = it.rk[q];
        for (int j = 0; j < it.nlv; ++j)
          for (int q = 0; q < 3; ++q) bp[off_r + (3 + 3 * j + q) * NT + i] = it.rk[3 + 3 * j + q];
        for (int c = 0; c < it.nce; ++c) bp[off_r + (3 + 3 * maxlv + c) * NT + i] = it.rk[3 + 3 * (kMaxLink + 1) + c];
        for (int q = 0; q < 6 + it.nlv; ++q) memcpy(bp + off_p + 4 * (q * NT + i), &it.pos[q], 4);
      }
      const int64_t E0 = hrp[n0], E1 = hrp[n1];
      const int seg = (int)(E1 - E0);
      if (bytes >= (1 << 24) || seg >= (1 << 16)) return false;
      O.tiles.insert(O.tiles.end(), {(int)(b0 / 16), bytes, n0, n1 - n0, (int)E0, seg, nitems, maxce,
                                     (int)O.runs.size() / 2, (int)rr.size(), off_s, off_r, off_p, maxlv, slots, 0});
      for (auto& x : rr) O.runs.insert(O.runs.end(), {x.first, x.second});
      O.max_seg = std::max(O.max_seg, seg);
      O.max_slots = std::max(O.max_slots, slots);
      O.max_blob = std::max(O.max_blob, bytes);
      return true;
    };
    struct CellRec {
      int c, la, lb, lo0, lo1;
    };
    for (int e = e_begin; e < e_end; ++e) {
      const int nce = hp[e + 1] - hp[e];
      if (nce < 1 || nce > max_link) return fail();
      CellRec cr[kMaxLink];
      int xv = -1, xw = -1;
      lw.nn = 0;
      for (int q = 0; q < nce; ++q) {
        const int code = hpairs[hp[e] + q], c = code / 10, l = code % 10;
        if (l < 4) return fail();
        int la = Simplex<3>::edge_a(l - 4), lb = Simplex<3>::edge_b(l - 4);
        const int32_t* x = &hx[(size_t)c * 4];
        if (q == 0) {
          xv = x[la];
          xw = x[lb];
        } else if (x[la] == xw && x[lb] == xv) {
          std::swap(la, lb);
        } else if (!(x[la] == xv && x[lb] == xw)) {
          return fail(); // one node on two mesh edges
        }
        int lo[2], no = 0;
        for (int j = 0; j < 4; ++j)
          if (j != la && j != lb) lo[no++] = j;
        cr[q] = {c, la, lb, lo[0], lo[1]};
        if (!lw.add(x[lo[0]], x[lo[0]], x[lo[1]], x[lo[1]])) return fail();
      }
      if (!lw.walk(nce, seq)) return fail();
      const bool ring = seq.front() == seq.back();
      const int nlv = ring ? nce : nce + 1;
      int nvp[kMaxLink + 1], nwp[kMaxLink + 1], npq[kMaxLink];
      for (int j = 0; j <= kMaxLink; ++j) nvp[j] = nwp[j] = -1;
      for (int i = 0; i < nce; ++i) {
        const CellRec* R = nullptr;
        int lp = -1, lq = -1;
        for (int q = 0; q < nce; ++q) {
          const int32_t* x = &hx[(size_t)cr[q].c * 4];
          if (x[cr[q].lo0] == seq[i] && x[cr[q].lo1] == seq[i + 1]) {
            R = &cr[q];
            lp = cr[q].lo0;
            lq = cr[q].lo1;
          } else if (x[cr[q].lo1] == seq[i] && x[cr[q].lo0] == seq[i + 1]) {
            R = &cr[q];
            lp = cr[q].lo1;
            lq = cr[q].lo0;
          }
        }
        if (!R) return fail();
        const int32_t* nd = &hv[(size_t)R->c * 10 + 4];
        if (nd[kEk[R->la][R->lb]] != e) return fail();
        const int j0 = i, j1 = (i + 1 == nce && ring) ? 0 : i + 1;
        const int a0 = nd[kEk[R->la][lp]], b0 = nd[kEk[R->lb][lp]], a1 = nd[kEk[R->la][lq]], b1 = nd[kEk[R->lb][lq]];
        if ((nvp[j0] >= 0 && (nvp[j0] != a0 || nwp[j0] != b0)) || (nvp[j1] >= 0 && (nvp[j1] != a1 || nwp[j1] != b1)))
          return fail(); // two nodes on one mesh edge
        nvp[j0] = a0;
        nwp[j0] = b0;
        nvp[j1] = a1;
        nwp[j1] = b1;
        npq[i] = nd[kEk[lp][lq]];
      }
      cols.clear();
      cols.push_back(xv);
      cols.push_back(xw);
      cols.push_back(e);
      for (int j = 0; j < nlv; ++j) {
        cols.push_back(seq[j]);
        cols.push_back(nvp[j]);
        cols.push_back(nwp[j]);
      }
      for (int i = 0; i < nce; ++i) cols.push_back(npq[i]);
      std::sort(cols.begin(), cols.end());
      if (std::adjacent_find(cols.begin(), cols.end()) != cols.end()) return fail();
      const int L = (int)cols.size();
      if (hrp[e + 1] - hrp[e] != L || L > 255) return fail();
      if ((int)items.size() == tile_rows || hrp[e + 1] - hrp[e0] >= 60000) {
        if (!emit(e0, e)) return fail();
        items.clear();
        e0 = e;
      }
      Item it{};
      it.nce = nce;
      it.nlv = nlv;
      it.xs[0] = xv;
      it.xs[1] = xw;
      for (int q = 0; q <= nce; ++q) it.xs[2 + q] = seq[q];
      it.rk[0] = (uint8_t)rank_in(cols, xv);
      it.rk[1] = (uint8_t)rank_in(cols, xw);
      it.rk[2] = (uint8_t)rank_in(cols, e);
      for (int j = 0; j < nlv; ++j) {
        it.rk[3 + 3 * j] = (uint8_t)rank_in(cols, seq[j]);
        it.rk[3 + 3 * j + 1] = (uint8_t)rank_in(cols, nvp[j]);
        it.rk[3 + 3 * j + 2] = (uint8_t)rank_in(cols, nwp[j]);
      }
      for (int i = 0; i < nce; ++i) it.rk[3 + 3 * (kMaxLink + 1) + i] = (uint8_t)rank_in(cols, npq[i]);
      const int64_t ps[6] = {vpos(xv, e), vpos(xw, e), vpos(xv, xw), vpos(xw, xv), dpos[xv], dpos[xw]};
      for (int q = 0; q < 6; ++q) {
        if (ps[q] < 0) return fail();
        it.pos[q] = (int32_t)ps[q];
      }
      for (int j = 0; j < nlv; ++j) {
        const int64_t p = vpos(seq[j], e);
        if (p < 0) return fail();
        it.pos[6 + j] = (int32_t)p;
      }
      uint32_t ownv = 0, ownw = 0;
      for (int i = 0; i < nce; ++i) {
        if (xw < seq[i] && xw < seq[i + 1]) ownv |= 1u << i; // (v, w) is v's edge to its smallest other vertex of the cell
        if (xv < seq[i] && xv < seq[i + 1]) ownw |= 1u << i;
      }
      it.own = ownv | ownw << 12 | (uint32_t)(e - e0) << 24; // + the row's index in its tile
      if (sp.det) {
        ev[e - nverts] = xv;
        ew[e - nverts] = xw;
      }
      it.hdr = (uint32_t)(hrp[e] - hrp[e0]) | (uint32_t)L << 16 | (uint32_t)nce << 24 | (ring ? 1u << 28 : 0u);
      items.push_back(it);
    }
    if (!items.empty() && !emit(e0, e_end)) return fail();
  });
  std::vector<int32_t> tiles, runs;
  std::vector<const std::vector<uint8_t>*> parts;
  size_t bytes_so_far = 0;
  for (int t = 0; t < ntch; ++t) {
    TileChunk& O = tch[t];
    if (!O.ok) return false;
    const int bshift = (int)(bytes_so_far / 16), rshift = (int)(runs.size() / 2);
    for (size_t q = 0; q < O.tiles.size(); q += 16) {
      O.tiles[q + 0] += bshift;
      O.tiles[q + 8] += rshift;
    }
    tiles.insert(tiles.end(), O.tiles.begin(), O.tiles.end());
    runs.insert(runs.end(), O.runs.begin(), O.runs.end());
    parts.push_back(&O.blob);
    bytes_so_far += O.blob.size();
    out.max_seg = std::max(out.max_seg, O.max_seg);
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_blob = std::max(out.max_blob, O.max_blob);
  }
  if (bytes_so_far / 16 >= (size_t)INT32_MAX) return false;
  plan_tick("wtile: tiles", s);
  upload_parts(out.blob, parts, s);
  tch.clear();
  out.ntiles = (int)tiles.size() / 16;
  out.nverts = nverts;
  auto upload = [&](auto& dst, const auto& src) {
    using T = typename std::decay_t<decltype(src)>::value_type;
    dst.alloc(src.size() + 16, s);
    if (!src.empty())
      LG_CUDA(cudaMemcpyAsync(dst.get(), src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
  };
  upload(out.tiles, tiles);
  upload(out.runs, runs);
  upload(out.dpos, dpos);
  out.det = sp.det;
  out.nedges = nedges;
  if (sp.det) { // per vertex: the diagonal-share slots (2 (e - nverts) + endpoint) of its edges, ascending
    std::vector<int32_t> dptr(nverts + 1, 0), dslots(2 * (size_t)nedges);
    for (int e = 0; e < nedges; ++e) {
      ++dptr[ev[e] + 1];
      ++dptr[ew[e] + 1];
    }
    for (int v = 0; v < nverts; ++v) dptr[v + 1] += dptr[v];
    std::vector<int32_t> cur(dptr.begin(), dptr.end() - 1);
    for (int e = 0; e < nedges; ++e) {
      dslots[cur[ev[e]]++] = 2 * e;
      dslots[cur[ew[e]]++] = 2 * e + 1;
    }
    upload(out.dptr, dptr);
    upload(out.dslots, dslots);
  }
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

// ===========================================================================
// Device side
// ===========================================================================

namespace {

struct WtileArgs {
  const int32_t* tiles;
  int ntiles;
  int* next_tile;
  int* reset_tile;
  const uint8_t* blob;
  const int32_t* runs;
  const double* coords;
  double* out;
  FormParams prm;
  int accumulate;
  int off_seg, off_buf, buf_bytes, b_win;
  double* dsum; // deterministic mode: the rows' diagonal shares by (edge, endpoint), summed by k_wt_dsum
  int nverts;
};

// Deterministic diagonals: vertex v = its edges' shares in edge order.
__global__ void k_wt_dsum(const int32_t* __restrict__ dpos, const int32_t* __restrict__ dptr,
                          const int32_t* __restrict__ dslots, int n, const double* __restrict__ dsum,
                          double* __restrict__ out, int accumulate) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double acc = 0.0;
  for (int q = dptr[v]; q < dptr[v + 1]; ++q) acc += dsum[dslots[q]];
  out[dpos[v]] = accumulate ? out[dpos[v]] + acc : acc;
}

__global__ void k_wt_zero(double* __restrict__ out, const int32_t* __restrict__ dpos, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[dpos[i]] = 0.0;
}

// vertex-vertex entry (a, b) of the P2 element matrix (the (a, b) entry of FormT<FORM, 3, 2>::row(a))
template <int FORM>
__device__ __forceinline__ double wt_vv(const Geom<3>& G, int a, int b, const FormParams& prm) {
  constexpr double qs = Simplex<3>::q_same, qd = Simplex<3>::q_diff, l1 = Simplex<3>::l1;
  constexpr double cs = 16.0 * qs - 8.0 * l1 + 1.0, co = 16.0 * qd - 8.0 * l1 + 1.0;
  constexpr double m0 = p2_mass_const<3>(0), m1 = p2_mass_const<3>(1);
  const double k = (a == b ? cs : co) * dot<3>(G.g[a], G.g[b]);
  const double m = a == b ? m0 : m1;
  double v;
  if constexpr (FORM == F_MASS) v = m;
  else if constexpr (FORM == F_STIFFNESS) v = k;
  else v = fma(prm.p[0], m, k);
  return G.V * v;
}

#ifndef LOAM_GPU_WT_MINB
#define LOAM_GPU_WT_MINB 3
#endif

// NT consumer threads (one per edge row of the tile) + one TMA producer warp.
template <int FORM, int STAGES>
__global__ void __launch_bounds__(kWtConsumers + 32, LOAM_GPU_WT_MINB) k_wtile(const __grid_constant__ WtileArgs a) {
  constexpr int NT = kWtConsumers;
  using F = FormT<FORM, 3, 2>;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  int* slot_tile = reinterpret_cast<int*>(sm + 48);
  int4* slot_meta = reinterpret_cast<int4*>(sm + 128); // the stage's tile record, passed on by the producer
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) grid_dep_launch(); // PDL: the next kernel's prologue may start
  auto ring = [&](int k) { return sm + a.off_buf + (k % STAGES) * a.buf_bytes; };
  if (tid >= NT) { // ---- producer warp: tile blob + coordinate window by TMA
    const int lane = tid & 31;
    auto grab = [&]() {
      int t = 0;
      if (lane == 0) t = atomicAdd(a.next_tile, 1);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    int nt = grab();
    int4 nm[4];
    int2 nrun = make_int2(0, 0);
    auto prefetch = [&]() {
      if (nt < a.ntiles) {
        const int4* t = reinterpret_cast<const int4*>(a.tiles + 16 * nt);
#pragma unroll
        for (int q = 0; q < 4; ++q) nm[q] = __ldg(t + q);
        nrun = first_run(reinterpret_cast<const int2*>(a.runs) + nm[2].x, nm[2].y, lane);
      }
    };
    prefetch();
    grid_dep_wait(); // the caller's data only after the previous kernel (PDL)
    for (int k = 0;; ++k) {
      const int tile = nt;
      const int4 m0 = nm[0], m1 = nm[1], m2 = nm[2], m3 = nm[3];
      const int2 run0 = nrun;
      if (k >= STAGES) mbar_wait_sleep(&empty[k % STAGES], (k / STAGES - 1) & 1);
      if (tile >= a.ntiles) {
        if (lane == 0) {
          slot_tile[k % STAGES] = -1;
          mbar_arrive(&full[k % STAGES]);
        }
        break;
      }
      if (lane == 0) {
        slot_tile[k % STAGES] = tile;
        int4* sm4 = slot_meta + 4 * (k % STAGES);
        sm4[0] = m0;
        sm4[1] = m1;
        sm4[2] = m2;
        sm4[3] = m3;
      }
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % STAGES];
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + m2.x, m2.y, a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), 3};
      const uint32_t tx = (uint32_t)m0.y + stage_runs<false>(rc, lane, bar, run0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, tx);
        bulk_g2s(buf, a.blob + (int64_t)m0.x * 16, (uint32_t)m0.y, bar);
      }
      __syncwarp();
      stage_runs<true>(rc, lane, bar, run0);
      nt = grab();
      prefetch();
    }
    return;
  }
  grid_dep_wait(); // (PDL) before the consumers read or write anything of the caller's
  // ---- consumers
  double* seg0 = reinterpret_cast<double*>(sm + a.off_seg);
  const bool acc = a.accumulate != 0;
  auto put = [&](int pos, double v) { a.out[pos] = acc ? a.out[pos] + v : v; };
  for (int k = 0;; ++k) {
    mbar_wait_sleep(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    const int4* sm4 = slot_meta + 4 * (k % STAGES);
    const int4 m1 = sm4[1], m2 = sm4[2], m3 = sm4[3];
    const int n0 = sm4[0].z; // the tile's first row
    const int E0 = m1.x, len = m1.y, nitems = m1.z, off_s = m2.z, off_r = m2.w, off_p = m3.x, maxlv = m3.y;
    const unsigned char* buf = ring(k);
    const uint32_t* H = reinterpret_cast<const uint32_t*>(buf);
    const uint16_t* S = reinterpret_cast<const uint16_t*>(buf + off_s);
    const uint8_t* R = buf + off_r;
    const int32_t* P = reinterpret_cast<const int32_t*>(buf + off_p);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    double* seg = seg0 + (E0 & 1); // 16-byte parity of the global destination (bulk store)
    if (tid == 0) bulk_wait_read<0>(); // the previous tile's store has read the segment
    named_bar(1, NT);
    if (tid < nitems) {
      const uint32_t hdr = H[tid], own = H[NT + tid];
      double* row = seg + (hdr & 0xffffu);
      const int nce = (hdr >> 24) & 0xf;
      const bool isring = (hdr >> 28) & 1u;
      auto ld = [&](int slot, double (&x)[3]) {
        const double* p = win + 3 * slot;
        x[0] = p[0];
        x[1] = p[1];
        x[2] = p[2];
      };
      double X[4][3];
      ld(S[tid], X[0]);
      ld(S[NT + tid], X[1]);
      ld(S[2 * NT + tid], X[2]);
      double av = 0, aw = 0, ae = 0, avw = 0, dv = 0, dw = 0;
      double c0 = 0, c1 = 0, c2 = 0, f0 = 0, f1 = 0, f2 = 0;
      for (int i = 0; i < nce; ++i) {
        ld(S[(3 + i) * NT + tid], X[3]);
        Geom<3> G;
        geometry<3>(X, G);
        double o[10];
        F::row(9, G, nullptr, a.prm, o); // the row of local edge (0, 1) of the cell (v, w, p_i, p_{i+1})
        av += o[0];
        aw += o[1];
        ae += o[9];
        // p_i's columns p, (v,p), (w,p) = o[2], o[8], o[6]; p_{i+1}'s = o[3], o[7], o[5]; (p,q) = o[4]
        const double p0 = c0 + o[2], p1 = c1 + o[8], p2 = c2 + o[6];
        if (i == 0 && isring) { // completed by the last cell of the ring
          f0 = p0;
          f1 = p1;
          f2 = p2;
        } else {
          row[R[(3 + 3 * i) * NT + tid]] = p0;
          row[R[(4 + 3 * i) * NT + tid]] = p1;
          row[R[(5 + 3 * i) * NT + tid]] = p2;
          put(P[(6 + i) * NT + tid], p0);
        }
        c0 = o[3];
        c1 = o[7];
        c2 = o[5];
        row[R[(3 + 3 * maxlv + i) * NT + tid]] = o[4];
        avw += wt_vv<FORM>(G, 0, 1, a.prm);
        if ((own >> i) & 1u) dv += wt_vv<FORM>(G, 0, 0, a.prm);
        if ((own >> (12 + i)) & 1u) dw += wt_vv<FORM>(G, 1, 1, a.prm);
#pragma unroll
        for (int d = 0; d < 3; ++d) X[2][d] = X[3][d];
      }
      {
        const int j = isring ? 0 : nce; // the link vertex the walk ends at
        const double p0 = c0 + f0, p1 = c1 + f1, p2 = c2 + f2;
        row[R[(3 + 3 * j) * NT + tid]] = p0;
        row[R[(4 + 3 * j) * NT + tid]] = p1;
        row[R[(5 + 3 * j) * NT + tid]] = p2;
        put(P[(6 + j) * NT + tid], p0);
      }
      row[R[tid]] = av;
      row[R[NT + tid]] = aw;
      row[R[2 * NT + tid]] = ae;
      // the vertex rows, by symmetry: A[v][e], A[w][e], A[v][w] = A[w][v], and the diagonal shares
      put(P[tid], av);
      put(P[NT + tid], aw);
      put(P[2 * NT + tid], avw);
      put(P[3 * NT + tid], avw);
      if (a.dsum) { // deterministic: the shares in slots, summed per vertex in edge order (k_wt_dsum)
        const int64_t ei = (int64_t)(n0 - a.nverts) + (own >> 24);
        a.dsum[2 * ei] = dv;
        a.dsum[2 * ei + 1] = dw;
      } else {
        if (dv != 0.0) atomicAdd(a.out + P[4 * NT + tid], dv);
        if (dw != 0.0) atomicAdd(a.out + P[5 * NT + tid], dw);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]); // the stage's records and window are read
    if (acc) {
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] += seg[t];
    } else {
      fence_async_shared();
      named_bar(1, NT);
      if (tid == 0) {
        double* dst = a.out + E0;
        const int h = E0 & 1, t1 = len - ((E0 + len) & 1);
        if (h && len > 0) dst[0] = seg[0];
        if (t1 > h) {
          bulk_s2g(dst + h, seg + h, (uint32_t)(t1 - h) * 8);
          bulk_commit();
        }
        if (t1 < len && t1 >= h) dst[t1] = seg[t1];
      }
    }
  }
  if (tid == 0) bulk_wait_read<0>();
  tile_counter_release(a.next_tile, a.reset_tile, NT, tid);
}

template <int FORM>
void go_wtile(const WtilePlan& p, WtileArgs& a, int off, cudaStream_t s) {
  static const int st = std::getenv("LOAM_GPU_WT_STAGES") ? std::atoi(std::getenv("LOAM_GPU_WT_STAGES")) : 2;
  auto go = [&](auto kern, int stages) {
    const size_t smem = (size_t)off + stages * (size_t)a.buf_bytes;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kWtConsumers + 32, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "walk-tile kernel does not fit on an SM");
    if (std::getenv("LOAM_GPU_WT_INFO")) // developer: plan maxima behind the shared-memory footprint
      fprintf(stderr, "wtile: tiles %d max_seg %d max_blob %d max_slots %d smem %zu CTAs/SM %d\n", p.ntiles, p.max_seg,
              p.max_blob, p.max_slots, smem, blocks);
    launch_pdl(kern, dim3(std::min(p.ntiles, blocks * kNumSMs)), dim3(kWtConsumers + 32), smem, s, a);
  };
  if (st >= 2) go(k_wtile<FORM, 2>, 2);
  else go(k_wtile<FORM, 1>, 1);
}

} // namespace

void launch_wtile(const WtilePlan& p, int form, const double* coords, double* out, const FormParams& prm,
                  bool accumulate, int* next_tile, int* reset_tile, cudaStream_t s) {
  if (p.ntiles == 0) return;
  DevBuf<double> dsum;
  if (p.det) {
    dsum.alloc(2 * (size_t)std::max(p.nedges, 1), s);
  } else if (!accumulate) { // the vertex diagonals are RED-summed: start from zero
    k_wt_zero<<<ceil_div(p.nverts, 256), 256, 0, s>>>(out, p.dpos.get(), p.nverts);
    count_launch();
  }
  WtileArgs a{};
  a.dsum = p.det ? dsum.get() : nullptr;
  a.nverts = p.nverts;
  a.tiles = p.tiles.get();
  a.ntiles = p.ntiles;
  a.next_tile = next_tile;
  a.reset_tile = reset_tile;
  a.blob = p.blob.get();
  a.runs = p.runs.get();
  a.coords = coords;
  a.out = out;
  a.prm = prm;
  a.accumulate = accumulate ? 1 : 0;
  int off = 128 + 3 * 64; // barriers + per-stage tile records
  a.off_seg = off;
  off += up16((p.max_seg + 2) * 8);
  a.off_buf = off;
  a.b_win = up16(p.max_blob);
  a.buf_bytes = a.b_win + up16(p.max_slots * 3 * 8 + 16);
  if (form == F_MASS) go_wtile<F_MASS>(p, a, off, s);
  else if (form == F_STIFFNESS) go_wtile<F_STIFFNESS>(p, a, off, s);
  else go_wtile<F_HELMHOLTZ>(p, a, off, s);
  count_launch();
  if (p.det) {
    k_wt_dsum<<<ceil_div(p.nverts, 256), 256, 0, s>>>(p.dpos.get(), p.dptr.get(), p.dslots.get(), p.nverts, dsum.get(), out,
                                                      accumulate ? 1 : 0);
    count_launch();
  }
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
