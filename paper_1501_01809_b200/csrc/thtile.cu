// thtile.cu -- the Taylor-Hood Stokes blocks A, B, B^T in one launch (see thtile.cuh).
//
// Reference path replaced: fem::assemble_blocks (fem/assemble.hpp:439-448) ->
// three executes (parloop.hpp:191-384) of the Stokes element kernels (restated
// in elements.cuh FormT<F_STOKES_A/_B/_BT>), Mat::addto (data.hpp:205-222)
// into the patterns of build_sparsity (data.hpp:149-179).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "linkwalk.cuh"
#include "stage.cuh"
#include "thtile.cuh"

namespace loam_gpu {

namespace {

inline int up16(int x) { return (x + 15) & ~15; }

constexpr int kThConsumers = 128; // consumer threads per CTA = items per tile at most
constexpr int kNoSlot = 0xffff;

// local edge k of a P2 triangle row joins the local vertices (ea, eb) (space.hpp:66-71)
inline int ea(int k) { return Simplex<2>::edge_a(k); }
inline int eb(int k) { return Simplex<2>::edge_b(k); }

} // namespace

bool build_thtile(ThtilePlan& out, const ThtileSpec& sp, int ncells, int nnodes, int nverts, const int32_t* vnm,
                  const int32_t* xmap, const PairPlan& pp, const int64_t* rpA, int64_t nnzA, const int64_t* rpB,
                  int64_t nnzB, const int64_t* rpT, int64_t nnzT, cudaStream_t s) {
  constexpr int NT = kThConsumers;
  const int64_t lim = int64_t(1) << 31;
  if (pp.nrn != 6 || ncells == 0 || nnzA >= lim || nnzB >= lim || nnzT >= lim || nverts >= nnodes) return false;
  if (pp.npairs != (int64_t)ncells * 6) return false;
  const int spoke_items = std::min(sp.spoke_items, NT), edge_items = std::min(sp.edge_items, NT);
  auto hv = host_array<int32_t>((size_t)ncells * 6), hx = host_array<int32_t>((size_t)ncells * 3),
       hpairs = host_array<int32_t>((size_t)pp.npairs), hp = host_array<int32_t>(nnodes + 1);
  auto hA = host_array<int64_t>((size_t)nnodes * 2 + 1), hB = host_array<int64_t>((size_t)nverts + 1),
       hT = host_array<int64_t>((size_t)nnodes * 2 + 1);
  parallel_d2h({{hv.data(), vnm, sizeof(int32_t) * hv.size()},
                {hx.data(), xmap, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * hpairs.size()},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * hp.size()},
                {hA.data(), rpA, sizeof(int64_t) * hA.size()},
                {hB.data(), rpB, sizeof(int64_t) * hB.size()},
                {hT.data(), rpT, sizeof(int64_t) * hT.size()}},
               s);
  plan_tick("thtile: D2H", s);
  // the velocity map is a P2 map over the coordinate map: vertex nodes = vertex ids, edge nodes above
  {
    std::vector<char> bad(plan_threads(), 0);
    parallel_chunks(ncells, 1, [&](int t, int64_t c0, int64_t c1) {
      for (int64_t c = c0; c < c1; ++c) {
        const int32_t* r = &hv[(size_t)c * 6];
        const int32_t* x = &hx[(size_t)c * 3];
        bool ok = x[0] != x[1] && x[0] != x[2] && x[1] != x[2];
        for (int j = 0; j < 3; ++j) ok = ok && r[j] == x[j] && x[j] >= 0 && x[j] < nverts && r[3 + j] >= nverts;
        if (!ok) bad[t] = 1;
      }
    });
    for (char b : bad)
      if (b) return false;
  }
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs, roff;
    std::vector<uint8_t> blob;
    int max_seg = 0, max_slots = 0, max_blob = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nnodes, 1, [&](int t, int64_t cb0, int64_t cb1) {
    TileChunk& O = tch[t];
    struct Stamps { // calloc'd generation stamps: only the pages a chunk touches are mapped
      int* p;
      explicit Stamps(size_t n) : p(static_cast<int*>(std::calloc(n + 1, sizeof(int)))) {
        if (!p) throw std::bad_alloc();
      }
      ~Stamps() { std::free(p); }
    } vstamp(nverts);
    int gen = 0;
    auto fail = [&] { O.ok = false; };
    std::vector<int> vid, seq, cols, pcols;
    std::vector<std::pair<int, int>> rr;
    std::vector<int> base;
    LinkWalk lw;
    struct Item {
      int xs[4];        // coordinate ids v, w, p, q (-1: no such cell)
      uint8_t rec[16];
    };
    std::vector<Item> items;
    std::vector<uint8_t> dinfo;
    auto rank_in = [](const std::vector<int>& sorted, int x) {
      return (int)(std::lower_bound(sorted.begin(), sorted.end(), x) - sorted.begin());
    };
    auto put16 = [](uint8_t* p, int v) {
      p[0] = (uint8_t)(v & 0xff);
      p[1] = (uint8_t)(v >> 8);
    };
    // one tile: kind 0 = the spokes of vertices [n0, n1), kind 1 = edge nodes [n0, n1)
    auto emit = [&](int kind, int n0, int n1) {
      ++gen;
      vid.clear();
      for (const Item& it : items)
        for (int q = 0; q < 4; ++q) {
          const int x = it.xs[q];
          if (x >= 0 && vstamp.p[x] != gen) {
            vstamp.p[x] = gen;
            vid.push_back(x);
          }
        }
      const int slots = link_runs(vid, nverts, rr);
      if (slots > sp.tile_slots || (int)rr.size() > sp.tile_runs || slots >= kNoSlot) return false;
      base.resize(rr.size());
      for (size_t q = 0, acc = 0; q < rr.size(); ++q) {
        base[q] = (int)acc;
        acc += rr[q].second - rr[q].first;
      }
      auto slot_in = [&](int v) {
        if (v < 0) return kNoSlot;
        size_t q = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
        return base[q] + v - rr[q].first;
      };
      const int nitems = (int)items.size(), ni2 = (nitems + 1) & ~1, nv = kind == 0 ? n1 - n0 : 0;
      const int recb = kind == 0 ? 8 : 16;
      const int off_rec = 8 * ni2, off_d = off_rec + up16(recb * nitems), bytes = off_d + 16 * nv;
      const size_t b0 = O.blob.size();
      O.blob.resize(b0 + bytes, 0);
      uint8_t* bp = O.blob.data() + b0;
      for (int i = 0; i < nitems; ++i) {
        for (int q = 0; q < 4; ++q) put16(bp + 8 * i + 2 * q, slot_in(items[i].xs[q]));
        memcpy(bp + off_rec + recb * i, items[i].rec, recb);
      }
      if (nv) memcpy(bp + off_d, dinfo.data(), (size_t)16 * nv);
      const int64_t A0 = hA[(size_t)2 * n0], A1 = hA[(size_t)2 * n1], T0 = hT[(size_t)2 * n0], T1 = hT[(size_t)2 * n1];
      const int64_t B0 = kind == 0 ? hB[n0] : 0, B1 = kind == 0 ? hB[n1] : 0;
      // 16-byte aligned, even-length segments (bulk stores)
      if ((A0 | A1 | B0 | B1 | T0 | T1) & 1) return false;
      const int seg = (int)((A1 - A0) + (B1 - B0) + (T1 - T0));
      if (bytes >= (1 << 16) || A1 - A0 >= (1 << 16) || B1 - B0 >= (1 << 16) || T1 - T0 >= (1 << 16) ||
          (int)rr.size() >= (1 << 15))
        return false;
      // 8 meta ints + the first 4 window runs (the producer's chain holds no dependent load for them):
      // blob offset / 16 | bytes, kind << 16, nv << 20 | nitems, run offset << 8 (packed at merge) |
      // A, B, B^T value offsets | lenA, lenB << 16 | lenT, run count << 16
      int rec[16] = {(int)(b0 / 16), bytes | kind << 16 | nv << 20, nitems, (int)A0, (int)B0, (int)T0,
                     (int)(A1 - A0) | (int)(B1 - B0) << 16, (int)(T1 - T0) | (int)rr.size() << 16,
                     0, 0, 0, 0, 0, 0, 0, 0};
      for (size_t q = 0; q < rr.size() && q < 4; ++q) {
        rec[8 + 2 * q] = rr[q].first;
        rec[9 + 2 * q] = rr[q].second;
      }
      O.tiles.insert(O.tiles.end(), rec, rec + 16);
      O.roff.push_back((int)O.runs.size() / 2);
      for (auto& x : rr) O.runs.insert(O.runs.end(), {x.first, x.second});
      O.max_seg = std::max(O.max_seg, seg);
      O.max_slots = std::max(O.max_slots, slots);
      O.max_blob = std::max(O.max_blob, bytes);
      return true;
    };
    // ---- vertex rows: the spokes of each vertex, in star order
    struct StarCell {
      int c, lv, a, b; // cell, local index of v, the two other vertex ids
    };
    std::vector<StarCell> sc;
    std::vector<Item> vitems; // the vertex being added
    const int vend = (int)std::min<int64_t>(cb1, nverts);
    int v0 = (int)cb0;
    items.clear();
    dinfo.clear();
    for (int v = (int)cb0; v < vend; ++v) {
      sc.clear();
      lw.nn = 0;
      for (int p = hp[v]; p < hp[v + 1]; ++p) {
        const int c = hpairs[p] / 6, lv = hpairs[p] % 6;
        if (lv >= 3) return fail();
        const int a = hx[(size_t)c * 3 + (lv + 1) % 3], b = hx[(size_t)c * 3 + (lv + 2) % 3];
        sc.push_back({c, lv, a, b});
        if (!lw.add(a, a, b, b)) return fail();
      }
      const int nc = (int)sc.size();
      if (nc == 0) { // a vertex of no cell (sub-mesh loops): its rows must be empty, nothing to compute
        if (hA[(size_t)2 * v + 2] != hA[(size_t)2 * v] || hB[v + 1] != hB[v] || hT[(size_t)2 * v + 2] != hT[(size_t)2 * v])
          return fail();
        seq.assign(1, -1);
      } else if (nc + 1 > LinkWalk::kMax || !lw.walk(nc, seq)) {
        return fail();
      }
      const bool ring = nc > 0 && seq.front() == seq.back();
      const int k = nc == 0 ? 0 : ring ? nc : nc + 1; // spokes
      if (k > spoke_items) return fail();
      // cell i of the walk = (v, seq[i], seq[i + 1])
      auto cell_of = [&](int a, int b) -> const StarCell* {
        for (const StarCell& q : sc)
          if ((q.a == a && q.b == b) || (q.a == b && q.b == a)) return &q;
        return nullptr;
      };
      auto local_of = [&](const StarCell& q, int x) { // local index of vertex id x in q's cell
        for (int j = 0; j < 3; ++j)
          if (hx[(size_t)q.c * 3 + j] == x) return j;
        return -1;
      };
      auto edge_node = [&](const StarCell& q, int la, int lb) { return hv[(size_t)q.c * 6 + 3 + (3 - la - lb)]; };
      cols.clear();
      pcols.clear();
      cols.push_back(v);
      pcols.push_back(v);
      struct Spoke {
        int w, p, q, nvw, nwp;
      };
      Spoke spk[LinkWalk::kMax];
      for (int i = 0; i < k; ++i) {
        Spoke& S = spk[i];
        S.w = seq[i];
        const StarCell* P = i < nc ? cell_of(seq[i], seq[i + 1]) : nullptr;
        const int iq = i > 0 ? i - 1 : (ring ? k - 1 : -1);
        const StarCell* Q = iq >= 0 ? cell_of(seq[iq], seq[iq + 1 == k && ring ? nc : iq + 1]) : nullptr;
        if ((i < nc && !P) || (iq >= 0 && !Q)) return fail();
        S.p = P ? seq[i + 1] : -1;
        S.q = Q ? seq[iq] : -1;
        S.nvw = S.nwp = -1;
        if (P) {
          const int lw_ = local_of(*P, S.w);
          S.nvw = edge_node(*P, P->lv, lw_);
          S.nwp = hv[(size_t)P->c * 6 + 3 + P->lv]; // the edge opposite v
          cols.push_back(S.nwp);
        }
        if (Q) {
          const int lw_ = local_of(*Q, S.w);
          const int n2 = edge_node(*Q, Q->lv, lw_);
          if (S.nvw >= 0 && S.nvw != n2) return fail(); // two nodes on one mesh edge
          S.nvw = n2;
        }
        cols.push_back(S.w);
        cols.push_back(S.nvw);
        pcols.push_back(S.w);
      }
      if (nc == 0) { // empty rows
        cols.clear();
        pcols.clear();
      }
      std::sort(cols.begin(), cols.end());
      std::sort(pcols.begin(), pcols.end());
      if (std::adjacent_find(cols.begin(), cols.end()) != cols.end()) return fail();
      const int L = (int)cols.size(), Lp = (int)pcols.size();
      const int64_t a0 = hA[(size_t)2 * v], a1 = hA[(size_t)2 * v + 1], a2 = hA[(size_t)2 * v + 2];
      const int64_t t0 = hT[(size_t)2 * v], t1 = hT[(size_t)2 * v + 1], t2 = hT[(size_t)2 * v + 2];
      if (a1 - a0 != 2 * L || a2 - a1 != 2 * L || hB[v + 1] - hB[v] != 2 * L || t1 - t0 != Lp || t2 - t1 != Lp ||
          L > 255 || Lp > 255)
        return fail();
      // close the tile before this vertex when it no longer fits
      auto fits = [&] {
        return (int)items.size() + k <= spoke_items && v - v0 < NT && hA[(size_t)2 * v + 2] - hA[(size_t)2 * v0] < 60000 &&
               hT[(size_t)2 * v + 2] - hT[(size_t)2 * v0] < 60000;
      };
      if (v > v0 && !fits()) {
        if (!items.empty() && !emit(0, v0, v)) return fail();
        items.clear();
        dinfo.clear();
        v0 = v;
      }
      uint8_t d[16] = {0};
      put16(d + 0, (int)(a0 - hA[(size_t)2 * v0]));
      put16(d + 2, (int)(hB[v] - hB[v0]));
      put16(d + 4, (int)(t0 - hT[(size_t)2 * v0]));
      d[6] = (uint8_t)L;
      d[7] = (uint8_t)Lp;
      d[8] = (uint8_t)rank_in(cols, v);
      d[9] = (uint8_t)rank_in(pcols, v);
      d[10] = (uint8_t)items.size();
      d[11] = (uint8_t)k;
      dinfo.insert(dinfo.end(), d, d + 16);
      for (int i = 0; i < k; ++i) {
        const Spoke& S = spk[i];
        Item it{};
        it.xs[0] = v;
        it.xs[1] = S.w;
        it.xs[2] = S.p;
        it.xs[3] = S.q;
        it.rec[0] = (uint8_t)(v - v0);
        it.rec[1] = (uint8_t)rank_in(cols, S.w);
        it.rec[2] = (uint8_t)rank_in(cols, S.nvw);
        it.rec[3] = (uint8_t)(S.nwp >= 0 ? rank_in(cols, S.nwp) : 0);
        it.rec[4] = (uint8_t)rank_in(pcols, S.w);
        it.rec[5] = (uint8_t)((S.p >= 0 ? 1 : 0) | (S.q >= 0 ? 2 : 0));
        items.push_back(it);
      }
    }
    if (!items.empty() && !emit(0, v0, vend)) return fail();
    // ---- edge rows
    items.clear();
    dinfo.clear();
    const int e_begin = (int)std::max<int64_t>(cb0, nverts), eend = (int)cb1;
    int e0 = e_begin;
    for (int e = e_begin; e < eend; ++e) {
      const int nce = hp[e + 1] - hp[e];
      if (nce == 0) { // a node of no cell: empty rows
        if (hA[(size_t)2 * e + 2] != hA[(size_t)2 * e] || hT[(size_t)2 * e + 2] != hT[(size_t)2 * e]) return fail();
        continue;
      }
      if (nce > 2) return fail();
      int xv = -1, xw = -1, xo[2] = {-1, -1}, nvo[2] = {-1, -1}, nwo[2] = {-1, -1};
      for (int q = 0; q < nce; ++q) {
        const int c = hpairs[hp[e] + q] / 6, l = hpairs[hp[e] + q] % 6;
        if (l < 3) return fail();
        const int k = l - 3;
        int la = ea(k), lb = eb(k);
        const int32_t* x = &hx[(size_t)c * 3];
        if (q == 0) {
          xv = x[la];
          xw = x[lb];
        } else {
          if (x[la] == xw && x[lb] == xv) std::swap(la, lb);
          else if (!(x[la] == xv && x[lb] == xw)) return fail(); // one node on two mesh edges
        }
        xo[q] = x[k];                                   // the vertex opposite the edge
        nvo[q] = hv[(size_t)c * 6 + 3 + lb];            // edge node (v, opposite)
        nwo[q] = hv[(size_t)c * 6 + 3 + la];            // edge node (w, opposite)
      }
      if (nce == 2 && xo[0] == xo[1]) return fail();
      // device order: v, w, e, p, (w,p), (v,p), q, (w,q), (v,q) | v, w, p, q
      const int order[9] = {xv, xw, e, xo[0], nwo[0], nvo[0], xo[1], nwo[1], nvo[1]};
      const int porder[4] = {xv, xw, xo[0], xo[1]};
      const int L = nce == 2 ? 9 : 6, Lp = nce == 2 ? 4 : 3;
      cols.assign(order, order + L);
      pcols.assign(porder, porder + Lp);
      std::sort(cols.begin(), cols.end());
      std::sort(pcols.begin(), pcols.end());
      if (std::adjacent_find(cols.begin(), cols.end()) != cols.end()) return fail();
      const int64_t a0 = hA[(size_t)2 * e], a1 = hA[(size_t)2 * e + 1], a2 = hA[(size_t)2 * e + 2];
      const int64_t t0 = hT[(size_t)2 * e], t1 = hT[(size_t)2 * e + 1], t2 = hT[(size_t)2 * e + 2];
      if (a1 - a0 != 2 * L || a2 - a1 != 2 * L || t1 - t0 != Lp || t2 - t1 != Lp) return fail();
      if ((int)items.size() == edge_items || a2 - hA[(size_t)2 * e0] >= 60000 || t2 - hT[(size_t)2 * e0] >= 60000) {
        if (!emit(1, e0, e)) return fail();
        items.clear();
        e0 = e;
      }
      Item it{};
      it.xs[0] = xv;
      it.xs[1] = xw;
      it.xs[2] = xo[0];
      it.xs[3] = xo[1];
      put16(it.rec + 0, (int)(a0 - hA[(size_t)2 * e0]));
      put16(it.rec + 2, (int)(t0 - hT[(size_t)2 * e0]));
      it.rec[4] = (uint8_t)(L | (nce == 2 ? 0x80 : 0));
      it.rec[5] = (uint8_t)Lp;
      for (int j = 0; j < L; ++j) it.rec[6 + j] = (uint8_t)rank_in(cols, order[j]);
      int packed = 0;
      for (int j = 0; j < Lp; ++j) packed |= rank_in(pcols, porder[j]) << (2 * j);
      it.rec[15] = (uint8_t)packed;
      items.push_back(it);
    }
    if (!items.empty() && !emit(1, e0, eend)) return fail();
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
      const int64_t ro = (int64_t)O.roff[q / 16] + rshift;
      if (ro >= (1 << 23)) return false;
      O.tiles[q + 2] |= (int)ro << 8;
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
  plan_tick("thtile: tiles", s);
  upload_parts(out.blob, parts, s);
  tch.clear();
  out.ntiles = (int)tiles.size() / 16;
  auto upload = [&](auto& dst, const auto& src) {
    using T = typename std::decay_t<decltype(src)>::value_type;
    dst.alloc(src.size() + 16, s);
    if (!src.empty())
      LG_CUDA(cudaMemcpyAsync(dst.get(), src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
  };
  upload(out.tiles, tiles);
  upload(out.runs, runs);
  LG_CUDA(cudaStreamSynchronize(s));
  return true;
}

// ===========================================================================
// Device side
// ===========================================================================

namespace {

struct ThtileArgs {
  const int32_t* tiles;
  int ntiles;
  const uint8_t* blob;
  const int32_t* runs;
  const double* coords;
  double* outA;
  double* outB;
  double* outT;
  double nu;
  int acc;
  int off_seg, off_scr, off_buf, buf_bytes, b_win;
};

#ifndef LOAM_GPU_TH_MINB
#define LOAM_GPU_TH_MINB 4
#endif

__device__ __forceinline__ void th_load(const double* win, int slot, double (&x)[2]) {
  const double2 p = *reinterpret_cast<const double2*>(win + 2 * slot);
  x[0] = p.x;
  x[1] = p.y;
}

// NT consumer threads (one per item of the tile) + one TMA producer warp.
template <int STAGES>
__global__ void __launch_bounds__(kThConsumers + 32, LOAM_GPU_TH_MINB) k_thtile(const __grid_constant__ ThtileArgs a) {
  constexpr int NT = kThConsumers;
  using FA = FormT<F_STOKES_A, 2, 2>;
  using FB = FormT<F_STOKES_B, 2, 2>;
  using FT = FormT<F_STOKES_BT, 2, 2>;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  int* slot_tile = reinterpret_cast<int*>(sm + 48);
  // tile records of this CTA, 8 tiles per batch, double-buffered (cp.async);
  // the meta of the tile in each stage, handed to the consumers with it
  __shared__ __align__(16) int meta_s[2][8 * 16];
  __shared__ int stage_meta[STAGES][8];
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
    // Static schedule (tile k of this CTA = blockIdx + k * grid; spoke tiles
    // first, edge tiles after, so every CTA gets the same mix).  The 64-byte
    // records (meta + the first window runs) arrive 8 tiles at a time by
    // cp.async, one batch ahead: no dependent global round trip per tile (a
    // dynamic counter cost an atomic, a record load and a run load per tile,
    // and the consumers spent 39 % of their stall samples waiting for data).
    const int lane = tid & 31;
    auto load_batch = [&](int b) { // tiles 8b..8b+7 -> meta_s[b & 1]; lane = (tile in batch, 16-byte part)
      const int kk = 8 * b + (lane >> 2), part = lane & 3;
      const int tile = blockIdx.x + kk * gridDim.x;
      if (tile < a.ntiles) cp_async16(&meta_s[b & 1][(lane >> 2) * 16 + part * 4], a.tiles + 16 * tile + part * 4);
      cp_async_commit();
    };
    load_batch(0);
    load_batch(1);
    for (int k = 0;; ++k) {
      const int tile = blockIdx.x + k * gridDim.x;
      if (k % 8 == 0) {
        cp_async_wait<1>(); // batch k / 8 has landed (the next one may still be in flight)
        __syncwarp();
      }
      const int* rec = &meta_s[(k / 8) & 1][(k % 8) * 16];
      int2 run0 = make_int2(0, 0);
      int cnt = 0, run_off = 0, m0 = 0, m1 = 0, mine = 0;
      if (tile < a.ntiles) { // (past the end the batch slot was never filled)
        m0 = rec[0];
        m1 = rec[1];
        mine = rec[lane & 7];
        cnt = rec[7] >> 16;
        run_off = (int)((unsigned)rec[2] >> 8);
        if (lane < cnt)
          run0 = lane < 4 ? reinterpret_cast<const int2*>(rec + 8)[lane]
                          : __ldg(reinterpret_cast<const int2*>(a.runs) + run_off + lane);
      }
      if (k % 8 == 7) {
        __syncwarp(); // every lane has read batch k / 8: refill its buffer
        load_batch(k / 8 + 2);
      }
      if (k >= STAGES) mbar_wait_sleep(&empty[k % STAGES], (k / STAGES - 1) & 1);
      if (tile >= a.ntiles) { // publish "no more tiles" through the stage
        if (lane == 0) {
          slot_tile[k % STAGES] = -1;
          mbar_arrive(&full[k % STAGES]);
        }
        break;
      }
      if (lane < 8) stage_meta[k % STAGES][lane] = mine;
      if (lane == 0) slot_tile[k % STAGES] = tile;
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % STAGES];
      const uint32_t bytes = (uint32_t)m1 & 0xffffu;
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + run_off, cnt, a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), 2};
      if (lane == 0) { // the plan's records (library-owned, immutable: safe before the PDL wait)
        mbar_expect_tx(bar, bytes);
        bulk_g2s(buf, a.blob + (int64_t)m0 * 16, bytes, bar);
      }
      if (k == 0) grid_dep_wait(); // the caller's coordinates only after the previous kernel (PDL)
      const uint32_t tx = stage_runs<false>(rc, lane, bar, run0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(bar, tx);
      __syncwarp();
      stage_runs<true>(rc, lane, bar, run0);
    }
    cp_async_wait<0>();
    return;
  }
  grid_dep_wait(); // (PDL) before the consumers read or write anything of the caller's
  // ---- consumers
  double* seg0 = reinterpret_cast<double*>(sm + a.off_seg);
  double* scr = reinterpret_cast<double*>(sm + a.off_scr);
  FormParams prm{{a.nu, 0, 0, 0}};
  for (int k = 0;; ++k) {
    mbar_wait_sleep(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    const int* sm8 = stage_meta[k % STAGES];
    const int m1 = sm8[1], m2 = sm8[2], m6 = sm8[6], m7 = sm8[7];
    const int kind = (m1 >> 16) & 0xf, nv = (m1 >> 20) & 0xff, nitems = m2 & 0xff, E0A = sm8[3], E0B = sm8[4],
              E0T = sm8[5], lenA = m6 & 0xffff, lenB = (int)((unsigned)m6 >> 16), lenT = m7 & 0xffff;
    const int off_rec = 8 * ((nitems + 1) & ~1), off_d = off_rec + (((kind == 0 ? 8 : 16) * nitems + 15) & ~15);
    const unsigned char* buf = ring(k);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    double* sA = seg0;
    double* sB = sA + lenA;
    double* sT = sB + lenB;
    const bool on = tid < nitems;
    if (kind == 1) {
      // ---- edge rows: node e = (v, w) with its cells (v, w, p) and (v, w, q)
      double av = 0, aw = 0, ae = 0, ap = 0, awp = 0, avp = 0, aq = 0, awq = 0, avq = 0;
      double tv[2] = {0, 0}, tw[2] = {0, 0}, tp[2] = {0, 0}, tq[2] = {0, 0};
      uint4 rec = make_uint4(0, 0, 0, 0);
      if (on) {
        const uint2 sl = reinterpret_cast<const uint2*>(buf)[tid];
        rec = reinterpret_cast<const uint4*>(buf + off_rec)[tid];
        double X[3][2];
        th_load(win, sl.x & 0xffffu, X[0]);
        th_load(win, sl.x >> 16, X[1]);
        th_load(win, sl.y & 0xffffu, X[2]);
        Geom<2> G;
        geometry<2>(X, G);
        double K[6], o[6];
        p2_rows<2, true, false>(5, G, K, nullptr);
        FT::row(5, G, nullptr, prm, o);
        const double sc = a.nu * G.V;
        av = sc * K[0];
        aw = sc * K[1];
        ap = sc * K[2];
        awp = sc * K[3];
        avp = sc * K[4];
        ae = sc * K[5];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          tv[c] = o[c * 3 + 0];
          tw[c] = o[c * 3 + 1];
          tp[c] = o[c * 3 + 2];
        }
        if (rec.y & 0x80u) { // (byte 4 bit 7) the second cell
          th_load(win, sl.y >> 16, X[2]);
          geometry<2>(X, G);
          p2_rows<2, true, false>(5, G, K, nullptr);
          FT::row(5, G, nullptr, prm, o);
          const double sq = a.nu * G.V;
          av = fma(sq, K[0], av);
          aw = fma(sq, K[1], aw);
          aq = sq * K[2];
          awq = sq * K[3];
          avq = sq * K[4];
          ae = fma(sq, K[5], ae);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            tv[c] += o[c * 3 + 0];
            tw[c] += o[c * 3 + 1];
            tq[c] = o[c * 3 + 2];
          }
        }
      }
      if (tid == 0) bulk_wait_read<0>(); // the previous tile's stores have read the segments
      named_bar(1, NT);
      if (on) {
        const int baseA = rec.x & 0xffffu, baseT = rec.x >> 16, L = rec.y & 0x7fu, Lp = (rec.y >> 8) & 0xffu;
        const bool two = rec.y & 0x80u;
        // ranks: bytes 6..14 = v, w, e, p, (w,p), (v,p), q, (w,q), (v,q); byte 15 = B^T ranks, 2 bits each
        double* r0 = sA + baseA;
        double* r1 = r0 + 2 * L;
        auto putA = [&](uint32_t r, double v) {
          *reinterpret_cast<double2*>(r0 + 2 * r) = make_double2(v, 0.0);
          *reinterpret_cast<double2*>(r1 + 2 * r) = make_double2(0.0, v);
        };
        putA((rec.y >> 16) & 0xffu, av);
        putA(rec.y >> 24, aw);
        putA(rec.z & 0xffu, ae);
        putA((rec.z >> 8) & 0xffu, ap);
        putA((rec.z >> 16) & 0xffu, awp);
        putA(rec.z >> 24, avp);
        const uint32_t pk = rec.w >> 24;
        double* t0 = sT + baseT;
        double* t1 = t0 + Lp;
        t0[pk & 3u] = tv[0];
        t1[pk & 3u] = tv[1];
        t0[(pk >> 2) & 3u] = tw[0];
        t1[(pk >> 2) & 3u] = tw[1];
        t0[(pk >> 4) & 3u] = tp[0];
        t1[(pk >> 4) & 3u] = tp[1];
        if (two) {
          putA(rec.w & 0xffu, aq);
          putA((rec.w >> 8) & 0xffu, awq);
          putA((rec.w >> 16) & 0xffu, avq);
          t0[(pk >> 6) & 3u] = tq[0];
          t1[(pk >> 6) & 3u] = tq[1];
        }
      }
    } else {
      // ---- vertex rows: spoke v -> w with the cells (v, w, p) [owned] and (v, w, q)
      double a_w = 0, a_vw = 0, a_wp = 0, dA = 0;
      double b_w[2] = {0, 0}, b_vw[2] = {0, 0}, b_wp[2] = {0, 0}, dB[2] = {0, 0}, t_w[2] = {0, 0};
      uint2 rec = make_uint2(0, 0);
      if (on) {
        const uint2 sl = reinterpret_cast<const uint2*>(buf)[tid];
        rec = reinterpret_cast<const uint2*>(buf + off_rec)[tid];
        const uint32_t fl = (rec.y >> 8) & 0xffu;
        double X[3][2];
        th_load(win, sl.x & 0xffffu, X[0]);
        th_load(win, sl.x >> 16, X[1]);
        Geom<2> G;
        double K[6], ob[12], ot[6];
        if (fl & 1u) {
          th_load(win, sl.y & 0xffffu, X[2]);
          geometry<2>(X, G);
          p2_rows<2, true, false>(0, G, K, nullptr);
          FB::row(0, G, nullptr, prm, ob);
          FT::row(0, G, nullptr, prm, ot);
          const double sc = a.nu * G.V;
          a_w = sc * K[1];
          a_vw = sc * K[5];
          a_wp = sc * K[3];
          dA = sc * K[0];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            b_w[c] = ob[2 + c];
            b_vw[c] = ob[10 + c];
            b_wp[c] = ob[6 + c];
            dB[c] = ob[c];
            t_w[c] = ot[c * 3 + 1];
          }
        }
        if (fl & 2u) {
          th_load(win, sl.y >> 16, X[2]);
          geometry<2>(X, G);
          p2_rows<2, true, false>(0, G, K, nullptr);
          FB::row(0, G, nullptr, prm, ob);
          FT::row(0, G, nullptr, prm, ot);
          const double sq = a.nu * G.V;
          a_w = fma(sq, K[1], a_w);
          a_vw = fma(sq, K[5], a_vw);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            b_w[c] += ob[2 + c];
            b_vw[c] += ob[10 + c];
            t_w[c] += ot[c * 3 + 1];
          }
        }
      }
      if (tid == 0) bulk_wait_read<0>();
      named_bar(1, NT);
      const uint4* dinfo = reinterpret_cast<const uint4*>(buf + off_d);
      if (on) {
        const uint4 d = dinfo[rec.x & 0xffu];
        const int baseA = d.x & 0xffffu, baseB = d.x >> 16, baseT = d.y & 0xffffu, L = (d.y >> 16) & 0xffu,
                  Lp = d.y >> 24;
        const uint32_t rw = (rec.x >> 8) & 0xffu, rvw = (rec.x >> 16) & 0xffu, rwp = rec.x >> 24,
                       rtw = rec.y & 0xffu, fl = (rec.y >> 8) & 0xffu;
        double* r0 = sA + baseA;
        double* r1 = r0 + 2 * L;
        double* rb = sB + baseB;
        auto put = [&](uint32_t r, double v, const double (&b)[2]) {
          *reinterpret_cast<double2*>(r0 + 2 * r) = make_double2(v, 0.0);
          *reinterpret_cast<double2*>(r1 + 2 * r) = make_double2(0.0, v);
          *reinterpret_cast<double2*>(rb + 2 * r) = make_double2(b[0], b[1]);
        };
        put(rw, a_w, b_w);
        put(rvw, a_vw, b_vw);
        if (fl & 1u) put(rwp, a_wp, b_wp);
        sT[baseT + rtw] = t_w[0];
        sT[baseT + Lp + rtw] = t_w[1];
        scr[3 * tid] = dA;
        scr[3 * tid + 1] = dB[0];
        scr[3 * tid + 2] = dB[1];
      }
      named_bar(1, NT);
      // the (v, v) entries: the spokes' owned cells in star order
      if (tid < nv) {
        const uint4 d = dinfo[tid];
        const int baseA = d.x & 0xffffu, baseB = d.x >> 16, baseT = d.y & 0xffffu, L = (d.y >> 16) & 0xffu,
                  Lp = d.y >> 24;
        const uint32_t selfA = d.z & 0xffu, selfT = (d.z >> 8) & 0xffu, first = (d.z >> 16) & 0xffu, ns = d.z >> 24;
        double s0 = 0, s1 = 0, s2 = 0;
        for (uint32_t i = 0; i < ns; ++i) {
          s0 += scr[3 * (first + i)];
          s1 += scr[3 * (first + i) + 1];
          s2 += scr[3 * (first + i) + 2];
        }
        if (ns) { // (a vertex of no cell has empty rows)
          double* r0 = sA + baseA + 2 * selfA;
          *reinterpret_cast<double2*>(r0) = make_double2(s0, 0.0);
          *reinterpret_cast<double2*>(r0 + 2 * L) = make_double2(0.0, s0);
          *reinterpret_cast<double2*>(sB + baseB + 2 * selfA) = make_double2(s1, s2);
          sT[baseT + selfT] = s1;
          sT[baseT + Lp + selfT] = s2;
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]); // the stage's records and window are read
    if (a.acc) { // add to the blocks that are not fresh
      named_bar(1, NT);
      if (a.acc & 1)
        for (int t = tid; t < lenA; t += NT) sA[t] += a.outA[(int64_t)E0A + t];
      if (a.acc & 2)
        for (int t = tid; t < lenB; t += NT) sB[t] += a.outB[(int64_t)E0B + t];
      if (a.acc & 4)
        for (int t = tid; t < lenT; t += NT) sT[t] += a.outT[(int64_t)E0T + t];
    }
    fence_async_shared();
    named_bar(1, NT);
    if (tid == 0) {
      if (lenA) bulk_s2g(a.outA + E0A, sA, (uint32_t)lenA * 8);
      if (lenB) bulk_s2g(a.outB + E0B, sB, (uint32_t)lenB * 8);
      if (lenT) bulk_s2g(a.outT + E0T, sT, (uint32_t)lenT * 8);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_read<0>();
}

} // namespace

void launch_thtile(const ThtilePlan& p, const double* coords, double* A, double* B, double* BT, double nu, int acc,
                   cudaStream_t s) {
  if (p.ntiles == 0) return;
  ThtileArgs a{};
  a.tiles = p.tiles.get();
  a.ntiles = p.ntiles;
  a.blob = p.blob.get();
  a.runs = p.runs.get();
  a.coords = coords;
  a.outA = A;
  a.outB = B;
  a.outT = BT;
  a.nu = nu;
  a.acc = acc;
  int off = 128; // barriers, stage tiles
  a.off_seg = off;
  off += up16(p.max_seg * 8 + 16);
  a.off_scr = off;
  off += kThConsumers * 3 * 8;
  a.off_buf = off;
  a.b_win = up16(p.max_blob);
  a.buf_bytes = a.b_win + up16(p.max_slots * 2 * 8 + 16);
  static const int st = std::getenv("LOAM_GPU_TH_STAGES") ? std::atoi(std::getenv("LOAM_GPU_TH_STAGES")) : 2;
  auto go = [&](auto kern, int stages) {
    const size_t smem = (size_t)off + stages * (size_t)a.buf_bytes;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kThConsumers + 32, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "Taylor-Hood tile kernel does not fit on an SM");
    if (std::getenv("LOAM_GPU_TH_INFO")) // developer: plan maxima behind the shared-memory footprint
      fprintf(stderr, "thtile: tiles %d max_seg %d max_blob %d max_slots %d smem %zu CTAs/SM %d\n", p.ntiles, p.max_seg,
              p.max_blob, p.max_slots, smem, blocks);
    launch_pdl(kern, dim3(std::min(p.ntiles, blocks * kNumSMs)), dim3(kThConsumers + 32), smem, s, a);
  };
  if (st >= 3) go(k_thtile<3>, 3);
  else if (st == 2) go(k_thtile<2>, 2);
  else go(k_thtile<1>, 1);
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
