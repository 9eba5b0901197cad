// etile.cu -- edge-tile assembly of scalar P2 matrices (see etile.cuh).
//
// Reference path replaced: assemble_matrix (fem/assemble.hpp:85-104) ->
// execute (parloop.hpp:191-384) with the P2 mass / stiffness / helmholtz
// element kernels (fem/form.hpp:201-320) and Mat::addto (data.hpp:205-222).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "async.cuh"
#include "etile.cuh"
#include "stage.cuh"

namespace loam_gpu {

int et_stages();

namespace {

const int kTriE[3][2] = {{1, 2}, {0, 2}, {0, 1}};                          // space.hpp:66-71
const int kTetE[6][2] = {{2, 3}, {1, 3}, {1, 2}, {0, 3}, {0, 2}, {0, 1}};  // elements.cuh Simplex<3>

int edge_index(int gd, int x, int y) {
  const int ne = gd == 2 ? 3 : 6;
  const int (*E)[2] = gd == 2 ? kTriE : kTetE;
  if (x > y) std::swap(x, y);
  for (int f = 0; f < ne; ++f)
    if (E[f][0] == x && E[f][1] == y) return f;
  return -1;
}

// packed upper-triangle index of the Gram entry (p, q) of nv vertices
int gram_index(int nv, int p, int q) {
  if (p > q) std::swap(p, q);
  int idx = 0;
  for (int r = 0; r < p; ++r) idx += nv - r;
  return idx + (q - p);
}

// windows of contiguous vertex ids (even-aligned runs, as the ptile plan)
int make_runs(std::vector<int>& ids, int limit, std::vector<std::pair<int, int>>& rr) {
  constexpr int kGap = 8;
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
}

inline int up16(int x) { return (x + 15) & ~15; }

} // namespace

bool build_etile(EtilePlan& out, const EtileSpec& sp, int gd, int ncells, int nrows_node,
                 const int32_t* sorted_rows, const int32_t* sorted_x, int nverts, const PairPlan& pp,
                 const int64_t* row_ptr, int64_t nnz, int cd, cudaStream_t s) {
  const int nv = gd + 1, ne = gd == 2 ? 3 : 6, nrn = nv + ne;
  if (cd != 1 && cd != 2) return false;
  const int (*E)[2] = gd == 2 ? kTriE : kTetE;
  if (pp.nrn != nrn || pp.ncn != nrn || nnz >= (int64_t(1) << 31) || ncells == 0 || ncells >= (1 << 30))
    return false;
  const int64_t np = pp.npairs;
  auto hrows = host_array<int32_t>((size_t)ncells * nrn), hx = host_array<int32_t>((size_t)ncells * nv),
       hpairs = host_array<int32_t>(np), hp = host_array<int32_t>(nrows_node + 1);
  auto hrank = host_array<uint8_t>((size_t)np * nrn);
  auto hrp = host_array<int64_t>((size_t)nrows_node * cd + 1);
  parallel_d2h({{hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size()},
                {hx.data(), sorted_x, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * (size_t)np},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * (size_t)(nrows_node + 1)},
                {hrank.data(), pp.ranks.get(), hrank.size()},
                {hrp.data(), row_ptr, sizeof(int64_t) * hrp.size()}},
               s);
  plan_tick("etile: D2H", s);
  // node-level pattern offsets (a cd x cd component-blocked CSR: node row i owns
  // dof rows cd*i .. cd*i+cd-1, each cd * L_i long)
  if (cd > 1) {
    for (int i = 0; i <= nrows_node; ++i) hrp[i] = hrp[(size_t)i * cd] / (cd * cd);
    hrp.resize(nrows_node + 1);
  }
  // value position of node entry (row node v, in-row rank): the (cd*v, cd*w) dof entry
  auto vpos = [&](int v, int rank) { return (int32_t)(cd * cd * hrp[v] + cd * rank); };
  auto vlen = [&](int v) { return (int32_t)(cd * (hrp[v + 1] - hrp[v])); }; // dof row length
  // ---- node roles: vertex nodes (local 0..gd) numbered before edge nodes
  std::vector<int8_t> role(nrows_node, 0);
  for (int c = 0; c < ncells; ++c)
    for (int i = 0; i < nrn; ++i) {
      const int node = hrows[(size_t)c * nrn + i];
      const int8_t r = i < nv ? 1 : 2;
      if (role[node] && role[node] != r) return false;
      role[node] = r;
    }
  int maxv = -1, mine = INT_MAX;
  for (int n = 0; n < nrows_node; ++n) {
    if (role[n] == 1) maxv = n;
    if (role[n] == 2) mine = std::min(mine, n);
  }
  if (mine == INT_MAX || maxv >= mine) return false;
  const int E0 = mine, nedge = nrows_node - E0;
  for (int n = E0; n < nrows_node; ++n)
    if (role[n] != 2) return false;
  // ---- edge node <-> vertex pair bijection
  std::vector<int32_t> eA(nedge), eB(nedge);
  std::vector<uint64_t> keys(nedge);
  for (int e = 0; e < nedge; ++e) {
    const int r = E0 + e;
    for (int p = hp[r]; p < hp[r + 1]; ++p) {
      const int c = hpairs[p] / nrn, k = hpairs[p] % nrn - nv;
      int a = hrows[(size_t)c * nrn + E[k][0]], b = hrows[(size_t)c * nrn + E[k][1]];
      if (a > b) std::swap(a, b);
      if (p == hp[r]) {
        eA[e] = a;
        eB[e] = b;
      } else if (a != eA[e] || b != eB[e]) {
        return false;
      }
    }
    keys[e] = (uint64_t)(uint32_t)eA[e] << 32 | (uint32_t)eB[e];
  }
  {
    // strictly increasing keys (the lexicographic edge numbering of
    // space.hpp:48-57) are distinct without a sort
    bool increasing = true;
    for (size_t e = 1; e < keys.size() && increasing; ++e) increasing = keys[e - 1] < keys[e];
    if (!increasing) {
      std::vector<uint64_t> ks(keys);
      std::sort(ks.begin(), ks.end());
      if (std::adjacent_find(ks.begin(), ks.end()) != ks.end()) return false;
    }
  }
  auto find_pair = [&](int w, int c) -> int64_t {
    for (int p = hp[w]; p < hp[w + 1]; ++p)
      if (hpairs[p] / nrn == c) return p;
    return -1;
  };
  plan_tick("etile: roles + edge keys", s);
  // ---- vertex diagonals
  std::vector<int32_t> dpos(E0, -1), diag;
  for (int v = 0; v < E0; ++v)
    if (hp[v + 1] > hp[v]) {
      const int p = hp[v], i = hpairs[p] % nrn;
      dpos[v] = vpos(v, hrank[(size_t)p * nrn + i]);
      diag.push_back(dpos[v]);
      if (cd == 2) diag.push_back(vlen(v));
    }
  // diagonal contribution of (cell, local vertex v) is carried by local edge (0,1) for
  // v = 0 and (0,v) otherwise
  auto assigned = [&](int v) { return edge_index(gd, 0, v == 0 ? 1 : v); };
  // ---- index table: per (local edge k, orientation) the Gram entries the canonical row reads
  const int ca = nv - 2, cb = nv - 1;
  uint32_t ktab[12] = {};
  auto sigma_of = [&](int k, int swap, int* sig) {
    const int la = E[k][swap], lb = E[k][1 - swap];
    sig[ca] = la;
    sig[cb] = lb;
    int q = 0;
    for (int v = 0; v < nv; ++v)
      if (v != la && v != lb) sig[q++] = v;
  };
  for (int k = 0; k < ne; ++k) // canonical vertex m <- original local vertex sigma(m), 4 bits each
    for (int sw = 0; sw < 2; ++sw) {
      int sig[4];
      sigma_of(k, sw, sig);
      uint32_t w = 0;
      for (int m = 0; m < nv; ++m) w |= (uint32_t)sig[m] << (4 * m);
      ktab[k * 2 + sw] = w;
    }
  // ---- per edge row: transposed positions, vertex-pair positions, records
  // (rows are independent: chunks of rows on all host cores, the variable-
  // length transposed-position lists concatenated in row order afterwards)
  const int rb = (2 + nrn + 3) & ~3;
  const int64_t p0e = hp[E0], npe = hp[nrows_node] - p0e;
  std::vector<int32_t> tptr(nedge + 1, 0), tpos, tlen;
  auto cellof = host_array<int32_t>(npe);
  std::vector<int4> xpos(nedge);
  std::vector<int2> xlen(cd == 2 ? nedge : 0);
  auto recs = host_array<uint8_t>((size_t)npe * rb); // zeroed by the parallel first touch
  struct RecChunk {
    int64_t eb = 0, ee = 0;
    bool ok = true;
    std::vector<int32_t> tpos, tlen, cnt;
  };
  std::vector<RecChunk> rch(plan_threads());
  const int nrch = parallel_chunks(nedge, 1, [&](int t, int64_t eb, int64_t ee) {
    RecChunk& C = rch[t];
    C.eb = eb;
    C.ee = ee;
    C.cnt.assign(ee - eb, 0);
    std::vector<std::pair<int, int>> vc; // (vertex node, cell carrying it)
    for (int64_t e = eb; e < ee; ++e) {
      const int r = E0 + (int)e, A = eA[e], B = eB[e];
      vc.clear();
      for (int p = hp[r]; p < hp[r + 1]; ++p) {
        const int c = hpairs[p] / nrn;
        for (int v = 0; v < nv; ++v) vc.emplace_back(hrows[(size_t)c * nrn + v], c);
      }
      std::sort(vc.begin(), vc.end());
      int last = -1;
      for (auto& x : vc) {
        if (x.first == last) continue;
        last = x.first;
        const int c = x.second;
        const int k = [&] {
          for (int p = hp[r]; p < hp[r + 1]; ++p)
            if (hpairs[p] / nrn == c) return hpairs[p] % nrn;
          return -1;
        }();
        const int64_t pw = find_pair(x.first, c);
        if (pw < 0 || k < 0) {
          C.ok = false;
          return;
        }
        C.tpos.push_back(vpos(x.first, hrank[(size_t)pw * nrn + k]));
        if (cd == 2) C.tlen.push_back(vlen(x.first));
        ++C.cnt[e - eb];
      }
      {
        const int p = hp[r], c = hpairs[p] / nrn, k = hpairs[p] % nrn - nv;
        const int la = E[k][0], lb = E[k][1];
        const int lA = hrows[(size_t)c * nrn + la] == A ? la : lb, lB = lA == la ? lb : la;
        const int64_t pA = find_pair(A, c), pB = find_pair(B, c);
        if (pA < 0 || pB < 0) {
          C.ok = false;
          return;
        }
        xpos[e] = make_int4(vpos(A, hrank[(size_t)pA * nrn + lB]), vpos(B, hrank[(size_t)pB * nrn + lA]), dpos[A],
                            dpos[B]);
        if (cd == 2) xlen[e] = make_int2(vlen(A), vlen(B));
      }
      for (int p = hp[r]; p < hp[r + 1]; ++p) {
        const int c = hpairs[p] / nrn, k = hpairs[p] % nrn - nv;
        const int swap = hrows[(size_t)c * nrn + E[k][0]] != A ? 1 : 0;
        int sig[4];
        sigma_of(k, swap, sig);
        const int fA = assigned(sig[ca]) == k, fB = assigned(sig[cb]) == k;
        uint8_t* rec = &recs[(size_t)(p - p0e) * rb];
        const uint16_t h = (uint16_t)(((k * 2 + swap) << 10) | (fA << 14) | (fB << 15));
        memcpy(rec, &h, 2);
        const uint8_t* rk = &hrank[(size_t)p * nrn];
        for (int m = 0; m < nv; ++m) rec[2 + m] = rk[sig[m]];
        for (int f = 0; f < ne; ++f) rec[2 + nv + f] = rk[nv + edge_index(gd, sig[E[f][0]], sig[E[f][1]])];
        cellof[p - p0e] = c;
      }
    }
  });
  for (int t = 0; t < nrch; ++t) {
    const RecChunk& C = rch[t];
    if (!C.ok) return false;
    for (int64_t e = C.eb; e < C.ee; ++e) tptr[e + 1] = tptr[e] + C.cnt[e - C.eb];
    tpos.insert(tpos.end(), C.tpos.begin(), C.tpos.end());
    tlen.insert(tlen.end(), C.tlen.begin(), C.tlen.end());
  }
  rch.clear();
  // deterministic diagonals: per diagonal (vertex order of `diag`), the slots
  // 2 e + endpoint of the edge rows that carry a contribution, edge-ascending
  std::vector<int32_t> dptr, dslots;
  if (sp.det) {
    std::vector<int32_t> didx(E0, -1);
    int nd = 0;
    for (int v = 0; v < E0; ++v)
      if (hp[v + 1] > hp[v]) didx[v] = nd++;
    std::vector<int32_t> cnt(nd + 1, 0);
    std::vector<uint8_t> has(2 * (size_t)nedge, 0);
    for (int e = 0; e < nedge; ++e)
      for (int p = hp[E0 + e]; p < hp[E0 + e + 1]; ++p) {
        uint16_t h;
        memcpy(&h, &recs[(size_t)(p - p0e) * rb], 2);
        has[2 * (size_t)e] |= (h >> 14) & 1;
        has[2 * (size_t)e + 1] |= (h >> 15) & 1;
      }
    for (int e = 0; e < nedge; ++e) {
      if (has[2 * (size_t)e]) ++cnt[didx[eA[e]] + 1];
      if (has[2 * (size_t)e + 1]) ++cnt[didx[eB[e]] + 1];
    }
    for (int d = 0; d < nd; ++d) cnt[d + 1] += cnt[d];
    dptr = cnt;
    dslots.resize(cnt[nd]);
    for (int e = 0; e < nedge; ++e) {
      if (has[2 * (size_t)e]) dslots[cnt[didx[eA[e]]]++] = 2 * e;
      if (has[2 * (size_t)e + 1]) dslots[cnt[didx[eB[e]]]++] = 2 * e + 1;
    }
  }
  plan_tick("etile: per-row records", s);
  // ---- compact records: with every edge row at most 32 entries long, a rank
  // fits in 5 bits; the ranks of the row's own edge and of its two endpoint
  // vertices (canonical columns ca, cb, nv) are the same for every pair of the
  // row and move to a per-row word; the others pack with the header into 8
  // bytes (tets) / 4 bytes (triangles)
  bool compact = !std::getenv("LOAM_GPU_ET_WIDE");
  for (int e = 0; e < nedge && compact; ++e) compact = hrp[E0 + e + 1] - hrp[E0 + e] <= 32;
  std::vector<int> ncj; // canonical columns whose rank varies per pair
  for (int j = 0; j < nrn; ++j)
    if (j != ca && j != cb && j != nv) ncj.push_back(j);
  std::vector<uint32_t> rconst(nedge, 0);
  for (int e = 0; e < nedge && compact; ++e)
    for (int p = hp[E0 + e]; p < hp[E0 + e + 1]; ++p) {
      const uint8_t* rec = &recs[(size_t)(p - p0e) * rb];
      const uint32_t rcv = (uint32_t)rec[2 + ca] | (uint32_t)rec[2 + cb] << 8 | (uint32_t)rec[2 + nv] << 16;
      if (p == hp[E0 + e]) rconst[e] = rcv;
      else if (rcv != rconst[e]) compact = false;
    }
  const int rbx = compact ? (gd == 3 ? 8 : 4) : rb; // record bytes in the blob
  auto pack = [&](const uint8_t* rec, uint8_t* dst) { // full record -> blob record
    if (!compact) {
      memcpy(dst, rec, rb);
      return;
    }
    uint64_t w = (uint64_t)rec[0] | (uint64_t)rec[1] << 8;
    for (size_t q = 0; q < ncj.size(); ++q) w |= (uint64_t)(rec[2 + ncj[q]] & 31) << (q < 3 ? 16 + 5 * q : 32 + 5 * (q - 3));
    memcpy(dst, &w, rbx);
  };
  // ---- edge tiles: consecutive edge rows, their distinct cells and coordinate window.
  // Per warp of rows the segment is lane-interleaved (entry j of lane r at
  // base + 32 j + r: conflict-free shared updates) and so are the pair
  // records (word q of pair p of lane r at base + 32 (p RBW + q) + r).  Lanes
  // take the tile's rows in order of their pair count, so a warp's rows have
  // equal loop lengths and record padding.  Chunks of whole tile-row blocks
  // are tiled on all host cores and concatenated (blob / run offsets shifted).
  const int trows = sp.tile_rows <= 64 ? 64 : 128, nwarps = trows / 32, rbw = rbx / 4;
  const int cell_cap = std::min(sp.tile_cells, 1023);
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs;
    std::vector<uint8_t> blob;
    int max_segT = 0, max_rows = 0, max_seg = 0, max_cells = 0, max_slots = 0, max_blob = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nedge, trows, [&](int t, int64_t cb0, int64_t cb1) {
  TileChunk& O = tch[t];
  std::vector<int32_t>& tiles = O.tiles;
  std::vector<int32_t>& runs = O.runs;
  std::vector<uint8_t>& blob = O.blob;
  std::vector<int> vid; // (no per-thread ncells-sized arrays: cell sets are sorted vectors)
  // generation stamps over all cells / vertices (calloc'd: only touched pages map)
  struct Stamps {
    int* p;
    explicit Stamps(size_t n) : p(static_cast<int*>(std::calloc(n + 1, sizeof(int)))) {
      if (!p) throw std::bad_alloc();
    }
    ~Stamps() { std::free(p); }
  } cstamp(ncells), vstamp(nverts), clocal(ncells);
  int gen = 0;
  std::vector<std::pair<int, int>> rr;
  int r0 = (int)cb0;
  const int rend = (int)cb1;
  std::vector<int> lrow; // lane -> tile row
  auto warp_sizes = [&](int a, int b, std::vector<int>& lmax, std::vector<int>& pmax) {
    lmax.assign(nwarps, 0);
    pmax.assign(nwarps, 0);
    lrow.resize(b - a);
    for (int r = a; r < b; ++r) lrow[r - a] = r - a;
    std::stable_sort(lrow.begin(), lrow.end(), [&](int x, int y) {
      return hp[E0 + a + x + 1] - hp[E0 + a + x] < hp[E0 + a + y + 1] - hp[E0 + a + y];
    });
    for (int l = 0; l < b - a; ++l) {
      const int w = l / 32, r = a + lrow[l];
      lmax[w] = std::max<int>(lmax[w], (int)(hrp[E0 + r + 1] - hrp[E0 + r]));
      pmax[w] = std::max(pmax[w], hp[E0 + r + 1] - hp[E0 + r]);
    }
    int st = 0;
    for (int w = 0; w < nwarps; ++w) st += 32 * lmax[w];
    return st;
  };
  std::vector<int> lmax, pmax;
  while (r0 < rend) {
    int r1 = std::min(rend, r0 + trows);
    std::vector<int> cells;
    int slots = 0;
    auto fits = [&](int a, int b) {
      if (hrp[E0 + b] - hrp[E0 + a] > sp.tile_seg) return false;
      if (warp_sizes(a, b, lmax, pmax) > sp.tile_seg) return false;
      if (hp[E0 + b] - hp[E0 + a] > sp.tile_pairs) return false;
      for (int r = a; r < b; ++r)
        if (hp[E0 + r + 1] - hp[E0 + r] > 255) return false;
      ++gen;
      cells.clear();
      vid.clear();
      for (int p = hp[E0 + a]; p < hp[E0 + b]; ++p) { // distinct cells (pair order) and their distinct vertices
        const int c = cellof[p - p0e];
        if (cstamp.p[c] == gen) continue;
        cstamp.p[c] = gen;
        clocal.p[c] = (int)cells.size();
        cells.push_back(c);
        for (int v = 0; v < nv; ++v) {
          const int x = hx[(size_t)c * nv + v];
          if (vstamp.p[x] != gen) {
            vstamp.p[x] = gen;
            vid.push_back(x);
          }
        }
      }
      if ((int)cells.size() > cell_cap) return false;
      slots = make_runs(vid, nverts, rr);
      return slots <= sp.tile_slots && (int)rr.size() <= sp.tile_runs;
    };
    while (!fits(r0, r1)) {
      if (r1 == r0 + 1) {
        O.ok = false;
        return;
      }
      r1 = r0 + (r1 - r0) / 2;
    }
    const int segT = warp_sizes(r0, r1, lmax, pmax);
    // cells in id order (the locality order: neighbouring cells share Gram /
    // gradient rows in shared memory), local ids renumbered to match
    std::sort(cells.begin(), cells.end());
    for (size_t q = 0; q < cells.size(); ++q) clocal.p[cells[q]] = (int)q;
    auto local_of = [&](int c) { return clocal.p[c]; };
    std::vector<int> base(rr.size());
    for (size_t q = 0, acc = 0; q < rr.size(); ++q) {
      base[q] = (int)acc;
      acc += rr[q].second - rr[q].first;
    }
    auto slot_in = [&](int v) {
      size_t q = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
      return base[q] + v - rr[q].first;
    };
    const int nrows = r1 - r0, ncell = (int)cells.size();
    const int T0 = tptr[r0], ntp = tptr[r1] - T0;
    int rwords = 0;
    for (int w = 0; w < nwarps; ++w) rwords += pmax[w] * rbw * 32;
    const int off_srow = 0, off_trow = up16((nrows + 1) * 2), off_np = off_trow + up16((nrows + 1) * 2),
              off_xpos = off_np + up16(6 * trows + 4 * nwarps), off_tpos = off_xpos + nrows * 16,
              off_tlen = off_tpos + up16(ntp * 4), off_xlen = off_tlen + (cd == 2 ? up16(ntp * 4) : 0),
              off_recs = off_xlen + (cd == 2 ? up16(nrows * 8) : 0), off_cells = off_recs + up16(rwords * 4),
              bytes = off_cells + up16(ncell * nv * 2);
    const size_t b0 = blob.size();
    blob.resize(b0 + bytes, 0);
    uint8_t* bp = blob.data() + b0;
    for (int r = 0; r <= nrows; ++r) {
      const uint16_t sr = (uint16_t)(hrp[E0 + r0 + r] - hrp[E0 + r0]);
      const uint16_t tr = (uint16_t)(tptr[r0 + r] - T0);
      memcpy(bp + off_srow + 2 * r, &sr, 2);
      memcpy(bp + off_trow + 2 * r, &tr, 2);
    }
    for (int r = 0; r < nrows; ++r) bp[off_np + r] = (uint8_t)(hp[E0 + r0 + r + 1] - hp[E0 + r0 + r]);
    for (int l = 0; l < nrows; ++l) bp[off_np + trows + 4 * nwarps + l] = (uint8_t)lrow[l];
    if (compact) memcpy(bp + off_np + 2 * trows + 4 * nwarps, &rconst[r0], (size_t)nrows * 4);
    {
      int sb = 0, wb = 0;
      for (int w = 0; w < nwarps; ++w) {
        const uint16_t s16 = (uint16_t)sb, w16 = (uint16_t)wb;
        memcpy(bp + off_np + trows + 4 * w, &s16, 2);
        memcpy(bp + off_np + trows + 4 * w + 2, &w16, 2);
        for (int l = 0; l < 32 && 32 * w + l < nrows; ++l) {
          const int r = r0 + lrow[32 * w + l];
          for (int p = hp[E0 + r]; p < hp[E0 + r + 1]; ++p) {
            const int64_t pe = p - p0e;
            uint8_t full_rec[16], rec[16];
            memcpy(full_rec, &recs[(size_t)pe * rb], rb);
            uint16_t h;
            memcpy(&h, full_rec, 2);
            h = (uint16_t)(h | local_of(cellof[pe]));
            memcpy(full_rec, &h, 2);
            pack(full_rec, rec);
            const int pi = p - hp[E0 + r];
            for (int q = 0; q < rbw; ++q)
              memcpy(bp + off_recs + 4 * ((size_t)wb + (pi * rbw + q) * 32 + l), rec + 4 * q, 4);
          }
        }
        sb += 32 * lmax[w];
        wb += pmax[w] * rbw * 32;
      }
    }
    memcpy(bp + off_xpos, &xpos[r0], (size_t)nrows * 16);
    if (ntp) memcpy(bp + off_tpos, &tpos[T0], (size_t)ntp * 4);
    if (cd == 2) {
      if (ntp) memcpy(bp + off_tlen, &tlen[T0], (size_t)ntp * 4);
      memcpy(bp + off_xlen, &xlen[r0], (size_t)nrows * 8);
    }
    for (int q = 0; q < ncell; ++q)
      for (int v = 0; v < nv; ++v) {
        const uint16_t sl = (uint16_t)slot_in(hx[(size_t)cells[q] * nv + v]);
        memcpy(bp + off_cells + 2 * (q * nv + v), &sl, 2);
      }
    const int seg = (int)(hrp[E0 + r1] - hrp[E0 + r0]);
    tiles.insert(tiles.end(), {(int)(b0 / 16), bytes, r0, nrows, (int)(cd * cd * hrp[E0 + r0]), seg, segT, ncell,
                               (int)runs.size() / 2, (int)rr.size(), off_srow, off_np, off_recs, off_cells, off_trow,
                               off_xpos});
    O.max_segT = std::max(O.max_segT, segT);
    for (auto& x : rr) runs.insert(runs.end(), {x.first, x.second});
    O.max_rows = std::max(O.max_rows, nrows);
    O.max_seg = std::max(O.max_seg, seg);
    O.max_cells = std::max(O.max_cells, ncell);
    O.max_slots = std::max(O.max_slots, slots);
    O.max_blob = std::max(O.max_blob, bytes);
    r0 = r1;
  }
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
    out.max_segT = std::max(out.max_segT, O.max_segT);
    out.max_rows = std::max(out.max_rows, O.max_rows);
    out.max_seg = std::max(out.max_seg, O.max_seg);
    out.max_cells = std::max(out.max_cells, O.max_cells);
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_blob = std::max(out.max_blob, O.max_blob);
  }
  upload_parts(out.blob, parts, s); // the chunks' blobs, uploaded in place (no host concatenation)
  tch.clear();
  plan_tick("etile: tiles", s);
  out.gd = gd;
  out.cd = cd;
  out.tile_threads = trows;
  out.compact = compact;
  out.ntiles = (int)tiles.size() / 16;
  out.e0 = E0;
  out.nedge = nedge;
  out.rec_bytes = rb;
  out.ndiag = (int64_t)diag.size() / cd;
  memcpy(out.ktab, ktab, sizeof(ktab));
  auto upload = [&](auto& dst, const auto& src) {
    using T = typename std::decay_t<decltype(src)>::value_type;
    dst.alloc(src.size() + 16, s);
    if (!src.empty())
      LG_CUDA(cudaMemcpyAsync(dst.get(), src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
  };
  upload(out.tiles, tiles);
  upload(out.runs, runs);
  upload(out.diag, diag);
  out.det = sp.det;
  if (sp.det) {
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

struct EtileArgs {
  const int32_t* tiles;
  int ntiles;
  int* next_tile;
  int* reset_tile;
  const uint8_t* blob;
  const int32_t* runs;
  const double* coords;
  double* out;
  FormParams prm;
  int accumulate, dynamic, dbg;
  int off_seg, off_geo, off_buf, buf_bytes, b_win;
  uint32_t ktab[12];
  double* dsum; // deterministic mode: diagonal partial sums by (edge row, endpoint)
};

template <int D>
struct EtT {
  static constexpr int NV = D + 1, NE = D == 2 ? 3 : 6, N = NV + NE;
  // per cell in shared memory: the Gram matrix G_xy = V g_x.g_y as NV rows of
  // 4 doubles (two 16-byte loads per row), then V; stride odd in 16-byte units
  static constexpr int GV = 4 * NV, GS = D == 2 ? 14 : 18;
  static constexpr int RB = (2 + N + 3) & ~3, RBW = RB / 4;
  static constexpr int CA = NV - 2, CB = NV - 1;   // canonical row edge = local edge 0
};

// Canonical P2 edge row (row node = local edge 0 = (CA, CB)) from the Gram
// entries G_xy = V g_x.g_y: same integrals as p2_rows (elements.cuh), with the
// cell measure folded into G.  Also returns the (CA, CB) vertex-vertex entry
// and the two vertex diagonals of this cell.
template <int FORM, int D>
__device__ __forceinline__ void et_row(const double (&Ga)[D + 1], const double (&Gb)[D + 1], double V,
                                       const FormParams& prm, double (&o)[EtT<D>::N], double& vab, double& dga,
                                       double& dgb) {
  using T = EtT<D>;
  using S = Simplex<D>;
  constexpr int NV = T::NV, NE = T::NE, a = T::CA, b = T::CB;
  constexpr double qs = S::q_same, qd = S::q_diff, l1 = S::l1;
  constexpr double cs = 16.0 * qs - 8.0 * l1 + 1.0, co = 16.0 * qd - 8.0 * l1 + 1.0;
  constexpr double es = 4.0 * qs - l1, ed = 4.0 * qd - l1;
  const double kV = prm.p[0] * V;
  auto comb = [&](double K, double M) {
    if constexpr (FORM == F_MASS) return V * M;
    else if constexpr (FORM == F_STIFFNESS) return K;
    else if constexpr (FORM == F_STOKES_A) return prm.p[0] * K; // nu grad u : grad v, per component
    else return fma(kV, M, K);
  };
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double K = 4.0 * ((j == b ? es : ed) * Ga[j] + (j == a ? es : ed) * Gb[j]);
    o[j] = comb(K, (j == a || j == b) ? p2_mass_const<D>(2) : p2_mass_const<D>(3));
  }
#pragma unroll
  for (int f = 0; f < NE; ++f) {
    const int c = S::edge_a(f), d = S::edge_b(f);
    const double K = 16.0 * ((b == d ? qs : qd) * Ga[c] + (b == c ? qs : qd) * Ga[d] + (a == d ? qs : qd) * Gb[c] +
                             (a == c ? qs : qd) * Gb[d]);
    const int shared = (a == c) + (a == d) + (b == c) + (b == d);
    const double M = f == 0 ? p2_mass_const<D>(4) : (shared == 1 ? p2_mass_const<D>(5) : p2_mass_const<D>(6));
    o[NV + f] = comb(K, M);
  }
  vab += comb(co * Ga[b], p2_mass_const<D>(1));
  dga = comb(cs * Ga[a], p2_mass_const<D>(0));
  dgb = comb(cs * Gb[b], p2_mass_const<D>(0));
}

// mbarrier wait that lets the warp sleep (up to the hint, ns) instead of
// spinning on try_wait: waiting consumers leave their issue slots to the
// other CTAs of the SM
__device__ __forceinline__ void et_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000)
      : "memory");
}

// v[i] for a runtime i in 0..3 without local memory or branches (selp.f64)
__device__ __forceinline__ double sel4(const double (&v)[4], int i) {
  double r;
  asm("{\n"
      ".reg .pred p0, p1;\n"
      ".reg .f64 lo, hi;\n"
      ".reg .b32 t;\n"
      "and.b32 t, %5, 1;\n"
      "setp.ne.s32 p0, t, 0;\n"
      "and.b32 t, %5, 2;\n"
      "setp.ne.s32 p1, t, 0;\n"
      "selp.f64 lo, %2, %1, p0;\n"
      "selp.f64 hi, %4, %3, p0;\n"
      "selp.f64 %0, hi, lo, p1;\n"
      "}\n"
      : "=d"(r)
      : "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "r"(i));
  return r;
}

// NT consumer threads (= edge rows per tile) + one TMA producer warp.
template <int FORM, int D, int CD, int NT, int STAGES, bool COMPACT>
__global__ void __launch_bounds__(NT + 32, 1) k_etile(const __grid_constant__ EtileArgs a) {
  using T = EtT<D>;
  constexpr int NV = T::NV, N = T::N;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  int* slot_tile = reinterpret_cast<int*>(sm + 48);
  uint32_t* ktab = reinterpret_cast<uint32_t*>(sm + 64);
  const int tid = threadIdx.x;
  if (tid < 12) ktab[tid] = a.ktab[tid];
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
  auto meta = [&](int tile, int (&m)[16]) {
    const int4* t = reinterpret_cast<const int4*>(a.tiles + 16 * tile);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 x = __ldg(t + q);
      m[4 * q] = x.x;
      m[4 * q + 1] = x.y;
      m[4 * q + 2] = x.z;
      m[4 * q + 3] = x.w;
    }
  };
  if (tid >= NT) { // ---- producer warp: tile blob + coordinate window by TMA
    const int lane = tid & 31;
    // static round-robin schedule (tiles are near-uniform); the dynamic
    // counter (a.dynamic) costs a dependent global atomic per tile
    int sched = 0;
    auto grab = [&]() {
      if (!a.dynamic) return (int)blockIdx.x + (sched++) * (int)gridDim.x;
      int t = 0;
      if (lane == 0) t = atomicAdd(a.next_tile, 1);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    int nt = grab();
    int nm[16];
    int2 nrun = make_int2(0, 0);
    auto prefetch = [&]() {
      if (nt < a.ntiles) {
        meta(nt, nm);
        nrun = first_run(reinterpret_cast<const int2*>(a.runs) + nm[8], nm[9], lane);
      }
    };
    prefetch();
    grid_dep_wait(); // the caller's data only after the previous kernel (PDL)
    for (int k = 0;; ++k) {
      const int tile = nt;
      int m[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) m[q] = nm[q];
      const int2 run0 = nrun;
      if (k >= STAGES) mbar_wait_sleep(&empty[k % STAGES], (k / STAGES - 1) & 1);
      if (tile >= a.ntiles) {
        if (lane == 0) {
          slot_tile[k % STAGES] = -1;
          mbar_arrive(&full[k % STAGES]);
        }
        break;
      }
      if (lane == 0) slot_tile[k % STAGES] = tile;
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % STAGES];
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + m[8], m[9], a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), D};
      const uint32_t tx = (uint32_t)m[1] + stage_runs<false>(rc, lane, bar, run0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, tx);
        bulk_g2s(buf, a.blob + (int64_t)m[0] * 16, (uint32_t)m[1], bar);
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
  constexpr int GS = T::GS, RBW = COMPACT ? (D == 3 ? 2 : 1) : T::RBW;
  double* segT = reinterpret_cast<double*>(sm + a.off_seg); // lane-interleaved row segments
  double* geo = reinterpret_cast<double*>(sm + a.off_geo);  // cell Gram matrices; then the contiguous segment
  const int lane = tid & 31, warp = tid >> 5;
  for (int k = 0;; ++k) {
    et_wait(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    int m[16];
    meta(tile, m);
    const int nrows = m[3], E0 = m[4], len = CD * CD * m[5], lenT = m[6], ncell = m[7];
    const unsigned char* buf = ring(k);
    const uint16_t* srow = reinterpret_cast<const uint16_t*>(buf + m[10]);
    const uint8_t* npair = buf + m[11];
    const uint16_t* wmeta = reinterpret_cast<const uint16_t*>(buf + m[11] + NT);
    const uint8_t* lrow = buf + m[11] + NT + 4 * (NT / 32);                        // lane -> row
    const uint32_t* rconst = reinterpret_cast<const uint32_t*>(buf + m[11] + 2 * NT + 4 * (NT / 32));
    const uint32_t* recs = reinterpret_cast<const uint32_t*>(buf + m[12]);
    const uint16_t* cslot = reinterpret_cast<const uint16_t*>(buf + m[13]);
    const uint16_t* trow = reinterpret_cast<const uint16_t*>(buf + m[14]);
    const int4* xpos = reinterpret_cast<const int4*>(buf + m[15]);
    const int32_t* tpos = reinterpret_cast<const int32_t*>(buf + m[15] + 16 * nrows);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    // the previous tile's bulk store reads the contiguous segment (in geo)
    if (tid == 0) bulk_wait_read<0>();
    named_bar(1, NT);
    // phase 1: the Gram matrix of every cell of the tile, once
    for (int c = tid; c < ((a.dbg & 2) ? 0 : ncell); c += NT) {
      double X[NV][D];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int sl = cslot[c * NV + v];
#pragma unroll
        for (int q = 0; q < D; ++q) X[v][q] = win[sl * D + q];
      }
      Geom<D> Gm;
      geometry<D>(X, Gm);
      double* g = geo + c * GS;
      if constexpr (FORM != F_MASS) {
        double vg[NV][D];
#pragma unroll
        for (int p = 0; p < NV; ++p)
#pragma unroll
          for (int q = 0; q < D; ++q) vg[p][q] = Gm.V * Gm.g[p][q];
        double Gr[NV][4];
#pragma unroll
        for (int p = 0; p < NV; ++p)
#pragma unroll
          for (int q = p; q < NV; ++q) {
            Gr[p][q] = dot<D>(vg[p], Gm.g[q]);
            Gr[q][p] = Gr[p][q];
          }
#pragma unroll
        for (int p = 0; p < NV; ++p) {
          if constexpr (NV < 4) Gr[p][3] = 0.0;
          reinterpret_cast<double2*>(g + 4 * p)[0] = make_double2(Gr[p][0], Gr[p][1]);
          reinterpret_cast<double2*>(g + 4 * p)[1] = make_double2(Gr[p][2], Gr[p][3]);
        }
      }
      g[T::GV] = Gm.V;
    }
    {
      double2* z = reinterpret_cast<double2*>(segT);
      for (int t = tid; t < (lenT >> 1); t += NT) z[t] = make_double2(0.0, 0.0); // this loop's contributions only
    }
    named_bar(1, NT);
    // phase 2: one thread per edge row
    int s0 = 0, L = 0;
    const int sb = wmeta[2 * warp], rbase = wmeta[2 * warp + 1];
    double* my = segT + sb + lane; // entry j of this row at my[32 j]
    const int row = tid < nrows ? lrow[tid] : 0;
    if (tid < nrows) {
      s0 = srow[row];
      L = srow[row + 1] - s0;
      const int np = (a.dbg & 1) ? 0 : npair[row];
      int pconst[3] = {0, 0, 0}; // compact: ranks of canonical columns CA, CB, NV (the row's own)
      double creg[3] = {0.0, 0.0, 0.0};
      if constexpr (COMPACT) {
        const uint32_t rc = rconst[row];
        pconst[0] = 32 * (int)(rc & 0xffu);
        pconst[1] = 32 * (int)((rc >> 8) & 0xffu);
        pconst[2] = 32 * (int)((rc >> 16) & 0xffu);
      }
      double vab = 0.0, dA = 0.0, dB = 0.0;
      bool hA = false, hB = false;
      const uint32_t* rq = recs + rbase + lane;
      for (int p = 0; p < np; ++p) {
        uint32_t w[RBW];
#pragma unroll
        for (int q = 0; q < RBW; ++q) w[q] = rq[(p * RBW + q) * 32];
        const uint32_t h = w[0] & 0xffffu;
        const uint32_t sg = ktab[(h >> 10) & 15u];
        const double* g = geo + (h & 1023u) * GS;
        const int la = (sg >> (4 * T::CA)) & 15, lb = (sg >> (4 * T::CB)) & 15;
        double GA[4], GB[4];
        {
          const double2* ra = reinterpret_cast<const double2*>(g + 4 * la);
          const double2* rb2 = reinterpret_cast<const double2*>(g + 4 * lb);
          const double2 a0 = ra[0], a1 = ra[1], b0 = rb2[0], b1 = rb2[1];
          GA[0] = a0.x; GA[1] = a0.y; GA[2] = a1.x; GA[3] = a1.y;
          GB[0] = b0.x; GB[1] = b0.y; GB[2] = b1.x; GB[3] = b1.y;
        }
        const double V = g[T::GV];
        // canonical order: canonical vertex mm is original local vertex sigma(mm)
        double Ga[NV], Gb[NV];
#pragma unroll
        for (int mm = 0; mm < NV; ++mm) {
          const int sv = (sg >> (4 * mm)) & 15;
          Ga[mm] = sel4(GA, sv);
          Gb[mm] = sel4(GB, sv);
        }
        double o[N], dga, dgb;
        et_row<FORM, D>(Ga, Gb, V, a.prm, o, vab, dga, dgb);
        int pos[N];
        if constexpr (COMPACT) {
          int q = 0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            if (j == T::CA) pos[j] = pconst[0];
            else if (j == T::CB) pos[j] = pconst[1];
            else if (j == NV) pos[j] = pconst[2];
            else {
              const int bit = q < 3 ? 16 + 5 * q : 5 * (q - 3);
              pos[j] = 32 * (int)((w[q < 3 ? 0 : 1] >> bit) & 31u);
              ++q;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) pos[j] = 32 * (int)((w[(2 + j) >> 2] >> (8 * ((2 + j) & 3))) & 0xffu);
        }
        if constexpr (COMPACT) {
          // the row's own edge and its two endpoint vertices: same entry for
          // every pair of the row -> register sums (same order), stored once
          // after the loop; the other columns by read-modify-write
          creg[0] += o[T::CA];
          creg[1] += o[T::CB];
          creg[2] += o[NV];
          double cur[N];
#pragma unroll
          for (int j = 0; j < N; ++j)
            if (j != T::CA && j != T::CB && j != NV) cur[j] = my[pos[j]];
#pragma unroll
          for (int j = 0; j < N; ++j)
            if (j != T::CA && j != T::CB && j != NV) my[pos[j]] = cur[j] + o[j];
        } else {
          double cur[N];
#pragma unroll
          for (int j = 0; j < N; ++j) cur[j] = my[pos[j]];
#pragma unroll
          for (int j = 0; j < N; ++j) my[pos[j]] = cur[j] + o[j];
        }
        if (h & 0x4000u) {
          dA += dga;
          hA = true;
        }
        if (h & 0x8000u) {
          dB += dgb;
          hB = true;
        }
      }
      if constexpr (COMPACT) {
        if (np > 0) {
          my[pconst[0]] = creg[0];
          my[pconst[1]] = creg[1];
          my[pconst[2]] = creg[2];
        }
      }
      // vertex rows: transposed vertex-column entries, the vertex pair, diagonals
      const int t0 = trow[row], t1 = (a.dbg & 4) ? t0 : trow[row + 1];
      const int ntp = trow[nrows];
      // CD = 2: the 2x2 block (v, v) / (v, w) is (x, 0; 0, x) at rows pos, pos + rowlen
      const int32_t* tlen = tpos + ((ntp + 3) & ~3);
      const int2* xlen = reinterpret_cast<const int2*>(tlen + ((ntp + 3) & ~3));
      auto put = [&](int pos, int rl, double v) {
        if constexpr (CD == 1) {
          a.out[pos] = a.accumulate ? a.out[pos] + v : v;
        } else {
          double2* r0 = reinterpret_cast<double2*>(a.out + pos);
          double2* r1 = reinterpret_cast<double2*>(a.out + pos + rl);
          if (a.accumulate) {
            double2 x0 = *r0, x1 = *r1;
            x0.x += v;
            x1.y += v;
            *r0 = x0;
            *r1 = x1;
          } else {
            *r0 = make_double2(v, 0.0);
            *r1 = make_double2(0.0, v);
          }
        }
      };
      for (int t = t0; t < t1; ++t) put(tpos[t], CD == 2 ? tlen[t] : 0, my[32 * (t - t0)]);
      const int4 xp = xpos[row];
      const int2 xl = CD == 2 ? xlen[row] : make_int2(0, 0);
      put(xp.x, xl.x, vab);
      put(xp.y, xl.y, vab);
      if (a.dsum) { // deterministic: partial sums in slots, summed in a fixed order (k_et_dsum)
        const int64_t e = (int64_t)m[2] + row;
        if (hA) a.dsum[2 * e] = dA;
        if (hB) a.dsum[2 * e + 1] = dB;
      } else {
        if (hA) {
          atomicAdd(a.out + xp.z, dA);
          if constexpr (CD == 2) atomicAdd(a.out + xp.z + xl.x + 1, dA);
        }
        if (hB) {
          atomicAdd(a.out + xp.w, dB);
          if constexpr (CD == 2) atomicAdd(a.out + xp.w + xl.y + 1, dB);
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]);
    named_bar(1, NT); // every Gram read done: geo becomes the contiguous segment
    double* seg = geo + (E0 & 1); // shares the 16-byte parity of its global destination
    if constexpr (CD == 1) {
      for (int j = 0; j < L; ++j) seg[s0 + j] = my[32 * j];
    } else { // node row -> dof rows 2r (x, 0, ...) and 2r+1 (0, x, ...); E0 is a multiple of 4
      double2* r0 = reinterpret_cast<double2*>(seg + 4 * s0);
      for (int j = 0; j < L; ++j) {
        const double v = my[32 * j];
        r0[j] = make_double2(v, 0.0);
        r0[L + j] = make_double2(0.0, v);
      }
    }
    if (a.accumulate) {
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] += seg[t];
    } else {
      // segment complete -> one TMA bulk store (doubles off the 16-byte grid stored directly)
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

__global__ void k_et_zero(const int32_t* __restrict__ pos, int64_t n, int cd, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (cd == 1) {
    out[pos[i]] = 0.0;
  } else { // the 2x2 diagonal block
    const int p = pos[2 * i], rl = pos[2 * i + 1];
    *reinterpret_cast<double2*>(out + p) = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(out + p + rl) = make_double2(0.0, 0.0);
  }
}

// Deterministic diagonals: diagonal d = its slots summed in list order.
__global__ void k_et_dsum(const int32_t* __restrict__ pos, const int32_t* __restrict__ dptr,
                          const int32_t* __restrict__ dslots, int64_t n, int cd, const double* __restrict__ dsum,
                          double* __restrict__ out, int accumulate) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  double acc = 0.0;
  for (int q = dptr[d]; q < dptr[d + 1]; ++q) acc += dsum[dslots[q]];
  if (cd == 1) {
    out[pos[d]] = accumulate ? out[pos[d]] + acc : acc;
  } else { // the 2x2 diagonal block (x, 0; 0, x)
    const int p = pos[2 * d], rl = pos[2 * d + 1];
    if (accumulate) {
      out[p] += acc;
      out[p + rl + 1] += acc;
    } else {
      *reinterpret_cast<double2*>(out + p) = make_double2(acc, 0.0);
      *reinterpret_cast<double2*>(out + p + rl) = make_double2(0.0, acc);
    }
  }
}

template <int FORM, int D, int CD>
void go_etile(const EtilePlan& p, const EtileArgs& a, size_t smem_base, size_t buf, cudaStream_t s) {
  auto go = [&](auto kern, int threads, int stages) {
    const size_t smem = smem_base + stages * buf;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, threads, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "edge-tile kernel does not fit on an SM");
    const int grid = std::min(p.ntiles, blocks * kNumSMs);
    launch_pdl(kern, dim3(grid), dim3(threads), smem, s, a);
  };
  const int st = et_stages();
  auto pick = [&](auto compact) {
    constexpr bool C = decltype(compact)::value;
    if (p.tile_threads == 64) {
      if (st >= 2) go(k_etile<FORM, D, CD, 64, 2, C>, 96, 2);
      else go(k_etile<FORM, D, CD, 64, 1, C>, 96, 1);
    } else {
      if (st >= 2) go(k_etile<FORM, D, CD, 128, 2, C>, 160, 2);
      else go(k_etile<FORM, D, CD, 128, 1, C>, 160, 1);
    }
  };
  if (p.compact) pick(std::true_type{});
  else pick(std::false_type{});
}

} // namespace

int et_stages() {
  // two stages: the next tile's blob and window land while this one computes
  static const int st = std::getenv("LOAM_GPU_ET_STAGES") ? std::atoi(std::getenv("LOAM_GPU_ET_STAGES")) : 2;
  return st;
}

void launch_etile(int form, const EtilePlan& p, const double* coords, double* out, const FormParams& prm,
                  bool accumulate, int* next_tile, int* reset_tile, cudaStream_t s) {
  if (!accumulate && p.ndiag && !p.det) {
    k_et_zero<<<ceil_div(p.ndiag, 256), 256, 0, s>>>(p.diag.get(), p.ndiag, p.cd, out);
    count_launch();
    LG_LAUNCH_CHECK();
  }
  DevBuf<double> dsum;
  if (p.det) dsum.alloc(2 * (size_t)std::max(p.nedge, 1), s);
  auto finish = [&] { // deterministic mode: the diagonals in a fixed order
    if (!p.det || !p.ndiag) return;
    k_et_dsum<<<ceil_div(p.ndiag, 256), 256, 0, s>>>(p.diag.get(), p.dptr.get(), p.dslots.get(), p.ndiag, p.cd,
                                                     dsum.get(), out, accumulate ? 1 : 0);
    count_launch();
    LG_LAUNCH_CHECK();
  };
  if (p.ntiles == 0) {
    finish();
    return;
  }
  EtileArgs a{};
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
  a.dynamic = std::getenv("LOAM_GPU_ET_STATIC") ? 0 : 1;
  a.dbg = std::getenv("LOAM_GPU_ET_DBG") ? std::atoi(std::getenv("LOAM_GPU_ET_DBG")) : 0; // developer: skip phases
  memcpy(a.ktab, p.ktab, sizeof(a.ktab));
  a.dsum = p.det ? dsum.get() : nullptr;
  int off = 128;
  a.off_seg = off;
  off += up16(p.max_segT * 8);
  a.off_geo = off;
  off += up16(std::max(p.max_cells * (p.gd == 2 ? 14 : 18), p.cd * p.cd * p.max_seg + 2) * 8);
  a.off_buf = off;
  a.b_win = up16(p.max_blob);
  a.buf_bytes = a.b_win + up16(p.max_slots * p.gd * 8 + 16);
  const size_t base = (size_t)off, buf = (size_t)a.buf_bytes;
  if (std::getenv("LOAM_GPU_ET_INFO")) // developer: plan maxima behind the shared-memory footprint
    fprintf(stderr, "etile: tiles %d max_segT %d max_seg %d max_cells %d max_blob %d max_slots %d stage %d fixed %d\n",
            p.ntiles, p.max_segT, p.max_seg, p.max_cells, p.max_blob, p.max_slots, a.buf_bytes, off);
  if (p.cd == 2) {
    require(p.gd == 2 && form == F_STOKES_A, LOAM_ERR(InvalidArgument), "edge tiles: cd = 2 is the Stokes A block");
    go_etile<F_STOKES_A, 2, 2>(p, a, base, buf, s);
  } else if (p.gd == 3) {
    if (form == F_MASS) go_etile<F_MASS, 3, 1>(p, a, base, buf, s);
    else if (form == F_STIFFNESS) go_etile<F_STIFFNESS, 3, 1>(p, a, base, buf, s);
    else go_etile<F_HELMHOLTZ, 3, 1>(p, a, base, buf, s);
  } else {
    if (form == F_MASS) go_etile<F_MASS, 2, 1>(p, a, base, buf, s);
    else if (form == F_STIFFNESS) go_etile<F_STIFFNESS, 2, 1>(p, a, base, buf, s);
    else go_etile<F_HELMHOLTZ, 2, 1>(p, a, base, buf, s);
  }
  count_launch();
  LG_LAUNCH_CHECK();
  finish();
}

} // namespace loam_gpu
