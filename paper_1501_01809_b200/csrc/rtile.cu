#include <atomic>
// rtile.cu -- row tiles with shared cell geometry (see rtile.cuh).
//
// Reference path replaced: the three par_loops of assemble_blocks for the
// Taylor-Hood coupling blocks (fem/assemble.hpp:439-448 -> parloop.hpp:191-384,
// Mat::addto data.hpp:205-222), element kernels restated in elements.cuh
// (FormT<F_STOKES_B / F_STOKES_BT>).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "rtile.cuh"
#include "stage.cuh"

namespace loam_gpu {

namespace {

inline int up16(int x) { return (x + 15) & ~15; }

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

} // namespace

// B^T (velocity rows: 2.4 M short rows of 3-7 pressure columns) measured
// faster on the pair tiles (0.135 vs 0.158 ms on config 5); B (pressure rows,
// 6 cells x 12 values) on the row tiles (0.106 vs 0.119 ms).  LOAM_GPU_RTILE_BT
// selects the row tiles for B^T as well.
bool rtile_form(int form) {
  static const bool bt = std::getenv("LOAM_GPU_RTILE_BT") != nullptr;
  static const bool av = std::getenv("LOAM_GPU_RTILE_A") != nullptr;
  return form == F_STOKES_B || (bt && form == F_STOKES_BT) || (av && form == F_STOKES_A);
}

bool build_rtile(RtilePlan& out, const RtileSpec& sp, int form, int gd, int nrn, int ncn, int rd, int cd,
                 int ncells, int nrows_node, const int32_t* sorted_rows, const int32_t* sorted_x, int nverts,
                 const PairPlan& pp, const int64_t* row_ptr, int64_t nnz, cudaStream_t s) {
  const int nv = gd + 1;
  (void)sorted_rows;
  if (!rtile_form(form) || pp.nrn != nrn || pp.ncn != ncn || nnz >= (int64_t(1) << 31) || ncells == 0) return false;
  const int64_t np = pp.npairs;
  auto hx = host_array<int32_t>((size_t)ncells * nv), hpairs = host_array<int32_t>(np),
       hp = host_array<int32_t>(nrows_node + 1);
  auto hrank = host_array<uint8_t>((size_t)np * ncn);
  auto hrp = host_array<int64_t>((size_t)nrows_node * rd + 1);
  parallel_d2h({{hx.data(), sorted_x, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * (size_t)np},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * (size_t)(nrows_node + 1)},
                {hrank.data(), pp.ranks.get(), hrank.size()},
                {hrp.data(), row_ptr, sizeof(int64_t) * hrp.size()}},
               s);
  std::vector<int64_t> nptr(nrows_node + 1); // node-level pattern offsets of the rd x cd blocked CSR
  for (int i = 0; i <= nrows_node; ++i) nptr[i] = hrp[(size_t)rd * i] / (rd * cd);
  // ---- canonical pair records: u32 header (tile cell | canonical->original
  // vertex map, 2 bits each | edge-row flag), then the column ranks in
  // canonical order
  const int rb = (4 + ncn + 3) & ~3, rbw = rb / 4;
  auto recs = host_array<uint8_t>((size_t)np * rb); // zeroed by the parallel first touch
  std::atomic<bool> recs_ok{true};
  parallel_chunks(nrows_node, 1, [&](int, int64_t rb0, int64_t rb1) {
  for (int r = (int)rb0; r < (int)rb1; ++r)
    for (int p = hp[r]; p < hp[r + 1]; ++p) {
      const int i = hpairs[p] % nrn;
      int sigma[4], inv[4], colpos[10];
      const int ci = canonical_sigma(gd, nrn, i, sigma);
      for (int v = 0; v < nv; ++v) inv[sigma[v]] = v;
      induced(gd, ncn, sigma, colpos);
      uint32_t h = 0;
      for (int m = 0; m < nv; ++m) h |= (uint32_t)inv[m] << (10 + 2 * m);
      if (ci) h |= 1u << 18;
      uint8_t* rec = &recs[(size_t)p * rb];
      memcpy(rec, &h, 4);
      const int L = (int)(nptr[r + 1] - nptr[r]);
      for (int j = 0; j < ncn; ++j) {
        const int rk = hrank[(size_t)p * ncn + j];
        if (rk >= L) {
          recs_ok = false;
          return;
        }
        rec[4 + colpos[j]] = (uint8_t)rk;
      }
    }
  });
  if (!recs_ok) return false;
  // ---- tiles of consecutive row nodes
  const int trows = sp.tile_rows <= 64 ? 64 : 128, nwarps = trows / 32, W = rd * cd;
  // chunks of whole tile-row blocks tiled on all host cores, concatenated
  // (blob / run offsets shifted)
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs;
    std::vector<uint8_t> blob;
    int max_seg = 0, max_segT = 0, max_cells = 0, max_slots = 0, max_blob = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nrows_node, trows, [&](int t, int64_t cb0, int64_t cb1) {
  TileChunk& O = tch[t];
  std::vector<int32_t>& tiles = O.tiles;
  std::vector<int32_t>& runs = O.runs;
  std::vector<uint8_t>& blob = O.blob;
  std::vector<int> vid, lrow;
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
  std::vector<int> lmax, pmax;
  auto warp_sizes = [&](int a, int b) {
    lmax.assign(nwarps, 0);
    pmax.assign(nwarps, 0);
    lrow.resize(b - a);
    for (int r = a; r < b; ++r) lrow[r - a] = r - a;
    std::stable_sort(lrow.begin(), lrow.end(),
                     [&](int x, int y) { return hp[a + x + 1] - hp[a + x] < hp[a + y + 1] - hp[a + y]; });
    for (int l = 0; l < b - a; ++l) {
      const int w = l / 32, r = a + lrow[l];
      lmax[w] = std::max<int>(lmax[w], (int)(nptr[r + 1] - nptr[r]));
      pmax[w] = std::max(pmax[w], hp[r + 1] - hp[r]);
    }
    int st = 0;
    for (int w = 0; w < nwarps; ++w) st += 32 * lmax[w] * W;
    return st;
  };
  int r0 = (int)cb0;
  const int rend = (int)cb1;
  while (r0 < rend) {
    int r1 = std::min(rend, r0 + trows);
    std::vector<int> cells;
    int slots = 0;
    auto fits = [&](int a, int b) {
      if (W * (nptr[b] - nptr[a]) > sp.tile_seg || warp_sizes(a, b) > sp.tile_seg) return false;
      if (hp[b] - hp[a] > sp.tile_pairs) return false;
      for (int r = a; r < b; ++r)
        if (hp[r + 1] - hp[r] > 255) return false;
      ++gen;
      cells.clear();
      vid.clear();
      for (int p = hp[a]; p < hp[b]; ++p) { // distinct cells (pair order) and their distinct vertices
        const int c = hpairs[p] / nrn;
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
      if ((int)cells.size() > std::min(sp.tile_cells, 1023)) return false;
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
    const int segT = warp_sizes(r0, r1);
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
    int rwords = 0;
    for (int w = 0; w < nwarps; ++w) rwords += pmax[w] * rbw * 32;
    if (rwords > 65535 || segT > 65535) {
      O.ok = false;
      return;
    }
    const int off_srow = 0, off_np = up16((nrows + 1) * 2), off_recs = off_np + up16(2 * trows + 8 * nwarps),
              off_cells = off_recs + up16(rwords * 4), bytes = off_cells + up16(ncell * nv * 2);
    const size_t b0 = blob.size();
    blob.resize(b0 + bytes, 0);
    uint8_t* bp = blob.data() + b0;
    for (int r = 0; r <= nrows; ++r) {
      const uint16_t sr = (uint16_t)(nptr[r0 + r] - nptr[r0]);
      memcpy(bp + off_srow + 2 * r, &sr, 2);
    }
    for (int r = 0; r < nrows; ++r) bp[off_np + r] = (uint8_t)(hp[r0 + r + 1] - hp[r0 + r]);
    for (int l = 0; l < nrows; ++l) bp[off_np + trows + 8 * nwarps + l] = (uint8_t)lrow[l];
    {
      int sb = 0, wb = 0;
      for (int w = 0; w < nwarps; ++w) {
        const uint16_t wm[4] = {(uint16_t)sb, (uint16_t)wb, (uint16_t)lmax[w], 0};
        memcpy(bp + off_np + trows + 8 * w, wm, 8);
        for (int l = 0; l < 32 && 32 * w + l < nrows; ++l) {
          const int r = r0 + lrow[32 * w + l];
          for (int p = hp[r]; p < hp[r + 1]; ++p) {
            uint8_t rec[16];
            memcpy(rec, &recs[(size_t)p * rb], rb);
            uint32_t h;
            memcpy(&h, rec, 4);
            h |= (uint32_t)local_of(hpairs[p] / nrn);
            memcpy(rec, &h, 4);
            const int pi = p - hp[r];
            for (int q = 0; q < rbw; ++q)
              memcpy(bp + off_recs + 4 * ((size_t)wb + (pi * rbw + q) * 32 + l), rec + 4 * q, 4);
          }
        }
        sb += 32 * lmax[w] * W;
        wb += pmax[w] * rbw * 32;
      }
    }
    for (int q = 0; q < ncell; ++q)
      for (int v = 0; v < nv; ++v) {
        const uint16_t sl = (uint16_t)slot_in(hx[(size_t)cells[q] * nv + v]);
        memcpy(bp + off_cells + 2 * (q * nv + v), &sl, 2);
      }
    const int seg = (int)(W * (nptr[r1] - nptr[r0]));
    tiles.insert(tiles.end(), {(int)(b0 / 16), bytes, r0, nrows, (int)(W * nptr[r0]), seg, segT, ncell,
                               (int)runs.size() / 2, (int)rr.size(), off_srow, off_np, off_recs, off_cells, 0, 0});
    for (auto& x : rr) runs.insert(runs.end(), {x.first, x.second});
    O.max_seg = std::max(O.max_seg, seg);
    O.max_segT = std::max(O.max_segT, segT);
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
    out.max_seg = std::max(out.max_seg, O.max_seg);
    out.max_segT = std::max(out.max_segT, O.max_segT);
    out.max_cells = std::max(out.max_cells, O.max_cells);
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_blob = std::max(out.max_blob, O.max_blob);
  }
  upload_parts(out.blob, parts, s); // the chunks' blobs, uploaded in place (no host concatenation)
  tch.clear();
  out.form = form;
  out.ntiles = (int)tiles.size() / 16;
  out.tile_threads = trows;
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

struct RtileArgs {
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
  int off_seg, off_geo, off_buf, buf_bytes, b_win;
};

__device__ __forceinline__ void rt_wait(uint64_t* bar, uint32_t parity) {
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

template <int D>
struct RtGeo { // per cell in shared memory: g_0..g_D (D doubles each), V; odd stride in 16-byte units
  static constexpr int GS = D == 2 ? 10 : 18, VOFF = (D + 1) * D;
};

template <class F, int NT, int STAGES>
__global__ void __launch_bounds__(NT + 32, 1) k_rtile(const __grid_constant__ RtileArgs a) {
  constexpr int GD = F::GD, NV = GD + 1, RD = F::RD, CD = F::CD, NCN = F::NCN, NC = F::NC;
  constexpr int GS = RtGeo<GD>::GS, VOFF = RtGeo<GD>::VOFF;
  constexpr int RB = (4 + NCN + 3) & ~3, RBW = RB / 4;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  int* slot_tile = reinterpret_cast<int*>(sm + 48);
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
    auto grab = [&]() {
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
                      reinterpret_cast<double*>(buf + a.b_win), GD};
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
  double* segT = reinterpret_cast<double*>(sm + a.off_seg); // lane-interleaved row segments
  double* geo = reinterpret_cast<double*>(sm + a.off_geo);  // cell geometry; then the contiguous segment
  const int lane = tid & 31, warp = tid >> 5;
  for (int k = 0;; ++k) {
    rt_wait(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    int m[16];
    meta(tile, m);
    const int nrows = m[3], E0 = m[4], len = m[5], lenT = m[6], ncell = m[7];
    const unsigned char* buf = ring(k);
    const uint16_t* srow = reinterpret_cast<const uint16_t*>(buf + m[10]);
    const uint8_t* npair = buf + m[11];
    const uint16_t* wmeta = reinterpret_cast<const uint16_t*>(buf + m[11] + NT);
    const uint8_t* lrow = buf + m[11] + NT + 8 * (NT / 32);
    const uint32_t* recs = reinterpret_cast<const uint32_t*>(buf + m[12]);
    const uint16_t* cslot = reinterpret_cast<const uint16_t*>(buf + m[13]);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    if (tid == 0) bulk_wait_read<0>(); // the previous tile's store has read the segment (in geo)
    named_bar(1, NT);
    // phase 1: gradients and measure of every cell of the tile, once
    for (int c = tid; c < ncell; c += NT) {
      double X[NV][GD];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int sl = cslot[c * NV + v];
#pragma unroll
        for (int q = 0; q < GD; ++q) X[v][q] = win[sl * GD + q];
      }
      Geom<GD> Gm;
      geometry<GD>(X, Gm);
      double* g = geo + c * GS;
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int q = 0; q < GD; ++q) g[v * GD + q] = Gm.g[v][q];
      g[VOFF] = Gm.V;
    }
    {
      double2* z = reinterpret_cast<double2*>(segT);
      for (int t = tid; t < (lenT >> 1); t += NT) z[t] = make_double2(0.0, 0.0);
    }
    named_bar(1, NT);
    // phase 2: one thread per row node (all RD dof rows)
    int s0 = 0, L = 0;
    const int sb = wmeta[4 * warp], rbase = wmeta[4 * warp + 1], Lm = wmeta[4 * warp + 2];
    double* my = segT + sb + lane; // entry (d, col) of this row at my[32 (d CD Lm + col)]
    if (tid < nrows) {
      const int row = lrow[tid];
      s0 = srow[row];
      L = srow[row + 1] - s0;
      const int np = npair[row];
      const uint32_t* rq = recs + rbase + lane;
      for (int p = 0; p < np; ++p) {
        uint32_t w[RBW];
#pragma unroll
        for (int q = 0; q < RBW; ++q) w[q] = rq[(p * RBW + q) * 32];
        const uint32_t h = w[0];
        const double* g = geo + (h & 1023u) * GS;
        double gv[NV][GD];
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int q = 0; q < GD; ++q) gv[v][q] = g[v * GD + q];
        Geom<GD> Gc; // canonical vertex mm = original local vertex inv(mm)
#pragma unroll
        for (int mm = 0; mm < NV; ++mm) {
          const int iv = (h >> (10 + 2 * mm)) & 3;
#pragma unroll
          for (int q = 0; q < GD; ++q) {
            double x = gv[0][q];
#pragma unroll
            for (int v = 1; v < NV; ++v) x = iv == v ? gv[v][q] : x;
            Gc.g[mm][q] = x;
          }
        }
        Gc.V = g[VOFF];
        double blk[RD * NC];
        if constexpr (F::NRN > NV) {
          if ((h >> 18) & 1u) F::row(NV, Gc, nullptr, a.prm, blk);
          else F::row(0, Gc, nullptr, a.prm, blk);
        } else {
          F::row(0, Gc, nullptr, a.prm, blk);
        }
        int pos[NCN];
#pragma unroll
        for (int j = 0; j < NCN; ++j) pos[j] = (int)((w[(4 + j) >> 2] >> (8 * ((4 + j) & 3))) & 0xffu);
#pragma unroll
        for (int d = 0; d < RD; ++d) {
          double cur[NC];
#pragma unroll
          for (int j = 0; j < NCN; ++j)
#pragma unroll
            for (int c = 0; c < CD; ++c)
              if (!diag_block<F>::value || d == c) cur[j * CD + c] = my[32 * (d * CD * Lm + pos[j] * CD + c)];
#pragma unroll
          for (int j = 0; j < NCN; ++j)
#pragma unroll
            for (int c = 0; c < CD; ++c)
              if (!diag_block<F>::value || d == c) // structurally zero blocks (Stokes A) keep the zero-fill
                my[32 * (d * CD * Lm + pos[j] * CD + c)] = cur[j * CD + c] + blk[d * NC + j * CD + c];
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]);
    named_bar(1, NT); // geometry reads done: geo becomes the contiguous segment
    double* seg = geo + (E0 & 1);
#pragma unroll
    for (int d = 0; d < RD; ++d) {
      const int rs = RD * CD * s0 + d * CD * L;
      for (int t = 0; t < CD * L; ++t) seg[rs + t] = my[32 * (d * CD * Lm + t)];
    }
    if (a.accumulate) {
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] += seg[t];
    } else {
      fence_async_shared();
      named_bar(1, NT);
      if (tid == 0) {
        double* dst = a.out + E0;
        const int hh = E0 & 1, t1 = len - ((E0 + len) & 1);
        if (hh && len > 0) dst[0] = seg[0];
        if (t1 > hh) {
          bulk_s2g(dst + hh, seg + hh, (uint32_t)(t1 - hh) * 8);
          bulk_commit();
        }
        if (t1 < len && t1 >= hh) dst[t1] = seg[t1];
      }
    }
  }
  if (tid == 0) bulk_wait_read<0>();
  tile_counter_release(a.next_tile, a.reset_tile, NT, tid);
}

template <class F>
void go_rtile(const RtilePlan& p, const RtileArgs& a, size_t base, size_t buf, cudaStream_t s) {
  auto go = [&](auto kern, int threads, int stages) {
    const size_t smem = base + stages * buf;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, threads, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "row-tile kernel does not fit on an SM");
    launch_pdl(kern, dim3(std::min(p.ntiles, blocks * kNumSMs)), dim3(threads), smem, s, a);
  };
  static const int st = std::getenv("LOAM_GPU_RT_STAGES") ? std::atoi(std::getenv("LOAM_GPU_RT_STAGES")) : 2;
  if (p.tile_threads == 64) {
    if (st >= 2) go(k_rtile<F, 64, 2>, 96, 2);
    else go(k_rtile<F, 64, 1>, 96, 1);
  } else {
    if (st >= 2) go(k_rtile<F, 128, 2>, 160, 2);
    else go(k_rtile<F, 128, 1>, 160, 1);
  }
}

} // namespace

void launch_rtile(const RtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s) {
  if (p.ntiles == 0) return;
  RtileArgs a{};
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
  int off = 128;
  a.off_seg = off;
  off += up16(p.max_segT * 8);
  a.off_geo = off;
  off += up16(std::max(p.max_cells * RtGeo<2>::GS, p.max_seg + 2) * 8);
  a.off_buf = off;
  a.b_win = up16(p.max_blob);
  a.buf_bytes = a.b_win + up16(p.max_slots * 2 * 8 + 16);
  if (p.form == F_STOKES_B) go_rtile<FormT<F_STOKES_B, 2, 2>>(p, a, off, a.buf_bytes, s);
  else if (p.form == F_STOKES_A) go_rtile<FormT<F_STOKES_A, 2, 2>>(p, a, off, a.buf_bytes, s);
  else if (p.form == F_STOKES_BT) go_rtile<FormT<F_STOKES_BT, 2, 2>>(p, a, off, a.buf_bytes, s);
  else fail(LOAM_ERR(InvalidArgument), "row tiles: unsupported form");
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
