#include <atomic>
#include <chrono>
// ntile.cu -- node-block tiles for vector P1 matrices (see ntile.cuh).
//
// Reference path replaced: assemble_matrix (fem/assemble.hpp:85-104) ->
// execute (parloop.hpp:191-384) with a dof-expanded map and the
// linear-elasticity element kernel (restated in elements.cuh FormT<F_ELASTICITY>),
// Mat::addto (data.hpp:205-222) on the 3x3-blocked pattern of
// build_sparsity(map, map, 3, 3) (data.hpp:149-179).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "ntile.cuh"
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

constexpr int kNV = 4;        // P1 tet
constexpr int kNtConsumers = 128; // consumer threads per CTA (= k_ntile's NT)
#ifndef LOAM_GPU_NT_SPLIT
#define LOAM_GPU_NT_SPLIT 4
#endif
constexpr int kDiagSplit = LOAM_GPU_NT_SPLIT; // threads per diagonal block (its 24 cells in chunks)
static_assert(kDiagSplit >= 1 && kDiagSplit <= 32 && (kDiagSplit & (kDiagSplit - 1)) == 0,
              "diagonal parts are combined within a power-of-two lane group");

} // namespace

bool build_ntile(NtilePlan& out, const NtileSpec& sp, int ncells, int nnodes, const int32_t* sorted_rows,
                 const int32_t* sorted_x, int nverts, const PairPlan& pp, const int64_t* row_ptr, int64_t nnz,
                 cudaStream_t s) {
  if (pp.nrn != kNV || pp.ncn != kNV || nnz >= (int64_t(1) << 31) || ncells == 0) return false;
  const int64_t np = pp.npairs;
  auto hrows = host_array<int32_t>((size_t)ncells * kNV), hx = host_array<int32_t>((size_t)ncells * kNV),
       hpairs = host_array<int32_t>(np), hp = host_array<int32_t>(nnodes + 1);
  auto hrank = host_array<uint8_t>((size_t)np * kNV);
  auto hrp = host_array<int64_t>((size_t)nnodes * 3 + 1);
  parallel_d2h({{hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size()},
                {hx.data(), sorted_x, sizeof(int32_t) * hx.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * (size_t)np},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * (size_t)(nnodes + 1)},
                {hrank.data(), pp.ranks.get(), hrank.size()},
                {hrp.data(), row_ptr, sizeof(int64_t) * hrp.size()}},
               s);
  plan_tick("ntile: D2H", s);
  std::vector<int64_t> nptr(nnodes + 1); // node-level pattern offsets of the 3x3-blocked CSR
  for (int i = 0; i <= nnodes; ++i) nptr[i] = hrp[(size_t)3 * i] / 9;
  // every pattern block of every row must be reached by some cell (exact (map, map) pattern)
  {
    std::atomic<bool> exact{true};
    parallel_chunks(nnodes, 1, [&](int, int64_t v0, int64_t v1) {
      std::vector<uint8_t> seen;
      for (int64_t v = v0; v < v1 && exact; ++v) {
        const int L = (int)(nptr[v + 1] - nptr[v]);
        seen.assign(L, 0);
        for (int p = hp[v]; p < hp[v + 1]; ++p)
          for (int j = 0; j < kNV; ++j) {
            const int r = hrank[(size_t)p * kNV + j];
            if (r >= L) {
              exact = false;
              return;
            }
            seen[r] = 1;
          }
        for (int r = 0; r < L; ++r)
          if (!seen[r]) {
            exact = false;
            return;
          }
      }
    });
    if (!exact) return false;
  }
  plan_tick("ntile: exact-pattern check", s);
  struct ItemRec { // 8 bytes
    uint16_t poff;
    uint8_t np, kind;
    uint16_t base, stride;
  };
  static_assert(sizeof(ItemRec) == 8, "item record");
  // tiles of consecutive node rows: chunks of rows tiled on all host cores and
  // concatenated (blob / run offsets shifted)
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs;
    std::vector<uint8_t> blob;
    int max_seg = 0, max_cells = 0, max_slots = 0, max_blob = 0, max_diag = 0;
    double t_fits = 0, t_items = 0, t_blob = 0; // developer timing (LOAM_GPU_PLAN_TIMING)
    int64_t n_fits = 0, n_tiles = 0;
  };
  std::vector<TileChunk> tch(plan_threads());
  const int ntch = parallel_chunks(nnodes, sp.tile_nodes, [&](int t, int64_t cb0, int64_t cb1) {
  TileChunk& O = tch[t];
  std::vector<int32_t>& tiles = O.tiles;
  std::vector<int32_t>& runs = O.runs;
  std::vector<uint8_t>& blob = O.blob;
  std::vector<int> vid;
  std::vector<std::pair<int, int>> rr;
  // per-tile scratch reused across tiles (no allocation in the hot loop)
  std::vector<uint32_t> flat;   // a row's per-rank lists, flattened: (cell << 4 | lv << 2 | lw)
  std::vector<int> lcnt, lpos;  // per-rank list offsets / fill cursors
  std::vector<ItemRec> items, ditems;
  std::vector<uint16_t> prec, diaginfo, dprec, inter;
  std::vector<int> cells, base;
  // generation stamps over all cells / vertices: calloc'd, so only the pages a
  // chunk touches are ever mapped (a chunk's tiles stay in a narrow id range)
  struct Stamps {
    int* p;
    explicit Stamps(size_t n) : p(static_cast<int*>(std::calloc(n + 1, sizeof(int)))) {
      if (!p) throw std::bad_alloc();
    }
    ~Stamps() { std::free(p); }
  } cstamp(ncells), vstamp(nverts), clocal(ncells);
  int gen = 0;
  const int vend = (int)cb1;
  int v0 = (int)cb0;
  while (v0 < vend) {
    int v1 = std::min(vend, v0 + sp.tile_nodes);
    int slots = 0;
    auto fits = [&](int a, int b) {
      if (9 * (nptr[b] - nptr[a]) > 60000) return false;
      int nit = 0, npr = 0;
      for (int v = a; v < b; ++v) {
        nit += (int)(nptr[v + 1] - nptr[v]) - 1 + kDiagSplit;
        npr += 4 * (hp[v + 1] - hp[v]);
      }
      if (nit > sp.tile_items || npr > sp.tile_pairs) return false;
      ++gen;
      cells.clear();
      vid.clear();
      for (int p = hp[a]; p < hp[b]; ++p) { // distinct cells (pair order) and their distinct vertices
        const int c = hpairs[p] / kNV;
        if (cstamp.p[c] == gen) continue;
        cstamp.p[c] = gen;
        clocal.p[c] = (int)cells.size();
        cells.push_back(c);
        for (int v = 0; v < kNV; ++v) {
          const int x = hx[(size_t)c * kNV + v];
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
    const auto tp0 = std::chrono::steady_clock::now();
    int nfits = 1;
    while (!fits(v0, v1)) {
      if (v1 == v0 + 1) { O.ok = false; return; }
      v1 = v0 + (v1 - v0) / 2;
      ++nfits;
    }
    const auto tp1 = std::chrono::steady_clock::now();
    O.t_fits += std::chrono::duration<double>(tp1 - tp0).count();
    O.n_fits += nfits;
    // cells in id order (the locality order: neighbouring cells share Gram /
    // gradient rows in shared memory), local ids renumbered to match
    std::sort(cells.begin(), cells.end());
    for (size_t q = 0; q < cells.size(); ++q) clocal.p[cells[q]] = (int)q;
    auto local_of = [&](int c) { return clocal.p[c]; };
    base.resize(rr.size());
    for (size_t q = 0, acc = 0; q < rr.size(); ++q) {
      base[q] = (int)acc;
      acc += rr[q].second - rr[q].first;
    }
    auto slot_in = [&](int v) {
      size_t q = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
      return base[q] + v - rr[q].first;
    };
    // items: off-diagonal blocks of every row first, then the diagonal blocks in kDiagSplit parts
    items.clear();
    prec.clear();
    diaginfo.clear();
    ditems.clear();
    dprec.clear();
    const int64_t S0 = nptr[v0];
    for (int v = v0; v < v1; ++v) {
      const int L = (int)(nptr[v + 1] - nptr[v]);
      // per-rank lists in (pair, lw) order, flattened by a counting pass
      lcnt.assign(L + 1, 0);
      for (int p = hp[v]; p < hp[v + 1]; ++p)
        for (int lw = 0; lw < kNV; ++lw) ++lcnt[hrank[(size_t)p * kNV + lw] + 1];
      for (int r = 0; r < L; ++r) lcnt[r + 1] += lcnt[r];
      lpos.assign(lcnt.begin(), lcnt.end() - 1);
      flat.resize(lcnt[L]);
      int self = -1;
      for (int p = hp[v]; p < hp[v + 1]; ++p) {
        const int c = hpairs[p] / kNV, lv = hpairs[p] % kNV;
        const uint32_t loc = (uint32_t)local_of(c) << 4;
        for (int lw = 0; lw < kNV; ++lw) {
          const int r = hrank[(size_t)p * kNV + lw];
          flat[lpos[r]++] = loc | (uint32_t)lv << 2 | (uint32_t)lw;
          if (lw == lv) self = r;
        }
      }
      const uint16_t rowb = (uint16_t)(9 * (nptr[v] - S0)), stride = (uint16_t)(3 * L);
      for (int r = 0; r < L; ++r) {
        if (r == self) continue;
        const int len = lcnt[r + 1] - lcnt[r];
        if (len > 255) { O.ok = false; return; }
        items.push_back(ItemRec{(uint16_t)prec.size(), (uint8_t)len, 0, (uint16_t)(rowb + 3 * r), stride});
        for (int q = lcnt[r]; q < lcnt[r + 1]; ++q) prec.push_back((uint16_t)flat[q]);
      }
      const int di = (int)diaginfo.size() / 2;
      diaginfo.push_back((uint16_t)(rowb + 3 * self));
      diaginfo.push_back(stride);
      const uint32_t* dl = flat.data() + lcnt[self];
      const int n = lcnt[self + 1] - lcnt[self];
      for (int part = 0; part < kDiagSplit; ++part) {
        const int a = n * part / kDiagSplit, b = n * (part + 1) / kDiagSplit;
        ditems.push_back(ItemRec{(uint16_t)dprec.size(), (uint8_t)(b - a), 1, (uint16_t)(di * kDiagSplit + part), 0});
        for (int q = a; q < b; ++q) dprec.push_back((uint16_t)dl[q]);
      }
    }
    // the kDiagSplit parts of a diagonal block sit on consecutive lanes of one
    // aligned lane group (combined by shuffles): pad with no-op items
    // blocks of equal pair counts share warps (a warp's pair loop runs to its longest item)
    std::stable_sort(items.begin(), items.end(), [](const ItemRec& x, const ItemRec& y) { return x.np > y.np; });
    while (items.size() % kDiagSplit) items.push_back(ItemRec{0, 0, 2, 0, 0});
    for (auto it : ditems) {
      it.poff = (uint16_t)(it.poff + prec.size());
      items.push_back(it);
    }
    prec.insert(prec.end(), dprec.begin(), dprec.end());
    // lane-interleaved records: the items run in rounds of kNtConsumers
    // threads; pair q of the item on lane l of round r sits at
    // block(r) + q * kNtConsumers + l (the lanes of a warp read consecutive
    // half-words: no shared-memory bank conflicts)
    {
      inter.clear();
      for (size_t r0i = 0; r0i < items.size(); r0i += kNtConsumers) {
        const size_t r1i = std::min(items.size(), r0i + kNtConsumers);
        int pm = 0;
        for (size_t i = r0i; i < r1i; ++i) pm = std::max<int>(pm, items[i].np);
        const size_t blk = inter.size();
        inter.resize(blk + (size_t)pm * kNtConsumers, 0);
        for (size_t i = r0i; i < r1i; ++i) {
          const int l = (int)(i - r0i);
          for (int q = 0; q < items[i].np; ++q) inter[blk + (size_t)q * kNtConsumers + l] = prec[items[i].poff + q];
          if (blk + l > 65535) { O.ok = false; return; }
          items[i].poff = (uint16_t)(blk + l);
        }
      }
      prec.swap(inter);
    }
    const auto tp2 = std::chrono::steady_clock::now();
    O.t_items += std::chrono::duration<double>(tp2 - tp1).count();
    const int nitems = (int)items.size(), npairs = (int)prec.size(), ncell = (int)cells.size(),
              ndiag = (int)diaginfo.size() / 2;
    const int off_items = 0, off_pairs = up16(nitems * 8), off_diag = off_pairs + up16(npairs * 2),
              off_cells = off_diag + up16(ndiag * 4), bytes = off_cells + up16(ncell * kNV * 2);
    const size_t b0 = blob.size();
    blob.resize(b0 + bytes, 0);
    uint8_t* bp = blob.data() + b0;
    memcpy(bp + off_items, items.data(), (size_t)nitems * 8);
    memcpy(bp + off_pairs, prec.data(), (size_t)npairs * 2);
    memcpy(bp + off_diag, diaginfo.data(), (size_t)ndiag * 4);
    for (int q = 0; q < ncell; ++q)
      for (int v = 0; v < kNV; ++v) {
        const uint16_t sl = (uint16_t)slot_in(hx[(size_t)cells[q] * kNV + v]);
        memcpy(bp + off_cells + 2 * (q * kNV + v), &sl, 2);
      }
    const int seg = (int)(9 * (nptr[v1] - nptr[v0]));
    tiles.insert(tiles.end(), {(int)(b0 / 16), bytes, v0, v1 - v0, (int)(9 * nptr[v0]), seg, nitems, ncell,
                               (int)runs.size() / 2, (int)rr.size(), off_items, off_pairs, off_cells, off_diag, ndiag,
                               0});
    for (auto& x : rr) runs.insert(runs.end(), {x.first, x.second});
    O.max_seg = std::max(O.max_seg, seg);
    O.max_cells = std::max(O.max_cells, ncell);
    O.max_slots = std::max(O.max_slots, slots);
    O.max_blob = std::max(O.max_blob, bytes);
    O.max_diag = std::max(O.max_diag, ndiag);
    O.t_blob += std::chrono::duration<double>(std::chrono::steady_clock::now() - tp2).count();
    ++O.n_tiles;
    v0 = v1;
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
    out.max_cells = std::max(out.max_cells, O.max_cells);
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_blob = std::max(out.max_blob, O.max_blob);
    out.max_diag = std::max(out.max_diag, O.max_diag);
  }
  if (std::getenv("LOAM_GPU_PLAN_TIMING")) {
    double f = 0, it = 0, bl = 0;
    int64_t nf = 0, nt = 0;
    for (int t = 0; t < ntch; ++t) {
      f += tch[t].t_fits; it += tch[t].t_items; bl += tch[t].t_blob; nf += tch[t].n_fits; nt += tch[t].n_tiles;
    }
    fprintf(stderr, "[plan] ntile: %d chunks, %lld tiles, %lld fits calls; thread-seconds fits %.3f items %.3f blob %.3f\n",
            ntch, (long long)nt, (long long)nf, f, it, bl);
  }
  plan_tick("ntile: tiles", s);
  upload_parts(out.blob, parts, s); // the chunks' blobs, uploaded in place (no host concatenation)
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

struct NtileArgs {
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
  int off_seg, off_geo, off_part, off_buf, buf_bytes, b_win;
};

__device__ __forceinline__ void nt_wait(uint64_t* bar, uint32_t parity) {
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

constexpr int kNtThreads = 128;
#ifndef LOAM_GPU_NT_GS
#define LOAM_GPU_NT_GS 12
#endif
// doubles per cell: sqrt(V) g_k as 4 x (x, y) then 4 x z (12: the smallest
// record; phase 2 reads random cells, so an odd 16-byte stride buys little
// and the smaller footprint fits 4 CTAs per SM)
constexpr int kGS = LOAM_GPU_NT_GS;
static_assert(kGS >= 12 && kGS % 2 == 0, "cell record");

template <int STAGES>
__global__ void __launch_bounds__(kNtThreads + 32, 1) k_ntile(const __grid_constant__ NtileArgs a) {
  constexpr int NT = kNtThreads;
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
  if (tid >= NT) { // ---- producer warp
    const int lane = tid & 31;
    int sched = 0; // static round-robin (uniform tiles) unless a.dynamic
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
      if (lane == 0) {
        slot_tile[k % STAGES] = tile;
        int4* sm4 = slot_meta + 4 * (k % STAGES);
#pragma unroll
        for (int q = 0; q < 4; ++q) sm4[q] = make_int4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
      }
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % STAGES];
      const RunSet rc{reinterpret_cast<const int2*>(a.runs) + m[8], m[9], a.coords,
                      reinterpret_cast<double*>(buf + a.b_win), 3};
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
  double* seg0 = reinterpret_cast<double*>(sm + a.off_seg);
  double* geo = reinterpret_cast<double*>(sm + a.off_geo);
  const double lam = a.prm.p[0], mu = a.prm.p[1];
  for (int k = 0;; ++k) {
    nt_wait(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    int m[16];
    {
      const int4* sm4 = slot_meta + 4 * (k % STAGES);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 x = sm4[q];
        m[4 * q] = x.x;
        m[4 * q + 1] = x.y;
        m[4 * q + 2] = x.z;
        m[4 * q + 3] = x.w;
      }
    }
    const int E0 = m[4], len = m[5], nitems = m[6], ncell = m[7], ndiag = m[14];
    const unsigned char* buf = ring(k);
    const uint2* items = reinterpret_cast<const uint2*>(buf + m[10]);
    const uint16_t* prec = reinterpret_cast<const uint16_t*>(buf + m[11]);
    const uint16_t* cslot = reinterpret_cast<const uint16_t*>(buf + m[12]);
    const uint16_t* dinfo = reinterpret_cast<const uint16_t*>(buf + m[13]);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    double* seg = seg0 + (E0 & 1); // 16-byte parity of the global destination (bulk store)
    // phase 1: barycentric gradients and measure of every cell of the tile, once
    for (int c = tid; c < ((a.dbg & 2) ? 0 : ncell); c += NT) {
      double X[4][3];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int sl = cslot[c * 4 + v];
#pragma unroll
        for (int q = 0; q < 3; ++q) X[v][q] = win[sl * 3 + q];
      }
      Geom<3> Gm;
      geometry<3>(X, Gm);
      // sqrt(V) g_k: a node block sums V g_a g_b^T = (sqrt(V) g_a)(sqrt(V) g_b)^T over its cells
      const double sv = sqrt(Gm.V);
      double* gc = geo + c * kGS;
      double2* g = reinterpret_cast<double2*>(gc);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        g[v] = make_double2(sv * Gm.g[v][0], sv * Gm.g[v][1]);
        gc[8 + v] = sv * Gm.g[v][2];
      }
    }
    if (tid == 0) bulk_wait_read<0>(); // the previous tile's store has read the segment (overlapped with phase 1)
    named_bar(1, NT);
    // phase 2: one thread per 3x3 node block (diagonal blocks: kDiagSplit threads)
    for (int it = tid; it < nitems; it += NT) {
      const uint2 ir = items[it];
      const int poff = ir.x & 0xffff, np = (a.dbg & 1) ? 0 : (ir.x >> 16) & 0xff, kind = ir.x >> 24;
      const int base = ir.y & 0xffff, stride = ir.y >> 16;
      // S = sum over the block's cells of V g_a g_b^T (9 FMAs per cell); the
      // element block of FormT<F_ELASTICITY>::row is linear in it:
      //   A_de = mu S_ed + lam S_de + d_de mu tr(S)
      double acc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      // software pipeline: pair q+1's record and gradients load during pair q's FMAs
      auto fetch = [&](int q, double (&ga)[3], double (&gb)[3]) {
        const uint32_t x = prec[poff + q * NT];
        const double* g = geo + (x >> 4) * kGS;
        const int lv = (x >> 2) & 3, lw = x & 3;
        const double2 a0 = reinterpret_cast<const double2*>(g)[lv];
        const double2 b0 = reinterpret_cast<const double2*>(g)[lw];
        ga[0] = a0.x;
        ga[1] = a0.y;
        ga[2] = g[8 + lv];
        gb[0] = b0.x;
        gb[1] = b0.y;
        gb[2] = g[8 + lw];
      };
      double ga[3] = {0, 0, 0}, gb[3] = {0, 0, 0};
      if (np > 0) fetch(0, ga, gb);
      for (int q = 0; q < np; ++q) {
        double na[3] = {0, 0, 0}, nb[3] = {0, 0, 0};
        if (q + 1 < np) fetch(q + 1, na, nb);
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) acc[d][e] = fma(ga[d], gb[e], acc[d][e]);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          ga[d] = na[d];
          gb[d] = nb[d];
        }
      }
      if (kind == 2) continue; // padding before the diagonal groups
      int wb = base, ws = stride;
      if (kind == 1) {
        // diagonal block: its kDiagSplit parts are on the consecutive lanes
        // of one aligned group; the first lane sums them in part order
        // ((p0 + p1) + p2) + p3 -- the same bits on every run
        const int lane = tid & 31, g0 = lane & ~(kDiagSplit - 1);
        const unsigned gmask = ((1u << kDiagSplit) - 1u) << g0;
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            double v = acc[d][e];
#pragma unroll
            for (int s = 1; s < kDiagSplit; ++s) {
              const double o = __shfl_sync(gmask, acc[d][e], s, kDiagSplit);
              v += o;
            }
            acc[d][e] = v;
          }
        if (lane != g0) continue;
        const int di = base / kDiagSplit;
        wb = dinfo[2 * di];
        ws = dinfo[2 * di + 1];
      }
      const double tr = mu * (acc[0][0] + acc[1][1] + acc[2][2]);
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          double v = fma(mu, acc[e][d], lam * acc[d][e]);
          if (d == e) v += tr;
          seg[wb + d * ws + e] = v;
        }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]);
    if (a.accumulate) {
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] += seg[t];
      named_bar(1, NT);
    } else if (a.dbg & 4) { // developer: coalesced thread stores instead of the bulk store
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] = seg[t];
      named_bar(1, NT);
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

} // namespace

void launch_ntile(const NtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s) {
  if (p.ntiles == 0) return;
  NtileArgs a{};
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
  a.off_geo = off;
  off += up16(p.max_cells * kGS * 8);
  a.off_buf = off;
  a.b_win = up16(p.max_blob);
  a.buf_bytes = a.b_win + up16(p.max_slots * 3 * 8 + 16);
  static const int st = std::getenv("LOAM_GPU_NT_STAGES") ? std::atoi(std::getenv("LOAM_GPU_NT_STAGES")) : 2;
  auto go = [&](auto kern, int stages) {
    const size_t smem = (size_t)off + stages * (size_t)a.buf_bytes;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kNtThreads + 32, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "node-tile kernel does not fit on an SM");
    launch_pdl(kern, dim3(std::min(p.ntiles, blocks * kNumSMs)), dim3(kNtThreads + 32), smem, s, a);
  };
  if (std::getenv("LOAM_GPU_NT_INFO")) // developer: plan maxima behind the shared-memory footprint
    fprintf(stderr, "ntile: tiles %d max_seg %d max_cells %d max_blob %d max_slots %d max_diag %d smem/stage %d fixed %d\n",
            p.ntiles, p.max_seg, p.max_cells, p.max_blob, p.max_slots, p.max_diag, a.buf_bytes, off);
  a.dynamic = std::getenv("LOAM_GPU_NT_STATIC") ? 0 : 1;
  a.dbg = std::getenv("LOAM_GPU_NT_DBG") ? std::atoi(std::getenv("LOAM_GPU_NT_DBG")) : 0; // developer: skip phases
  if (st >= 3) go(k_ntile<3>, 3);
  else if (st == 2) go(k_ntile<2>, 2);
  else go(k_ntile<1>, 1);
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
