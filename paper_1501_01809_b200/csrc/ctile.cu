// ctile.cu -- cell tiles for P2 actions (see ctile.cuh).
//
// Reference path replaced: assemble_vector (fem/assemble.hpp:108-135) ->
// execute (parloop.hpp:191-384): stage-in gather (:268-273), the element
// kernel (the P2 Helmholtz action restated in elements.cuh / patch_kernels.cuh
// ElemVec), indirect INC stage-out (:301-308).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "ctile.cuh"
#include "patch_kernels.cuh"
#include "stage.cuh"

namespace loam_gpu {

namespace {

inline int up16(int x) { return (x + 15) & ~15; }

// windows of contiguous ids (even-aligned runs merged across gaps of <= 8)
int id_runs(std::vector<int>& ids, int limit, std::vector<std::pair<int, int>>& rr) {
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

#ifndef LOAM_GPU_CT_CELLS
#define LOAM_GPU_CT_CELLS 128
#endif
#ifndef LOAM_GPU_CT_THREADS
#define LOAM_GPU_CT_THREADS 128
#endif
constexpr int kCtCells = LOAM_GPU_CT_CELLS;     // cells per tile
constexpr int kCtThreadsN = LOAM_GPU_CT_THREADS; // consumer threads per CTA
constexpr int kCtMinBlocks = 512 / kCtThreadsN;  // CTAs per SM the register budget is sized for
constexpr int kCtMaxSlots = 4096, kCtMaxRuns = 64;

} // namespace

bool build_ctile(CtilePlan& out, int gd, int nrn, int ncells, const int32_t* sorted_rows, int nnodes, int nverts,
                 cudaStream_t s) {
  const int nv = gd + 1;
  if (ncells == 0 || nrn > 16) return false;
  std::vector<int32_t> hrows((size_t)ncells * nrn);
  LG_CUDA(cudaMemcpyAsync(hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size(), cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  plan_tick("ctile: D2H", s);
  // one tile per kCtCells consecutive sorted cells; chunks of tiles on all host cores
  struct Chunk {
    bool ok = true;
    std::vector<int32_t> tiles, xruns, cruns;
    std::vector<uint8_t> blob;
    int max_blob = 0, max_xslots = 0, max_cslots = 0;
  };
  std::vector<Chunk> ch(plan_threads());
  const int nch = parallel_chunks(ncells, kCtCells, [&](int t, int64_t cb0, int64_t cb1) {
    Chunk& O = ch[t];
    std::vector<int> vid, nid;
    std::vector<std::pair<int, int>> xr, cr;
    std::vector<int> xbase, cbase, cnt;
    std::vector<uint16_t> lst;
    for (int64_t c0 = cb0; c0 < cb1; c0 += kCtCells) {
      const int nc = (int)std::min<int64_t>(kCtCells, cb1 - c0);
      vid.clear();
      nid.clear();
      for (int c = 0; c < nc; ++c) {
        const int32_t* row = &hrows[(size_t)(c0 + c) * nrn];
        for (int i = 0; i < nv; ++i) vid.push_back(row[i]);
        for (int i = 0; i < nrn; ++i) nid.push_back(row[i]);
      }
      const int xs = id_runs(vid, nverts, xr), cs = id_runs(nid, nnodes, cr);
      if (xs > kCtMaxSlots || cs > kCtMaxSlots || (int)xr.size() > kCtMaxRuns || (int)cr.size() > kCtMaxRuns) {
        O.ok = false;
        return;
      }
      auto bases = [](const std::vector<std::pair<int, int>>& R, std::vector<int>& b) {
        b.resize(R.size());
        for (size_t k = 0, acc = 0; k < R.size(); ++k) {
          b[k] = (int)acc;
          acc += R[k].second - R[k].first;
        }
      };
      bases(xr, xbase);
      bases(cr, cbase);
      auto slot_in = [](const std::vector<std::pair<int, int>>& R, const std::vector<int>& b, int v) {
        const size_t k = std::upper_bound(R.begin(), R.end(), std::make_pair(v, INT32_MAX)) - R.begin() - 1;
        return b[k] + v - R[k].first;
      };
      // sections (16-byte aligned): vertex slots u16 [nc x nv], node slots u16
      // [nc x nrn], per node slot the entry-list offsets u16 [cs + 1], the
      // entries u16 (cell * nrn + i, ascending per slot) [nc x nrn], the node
      // runs int4 (lo, hi, slot base, 0) [ncr]
      const int off_x = 0, off_c = off_x + up16(nc * nv * 2), off_o = off_c + up16(nc * nrn * 2),
                off_l = off_o + up16((cs + 1) * 2), off_r = off_l + up16(nc * nrn * 2),
                off_ri = off_r + (int)cr.size() * 16, bytes = off_ri + up16(cs);
      const size_t b0 = O.blob.size();
      O.blob.resize(b0 + bytes, 0);
      uint8_t* bp = O.blob.data() + b0;
      cnt.assign(cs + 1, 0);
      std::vector<uint16_t> cslot((size_t)nc * nrn);
      for (int c = 0; c < nc; ++c) {
        const int32_t* row = &hrows[(size_t)(c0 + c) * nrn];
        for (int i = 0; i < nv; ++i) {
          const uint16_t sl = (uint16_t)slot_in(xr, xbase, row[i]);
          memcpy(bp + off_x + 2 * (c * nv + i), &sl, 2);
        }
        for (int i = 0; i < nrn; ++i) {
          const int sl = slot_in(cr, cbase, row[i]);
          cslot[(size_t)c * nrn + i] = (uint16_t)sl;
          ++cnt[sl + 1];
        }
      }
      memcpy(bp + off_c, cslot.data(), cslot.size() * 2);
      for (int q = 0; q < cs; ++q) cnt[q + 1] += cnt[q];
      for (int q = 0; q <= cs; ++q) {
        const uint16_t o = (uint16_t)cnt[q];
        memcpy(bp + off_o + 2 * q, &o, 2);
      }
      lst.assign((size_t)nc * nrn, 0);
      for (int e = 0; e < nc * nrn; ++e) lst[cnt[cslot[e]]++] = (uint16_t)e; // entries ascending per slot
      memcpy(bp + off_l, lst.data(), lst.size() * 2);
      for (size_t k = 0; k < cr.size(); ++k) {
        const int4 r = make_int4(cr[k].first, cr[k].second, cbase[k], 0);
        memcpy(bp + off_r + 16 * k, &r, 16);
        for (int q = cbase[k]; q < cbase[k] + cr[k].second - cr[k].first; ++q) bp[off_ri + q] = (uint8_t)k;
      }
      O.tiles.insert(O.tiles.end(), {(int)(b0 / 16), bytes, (int)c0, nc, cs, (int)cr.size(),
                                     (int)O.xruns.size() / 2, (int)xr.size(), (int)O.cruns.size() / 2, (int)cr.size(),
                                     off_c, off_o, off_l, off_r, xs, off_ri});
      for (auto& x : xr) O.xruns.insert(O.xruns.end(), {x.first, x.second});
      for (auto& x : cr) O.cruns.insert(O.cruns.end(), {x.first, x.second});
      O.max_blob = std::max(O.max_blob, bytes);
      O.max_xslots = std::max(O.max_xslots, xs);
      O.max_cslots = std::max(O.max_cslots, cs);
    }
  });
  std::vector<int32_t> tiles, xruns, cruns;
  std::vector<uint8_t> blob;
  for (int t = 0; t < nch; ++t) {
    Chunk& O = ch[t];
    if (!O.ok) return false;
    const int bshift = (int)(blob.size() / 16), xshift = (int)(xruns.size() / 2), cshift = (int)(cruns.size() / 2);
    for (size_t q = 0; q < O.tiles.size(); q += 16) {
      O.tiles[q + 0] += bshift;
      O.tiles[q + 6] += xshift;
      O.tiles[q + 8] += cshift;
    }
    tiles.insert(tiles.end(), O.tiles.begin(), O.tiles.end());
    xruns.insert(xruns.end(), O.xruns.begin(), O.xruns.end());
    cruns.insert(cruns.end(), O.cruns.begin(), O.cruns.end());
    blob.insert(blob.end(), O.blob.begin(), O.blob.end());
    out.max_blob = std::max(out.max_blob, O.max_blob);
    out.max_xslots = std::max(out.max_xslots, O.max_xslots);
    out.max_cslots = std::max(out.max_cslots, O.max_cslots);
  }
  ch.clear();
  out.ntiles = (int)tiles.size() / 16;
  out.nrn = nrn;
  out.nv = nv;
  out.tile_cells = kCtCells;
  auto upload = [&](auto& dst, const auto& src) {
    using T = typename std::decay_t<decltype(src)>::value_type;
    dst.alloc(src.size() + 16, s);
    if (!src.empty())
      LG_CUDA(cudaMemcpyAsync(dst.get(), src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s));
  };
  upload(out.tiles, tiles);
  upload(out.blob, blob);
  upload(out.xruns, xruns);
  upload(out.cruns, cruns);
  LG_CUDA(cudaStreamSynchronize(s));
  plan_tick("ctile: tiles", s);
  return true;
}

// ===========================================================================
// Device side
// ===========================================================================

namespace {

struct CtileArgs {
  const int32_t* tiles;
  int ntiles;
  int* next_tile;
  int* reset_tile;
  const uint8_t* blob;
  const int32_t* xruns;
  const int32_t* cruns;
  const double* coords;
  const double* coeff;
  double* out;
  FormParams prm;
  int off_ent, off_buf, buf_bytes, b_xwin, b_cwin;
};

constexpr int kCtThreads = kCtThreadsN; // consumers: cells strided (phase 1), entry chunks (phase 2)
constexpr int kCtStages = 2;

template <class F>
__global__ void __launch_bounds__(kCtThreads + 32, kCtMinBlocks) k_ctile(const __grid_constant__ CtileArgs a) {
  constexpr int NT = kCtThreads, NRN = F::NRN, GD = F::GD, NV = GD + 1, ST = kCtStages;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + ST;
  int* slot_tile = reinterpret_cast<int*>(sm + 48);
  __shared__ int stage_meta[ST][16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto ring = [&](int k) { return sm + a.off_buf + (k % ST) * a.buf_bytes; };
  __shared__ __align__(16) int feed_buf[2 * 8 * 16];
  if (tid >= NT) { // ---- producer warp: tile blob + vertex and node windows by TMA
    // static schedule (uniform tiles), records prefetched 8 at a time, the
    // next tile's first window runs loaded one tile ahead: no dependent
    // global round trip in the per-tile chain
    const int lane = tid & 31;
    const TileFeedT<16> feed{feed_buf, a.tiles, a.ntiles};
    feed.start(lane);
    int nm[16];
    int2 nxr = make_int2(0, 0), ncr = make_int2(0, 0);
    auto read = [&](int k) {
      const int* rec = feed.at(k);
      if (feed.tile(k) < a.ntiles) {
#pragma unroll
        for (int q = 0; q < 16; ++q) nm[q] = rec[q];
        nxr = first_run(reinterpret_cast<const int2*>(a.xruns) + nm[6], nm[7], lane);
        ncr = first_run(reinterpret_cast<const int2*>(a.cruns) + nm[8], nm[9], lane);
      }
      feed.done(k, lane);
    };
    read(0);
    for (int k = 0;; ++k) {
      const int tile = feed.tile(k);
      int m[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) m[q] = nm[q];
      const int2 xr0 = nxr, cr0 = ncr;
      if (k >= ST) mbar_wait_sleep(&empty[k % ST], (k / ST - 1) & 1);
      if (tile >= a.ntiles) {
        if (lane == 0) {
          slot_tile[k % ST] = -1;
          mbar_arrive(&full[k % ST]);
        }
        break;
      }
      if (lane < 16) stage_meta[k % ST][lane] = m[lane];
      if (lane == 0) slot_tile[k % ST] = tile;
      unsigned char* buf = ring(k);
      uint64_t* bar = &full[k % ST];
      const RunSet rx{reinterpret_cast<const int2*>(a.xruns) + m[6], m[7], a.coords,
                      reinterpret_cast<double*>(buf + a.b_xwin), GD};
      const RunSet rc{reinterpret_cast<const int2*>(a.cruns) + m[8], m[9], a.coeff,
                      reinterpret_cast<double*>(buf + a.b_cwin), 1};
      const uint32_t tx = (uint32_t)m[1] + stage_runs<false>(rx, lane, bar, xr0) + stage_runs<false>(rc, lane, bar, cr0);
      fence_async_shared();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(bar, tx);
        bulk_g2s(buf, a.blob + (int64_t)m[0] * 16, (uint32_t)m[1], bar);
      }
      __syncwarp();
      stage_runs<true>(rx, lane, bar, xr0);
      stage_runs<true>(rc, lane, bar, cr0);
      read(k + 1);
    }
    feed.drain();
    return;
  }
  // ---- consumers
  double* ent = reinterpret_cast<double*>(sm + a.off_ent); // element-vector entries, cell-major
  for (int k = 0;; ++k) {
    mbar_wait(&full[k % ST], (k / ST) & 1);
    const int tile = slot_tile[k % ST];
    if (tile < 0) break;
    int m[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) m[q] = stage_meta[k % ST][q];
    const int nc = m[3], ncs = m[4];
    const unsigned char* buf = ring(k);
    const uint16_t* xslot = reinterpret_cast<const uint16_t*>(buf);
    const uint16_t* cslot = reinterpret_cast<const uint16_t*>(buf + m[10]);
    const uint16_t* soff = reinterpret_cast<const uint16_t*>(buf + m[11]);
    const uint16_t* lst = reinterpret_cast<const uint16_t*>(buf + m[12]);
    const int4* crun = reinterpret_cast<const int4*>(buf + m[13]);
    const uint8_t* rix = buf + m[15]; // run index of every node slot
    const double* xwin = reinterpret_cast<const double*>(buf + a.b_xwin);
    const double* cwin = reinterpret_cast<const double*>(buf + a.b_cwin);
    // phase 1: one cell per thread, element vector into shared memory
#pragma unroll 2
    for (int c = tid; c < nc; c += NT) {
      double X[NV][GD], C[F::NCOEFF];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int sl = xslot[c * NV + v];
#pragma unroll
        for (int d = 0; d < GD; ++d) X[v][d] = xwin[sl * GD + d];
      }
#pragma unroll
      for (int q = 0; q < F::NCOEFF; ++q) C[q] = cwin[cslot[c * NRN + q]];
      Geom<GD> G;
      geometry<GD>(X, G);
      double y[NRN];
      ElemVec<F>::all(G, C, a.prm, y);
#pragma unroll
      for (int i = 0; i < NRN; ++i) ent[c * NRN + i] = y[i];
    }
    named_bar(1, NT);
    // phase 2: the tile's entries in node-slot order (lst), split into equal
    // contiguous chunks, one per thread; a thread sums each run of equal
    // slots in order (cells ascending) and issues one RED per run -- one per
    // distinct node of the tile, plus one where a node straddles two chunks
    {
      const int E = nc * NRN, e0 = (int)((int64_t)tid * E / NT), e1 = (int)((int64_t)(tid + 1) * E / NT);
      int cur = -1;
      double acc = 0.0;
      auto flush = [&] {
        const int4 run = crun[rix[cur]]; // (lo, hi, slot base)
        atomicAdd(a.out + run.x + (cur - run.z), acc);
      };
      for (int p = e0; p < e1; ++p) {
        const int e = lst[p];
        const int sl = cslot[e];
        const double v = ent[e];
        if (sl != cur) {
          if (cur >= 0) flush();
          cur = sl;
          acc = v;
        } else {
          acc += v;
        }
      }
      if (cur >= 0) flush();
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % ST]);
    named_bar(1, NT); // entries consumed before the next tile overwrites them
  }
  tile_counter_release(a.next_tile, a.reset_tile, NT, tid);
}

template <class F>
void go_ctile(const CtileArgs& a, size_t smem, int ntiles, cudaStream_t s) {
  ensure_dynamic_smem(reinterpret_cast<const void*>(k_ctile<F>), smem);
  int blocks = 1;
  LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_ctile<F>, kCtThreads + 32, smem));
  require(blocks > 0, LOAM_GPU_ERR_CUDA, "cell-tile kernel does not fit on an SM");
  k_ctile<F><<<std::min(ntiles, blocks * kNumSMs), kCtThreads + 32, smem, s>>>(a);
}

} // namespace

void launch_ctile(int form, const CtilePlan& p, const double* coords, const double* coeff, double* out,
                  int64_t nout, const FormParams& prm, bool accumulate, int* next_tile, int* reset_tile,
                  cudaStream_t s) {
  if (!accumulate) LG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)nout, s));
  if (p.ntiles == 0) return;
  CtileArgs a{};
  a.tiles = p.tiles.get();
  a.ntiles = p.ntiles;
  a.next_tile = next_tile;
  a.reset_tile = reset_tile;
  a.blob = p.blob.get();
  a.xruns = p.xruns.get();
  a.cruns = p.cruns.get();
  a.coords = coords;
  a.coeff = coeff;
  a.out = out;
  a.prm = prm;
  int off = 128;
  a.off_ent = off;
  off += up16(kCtCells * p.nrn * 8);
  a.off_buf = off;
  const int gd = p.nv - 1;
  a.b_xwin = up16(p.max_blob);
  a.b_cwin = a.b_xwin + up16(p.max_xslots * gd * 8 + 16);
  a.buf_bytes = a.b_cwin + up16(p.max_cslots * 8 + 16);
  const size_t smem = (size_t)off + kCtStages * (size_t)a.buf_bytes;
  if (std::getenv("LOAM_GPU_CT_INFO")) // developer: plan maxima behind the shared-memory footprint
    fprintf(stderr, "ctile: tiles %d max_blob %d max_xslots %d max_cslots %d stage %d smem %zu\n", p.ntiles,
            p.max_blob, p.max_xslots, p.max_cslots, a.buf_bytes, smem);
  if (gd == 3 && p.nrn == 10) {
    if (form == F_HELMHOLTZ_ACTION) go_ctile<FormT<F_HELMHOLTZ_ACTION, 3, 2>>(a, smem, p.ntiles, s);
    else if (form == F_STIFFNESS_ACTION) go_ctile<FormT<F_STIFFNESS_ACTION, 3, 2>>(a, smem, p.ntiles, s);
    else go_ctile<FormT<F_MASS_ACTION, 3, 2>>(a, smem, p.ntiles, s);
  } else if (gd == 2 && p.nrn == 6) {
    if (form == F_HELMHOLTZ_ACTION) go_ctile<FormT<F_HELMHOLTZ_ACTION, 2, 2>>(a, smem, p.ntiles, s);
    else if (form == F_STIFFNESS_ACTION) go_ctile<FormT<F_STIFFNESS_ACTION, 2, 2>>(a, smem, p.ntiles, s);
    else go_ctile<FormT<F_MASS_ACTION, 2, 2>>(a, smem, p.ntiles, s);
  } else {
    fail(LOAM_ERR(InvalidArgument), "cell tiles: P2 triangle / tetrahedron actions only");
  }
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
