// ltile.cu -- edge-link tiles for vector P1 matrices on tetrahedra (see ltile.cuh).
//
// Reference path replaced: assemble_matrix (fem/assemble.hpp:85-104) ->
// execute (parloop.hpp:191-384) with a dof-expanded map and the
// linear-elasticity element kernel (restated in elements.cuh FormT<F_ELASTICITY>),
// Mat::addto (data.hpp:205-222) on the 3x3-blocked pattern of
// build_sparsity(map, map, 3, 3) (data.hpp:149-179).
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "linkwalk.cuh"
#include "ltile.cuh"
#include "stage.cuh"

namespace loam_gpu {

namespace {

inline int up16(int x) { return (x + 15) & ~15; }

constexpr int kNV = 4;            // P1 tet
#ifndef LOAM_GPU_LT_NT
#define LOAM_GPU_LT_NT 128
#endif
constexpr int kLtConsumers = LOAM_GPU_LT_NT; // consumer threads per CTA = blocks per tile at most

} // namespace

bool build_ltile(LtilePlan& out, const LtileSpec& sp, int ncells, int nnodes, const int32_t* sorted_rows,
                 const int32_t* sorted_x, int nverts, const PairPlan& pp, const int64_t* row_ptr, int64_t nnz,
                 cudaStream_t s) {
  if (pp.nrn != kNV || pp.ncn != kNV || nnz >= (int64_t(1) << 31) || ncells == 0) return false;
  constexpr int NT = kLtConsumers;
  const int64_t np = pp.npairs;
  // (sorted_x == sorted_rows: the coordinate map is the node map -- one download serves both)
  const bool same_x = sorted_x == sorted_rows;
  auto hrows = host_array<int32_t>((size_t)ncells * kNV), hx_own = host_array<int32_t>(same_x ? 0 : (size_t)ncells * kNV),
       hpairs = host_array<int32_t>(np), hp = host_array<int32_t>(nnodes + 1);
  auto hrank = host_array<uint8_t>((size_t)np * kNV);
  auto hrp = host_array<int64_t>((size_t)nnodes * 3 + 1);
  parallel_d2h({{hrows.data(), sorted_rows, sizeof(int32_t) * hrows.size()},
                {hx_own.data(), sorted_x, sizeof(int32_t) * hx_own.size()},
                {hpairs.data(), pp.pairs.get(), sizeof(int32_t) * (size_t)np},
                {hp.data(), pp.ptr.get(), sizeof(int32_t) * (size_t)(nnodes + 1)},
                {hrank.data(), pp.ranks.get(), hrank.size()},
                {hrp.data(), row_ptr, sizeof(int64_t) * hrp.size()}},
               s);
  const int32_t* hx = same_x ? hrows.data() : hx_own.data();
  plan_tick("ltile: D2H", s);
  std::vector<int64_t> nptr(nnodes + 1); // node-level pattern offsets of the 3x3-blocked CSR
  for (int i = 0; i <= nnodes; ++i) nptr[i] = hrp[(size_t)3 * i] / 9;
  struct TileChunk {
    bool ok = true;
    std::vector<int32_t> tiles, runs;
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
    } cstamp(ncells), vstamp(nverts);
    int gen = 0;
    std::vector<int> vid, seq, lcnt, lpos;
    std::vector<std::pair<int, int>> rr;
    std::vector<int> base;
    std::vector<uint32_t> flat; // a row's per-rank cell lists: cell << 4 | lv << 2 | lw
    struct Item {
      uint32_t A, B;
      int roff, nent;
    };
    std::vector<Item> items;
    std::vector<uint16_t> ring, dinfo;
    LinkWalk lw_;
    const int vend = (int)cb1;
    int v0 = (int)cb0;
    auto fail = [&] { O.ok = false; };
    while (v0 < vend) {
      // rows while their off-diagonal blocks fit one round of NT threads
      int v1 = v0, nit = 0;
      while (v1 < vend && v1 - v0 < sp.tile_nodes) {
        const int L = (int)(nptr[v1 + 1] - nptr[v1]);
        if (L < 1) return fail();
        if (nit + L - 1 > NT || 9 * (nptr[v1 + 1] - nptr[v0]) > 60000) break;
        nit += L - 1;
        ++v1;
      }
      if (v1 == v0) return fail();
      int slots = 0;
      auto window = [&](int a, int b) {
        ++gen;
        vid.clear();
        for (int p = hp[a]; p < hp[b]; ++p) {
          const int c = hpairs[p] / kNV;
          if (cstamp.p[c] == gen) continue;
          cstamp.p[c] = gen;
          for (int v = 0; v < kNV; ++v) {
            const int x = hx[(size_t)c * kNV + v];
            if (vstamp.p[x] != gen) {
              vstamp.p[x] = gen;
              vid.push_back(x);
            }
          }
        }
        slots = link_runs(vid, nverts, rr);
        return slots <= sp.tile_slots && (int)rr.size() <= sp.tile_runs;
      };
      while (!window(v0, v1)) {
        if (v1 == v0 + 1) return fail();
        --v1;
      }
      base.resize(rr.size());
      for (size_t q = 0, acc = 0; q < rr.size(); ++q) {
        base[q] = (int)acc;
        acc += rr[q].second - rr[q].first;
      }
      auto slot_in = [&](int v) {
        size_t q = std::upper_bound(rr.begin(), rr.end(), std::make_pair(v, INT32_MAX)) - rr.begin() - 1;
        return base[q] + v - rr[q].first;
      };
      items.clear();
      ring.clear();
      dinfo.clear();
      const int64_t S0 = nptr[v0];
      for (int v = v0; v < v1; ++v) {
        const int L = (int)(nptr[v + 1] - nptr[v]);
        lcnt.assign(L + 1, 0);
        int self = -1;
        for (int p = hp[v]; p < hp[v + 1]; ++p) {
          const int lv = hpairs[p] % kNV;
          for (int lw = 0; lw < kNV; ++lw) {
            const int r = hrank[(size_t)p * kNV + lw];
            if (r >= L) return fail();
            if (lw == lv) {
              if (self >= 0 && self != r) return fail();
              self = r;
            } else ++lcnt[r + 1];
          }
        }
        if (self < 0) return fail();
        for (int r = 0; r < L; ++r) lcnt[r + 1] += lcnt[r];
        lpos.assign(lcnt.begin(), lcnt.end() - 1);
        flat.resize(lcnt[L]);
        for (int p = hp[v]; p < hp[v + 1]; ++p) {
          const int c = hpairs[p] / kNV, lv = hpairs[p] % kNV;
          for (int lw = 0; lw < kNV; ++lw)
            if (lw != lv) flat[lpos[hrank[(size_t)p * kNV + lw]]++] = (uint32_t)c << 4 | (uint32_t)lv << 2 | (uint32_t)lw;
        }
        const uint32_t rowb = (uint32_t)(9 * (nptr[v] - S0)), stride = (uint32_t)(3 * L);
        for (int r = 0; r < L; ++r) {
          if (r == self) {
            if (lcnt[r + 1] != lcnt[r]) return fail();
            continue;
          }
          const int nc = lcnt[r + 1] - lcnt[r];
          // every pattern block is reached by a cell (exact (map, map) pattern), by few enough cells
          if (nc < 1 || nc + 1 > sp.max_link || nc + 1 > LinkWalk::kMax) return fail();
          lw_.nn = 0;
          int xv = -1, xw = -1;
          for (int q = lcnt[r]; q < lcnt[r + 1]; ++q) {
            const uint32_t f = flat[q];
            const int c = (int)(f >> 4), lv = (f >> 2) & 3, lw = f & 3;
            int o[2], no = 0;
            for (int j = 0; j < kNV; ++j)
              if (j != lv && j != lw) o[no++] = j;
            const size_t cb = (size_t)c * kNV;
            const int cxv = hx[cb + lv], cxw = hx[cb + lw];
            if (xv < 0) {
              xv = cxv;
              xw = cxw;
            } else if (xv != cxv || xw != cxw) return fail(); // node and coordinate maps disagree
            if (!lw_.add(hrows[cb + o[0]], hx[cb + o[0]], hrows[cb + o[1]], hx[cb + o[1]])) return fail();
          }
          if (!lw_.walk(nc, seq)) return fail();
          Item it;
          it.A = (rowb + 3u * (uint32_t)r) | stride << 16;
          it.B = (uint32_t)slot_in(xv) | (uint32_t)slot_in(xw) << 16;
          it.roff = (int)ring.size();
          it.nent = (int)seq.size();
          for (int x : seq) ring.push_back((uint16_t)slot_in(x));
          items.push_back(it);
        }
        dinfo.insert(dinfo.end(), {(uint16_t)rowb, (uint16_t)L, (uint16_t)self, 0});
      }
      if ((int)items.size() > NT) return fail();
      // blocks of equal link lengths share warps (a warp's loop runs to its longest link)
      std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) { return x.nent > y.nent; });
      const int nitems = (int)items.size(), nv = v1 - v0, maxent = nitems ? items[0].nent : 0;
      const int off_ring = 9 * NT, off_d = off_ring + up16(maxent * NT * 2), bytes = off_d + up16(nv * 8);
      const size_t b0 = O.blob.size();
      O.blob.resize(b0 + bytes, 0);
      uint8_t* bp = O.blob.data() + b0;
      for (int i = 0; i < nitems; ++i) {
        memcpy(bp + 4 * i, &items[i].A, 4);
        memcpy(bp + 4 * NT + 4 * i, &items[i].B, 4);
        bp[8 * NT + i] = (uint8_t)items[i].nent;
        for (int q = 0; q < items[i].nent; ++q) memcpy(bp + off_ring + 2 * (q * NT + i), &ring[items[i].roff + q], 2);
      }
      memcpy(bp + off_d, dinfo.data(), (size_t)nv * 8);
      const int seg = (int)(9 * (nptr[v1] - nptr[v0]));
      O.tiles.insert(O.tiles.end(), {(int)(b0 / 16), bytes, v0, nv, (int)(9 * nptr[v0]), seg, nitems, maxent,
                                     (int)O.runs.size() / 2, (int)rr.size(), off_ring, off_d, slots, 0, 0, 0});
      for (auto& x : rr) O.runs.insert(O.runs.end(), {x.first, x.second});
      O.max_seg = std::max(O.max_seg, seg);
      O.max_slots = std::max(O.max_slots, slots);
      O.max_blob = std::max(O.max_blob, bytes);
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
    out.max_slots = std::max(out.max_slots, O.max_slots);
    out.max_blob = std::max(out.max_blob, O.max_blob);
  }
  if (bytes_so_far / 16 >= (size_t)INT32_MAX) return false;
  plan_tick("ltile: tiles", s);
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

struct LtileArgs {
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
};

__device__ __forceinline__ void lt_wait(uint64_t* bar, uint32_t parity) {
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

#ifndef LOAM_GPU_LT_MINB
#define LOAM_GPU_LT_MINB 4
#endif

// NT consumer threads (one per off-diagonal 3x3 block of the tile) + one TMA producer warp.
template <int STAGES>
__global__ void __launch_bounds__(kLtConsumers + 32, LOAM_GPU_LT_MINB) k_ltile(const __grid_constant__ LtileArgs a) {
  constexpr int NT = kLtConsumers;
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
    int4 nm[3];
    int2 nrun = make_int2(0, 0);
    auto prefetch = [&]() {
      if (nt < a.ntiles) {
        const int4* t = reinterpret_cast<const int4*>(a.tiles + 16 * nt);
#pragma unroll
        for (int q = 0; q < 3; ++q) nm[q] = __ldg(t + q);
        nrun = first_run(reinterpret_cast<const int2*>(a.runs) + nm[2].x, nm[2].y, lane);
      }
    };
    prefetch();
    grid_dep_wait(); // the caller's data only after the previous kernel (PDL)
    for (int k = 0;; ++k) {
      const int tile = nt;
      const int4 m0 = nm[0], m1 = nm[1], m2 = nm[2];
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
  const double lam = a.prm.p[0], mu = a.prm.p[1];
  for (int k = 0;; ++k) {
    lt_wait(&full[k % STAGES], (k / STAGES) & 1);
    const int tile = slot_tile[k % STAGES];
    if (tile < 0) break;
    const int4* sm4 = slot_meta + 4 * (k % STAGES);
    const int4 m0 = sm4[0], m1 = sm4[1], m2 = sm4[2];
    const int nv = m0.w, E0 = m1.x, len = m1.y, nitems = m1.z, off_ring = m2.z, off_d = m2.w;
    const unsigned char* buf = ring(k);
    const uint32_t* recA = reinterpret_cast<const uint32_t*>(buf);
    const uint32_t* recB = recA + NT;
    const uint8_t* nent = buf + 8 * NT;
    const uint16_t* lnk = reinterpret_cast<const uint16_t*>(buf + off_ring);
    const uint16_t* dinfo = reinterpret_cast<const uint16_t*>(buf + off_d);
    const double* win = reinterpret_cast<const double*>(buf + a.b_win);
    double* seg = seg0 + (E0 & 1); // 16-byte parity of the global destination (bulk store)
    // one thread per off-diagonal block: walk the link of its edge
    double S[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    uint32_t A = 0;
    if (tid < nitems) {
      A = recA[tid];
      const uint32_t B = recB[tid];
      const int ne = nent[tid];
      const double* pv = win + 3 * (B & 0xffffu);
      const double* pw = win + 3 * (B >> 16);
      const double xv[3] = {pv[0], pv[1], pv[2]};
      const double e[3] = {pw[0] - xv[0], pw[1] - xv[1], pw[2] - xv[2]};
      double a0[3], c0[3]; // p - v and (p - v) x e of the previous link vertex
      auto vertex = [&](int slot, double (&aa)[3], double (&cc)[3]) {
        const double* p = win + 3 * slot;
        aa[0] = p[0] - xv[0];
        aa[1] = p[1] - xv[1];
        aa[2] = p[2] - xv[2];
        cc[0] = aa[1] * e[2] - aa[2] * e[1];
        cc[1] = aa[2] * e[0] - aa[0] * e[2];
        cc[2] = aa[0] * e[1] - aa[1] * e[0];
      };
      vertex(lnk[tid], a0, c0);
      int nslot = ne > 1 ? lnk[NT + tid] : 0;
      for (int i = 1; i < ne; ++i) {
        double a1[3], c1[3];
        vertex(nslot, a1, c1);
        if (i + 1 < ne) nslot = lnk[(i + 1) * NT + tid];
        // cell (v, w, p, q): n = (p - v) x (q - v), D = e . n = 6 V (signed),
        // m = (q - w) x (p - w) = c_p - c_q - n; V g_v g_w^T = m n^T / (6 |D|)
        double n[3];
        n[0] = a0[1] * a1[2] - a0[2] * a1[1];
        n[1] = a0[2] * a1[0] - a0[0] * a1[2];
        n[2] = a0[0] * a1[1] - a0[1] * a1[0];
        const double D = fma(e[0], n[0], fma(e[1], n[1], e[2] * n[2]));
        const double r = fast_rcp(6.0 * fabs(D));
        double tm[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) tm[d] = r * (c0[d] - c1[d] - n[d]);
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int f = 0; f < 3; ++f) S[d][f] = fma(tm[d], n[f], S[d][f]);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          a0[d] = a1[d];
          c0[d] = c1[d];
        }
      }
    }
    if (tid == 0) bulk_wait_read<0>(); // the previous tile's store has read the segment
    named_bar(1, NT);
    if (tid < nitems) {
      // the element block of FormT<F_ELASTICITY>::row is linear in S: A_de = mu S_ed + lam S_de + d_de mu tr(S)
      const int wb = A & 0xffffu, ws = A >> 16;
      const double tr = mu * (S[0][0] + S[1][1] + S[2][2]);
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          double v = fma(mu, S[f][d], lam * S[d][f]);
          if (d == f) v += tr;
          seg[wb + d * ws + f] = v;
        }
    }
    named_bar(1, NT);
    // diagonal blocks: minus the row's off-diagonal blocks, in column order
    // (the gradients of a cell sum to zero, so every block row sums to zero)
    for (int t = tid; t < 9 * nv; t += NT) {
      const int vi = t / 9, de = t - 9 * vi, d = de / 3, f = de - 3 * d;
      const int rowb = dinfo[4 * vi], L = dinfo[4 * vi + 1], self = dinfo[4 * vi + 2];
      const double* row = seg + rowb + d * 3 * L + f;
      double sum = 0.0;
      for (int r = 0; r < L; ++r)
        if (r != self) sum += row[3 * r];
      seg[rowb + d * 3 * L + 3 * self + f] = -sum;
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[k % STAGES]); // the stage's records and window are read
    if (a.accumulate) {
      named_bar(1, NT);
      for (int t = tid; t < len; t += NT) a.out[(int64_t)E0 + t] += seg[t];
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

void launch_ltile(const LtilePlan& p, const double* coords, double* out, const FormParams& prm, bool accumulate,
                  int* next_tile, int* reset_tile, cudaStream_t s) {
  if (p.ntiles == 0) return;
  LtileArgs a{};
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
  static const int st = std::getenv("LOAM_GPU_LT_STAGES") ? std::atoi(std::getenv("LOAM_GPU_LT_STAGES")) : 2;
  auto go = [&](auto kern, int stages) {
    const size_t smem = (size_t)off + stages * (size_t)a.buf_bytes;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int blocks = 1;
    LG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, kLtConsumers + 32, smem));
    require(blocks > 0, LOAM_GPU_ERR_CUDA, "link-tile kernel does not fit on an SM");
    if (std::getenv("LOAM_GPU_LT_INFO")) // developer: plan maxima behind the shared-memory footprint
      fprintf(stderr, "ltile: tiles %d max_seg %d max_blob %d max_slots %d smem %zu CTAs/SM %d\n", p.ntiles, p.max_seg,
              p.max_blob, p.max_slots, smem, blocks);
    launch_pdl(kern, dim3(std::min(p.ntiles, blocks * kNumSMs)), dim3(kLtConsumers + 32), smem, s, a);
  };
  if (st >= 3) go(k_ltile<3>, 3);
  else if (st == 2) go(k_ltile<2>, 2);
  else go(k_ltile<1>, 1);
  count_launch();
  LG_LAUNCH_CHECK();
}

} // namespace loam_gpu
