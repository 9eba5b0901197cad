// stage.cuh -- warp-cooperative TMA staging of id-run windows (sm_100a).
//
// A tile's vertex (or coefficient) window is the union of a few contiguous id
// runs of an AoS fp64 array; the producer warp copies every run into
// consecutive shared-memory slots with cp.async.bulk (async.cuh).
#pragma once
#include <cstdint>

#include "async.cuh"

namespace loam_gpu {

__device__ __forceinline__ int skew_of(int lo, int es) { return ((lo * es) & 15) / es; }

// Warp-cooperative staging of a tile's id runs [lo, hi) of an es-doubles-per-id
// array into consecutive window slots: lane r handles run r (32 at a time),
// slots from a warp scan.  A run whose byte count is not a multiple of 16 gets
// its last double stored by the lane itself (bulk copies move 16-byte units;
// runs start at even ids so the source side is aligned).  prepare() does the
// tail stores and returns the warp-total bulk bytes; issue() launches copies.
struct RunSet {
  const int2* runs;
  int cnt;
  const double* src;
  double* dst;
  int es;
};
// `first`: the lane's run of the first chunk, prefetched by the caller.
__device__ __forceinline__ int2 first_run(const int2* runs, int cnt, int lane) {
  return lane < cnt ? __ldg(runs + lane) : make_int2(0, 0);
}
template <bool ISSUE>
__device__ __forceinline__ uint32_t stage_runs(const RunSet& s, int lane, uint64_t* bar, int2 first) {
  uint32_t tx = 0;
  int base = 0;
  for (int r0 = 0; r0 < s.cnt; r0 += 32) {
    int lo = first.x, hi = first.y;
    if (r0 > 0) {
      const int2 p = r0 + lane < s.cnt ? __ldg(s.runs + r0 + lane) : make_int2(0, 0);
      lo = p.x;
      hi = p.y;
    }
    const int n = hi - lo;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int slot = base + incl - n;
    const uint32_t nb = (uint32_t)n * s.es * 8;
    if (ISSUE) {
      if (nb >= 16) bulk_g2s(s.dst + (int64_t)slot * s.es, s.src + (int64_t)lo * s.es, nb & ~15u, bar);
    } else {
      if (nb & 15) s.dst[(int64_t)(slot + n) * s.es - 1] = s.src[(int64_t)hi * s.es - 1];
      tx += nb & ~15u;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (!ISSUE)
#pragma unroll
    for (int o = 16; o; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
  return tx;
}

// Static tile schedule with prefetched tile records (RI ints each, RI % 4 ==
// 0).  Tile k of a CTA is blockIdx + k * grid; the producer warp pulls the
// records of 8 tiles at a time into shared memory by cp.async (one 16-byte
// part per lane), one batch ahead in a double buffer, so its per-tile chain
// holds no dependent global round trip for the tile's meta (a dynamic counter
// costs an atomic plus a record load per tile).  For tiles of uniform cost.
// buf: shared int[2][8 * RI], 16-byte aligned.  Per tile: rec = at(k), read
// it into registers, then done(k).
template <int RI>
struct TileFeedT {
  static_assert(RI % 4 == 0 && RI <= 16, "record of whole 16-byte parts, one per lane");
  static constexpr int kParts = RI / 4;
  int* buf;
  const int32_t* tiles;
  int ntiles;
  __device__ __forceinline__ int tile(int k) const { return (int)blockIdx.x + k * (int)gridDim.x; }
  __device__ __forceinline__ void load(int b, int lane) const { // tiles 8b..8b+7 -> buf[b & 1]
    const int q = lane / kParts, part = lane - q * kParts;
    const int t = tile(8 * b + q);
    if (q < 8 && t < ntiles) cp_async16(buf + (b & 1) * 8 * RI + q * RI + part * 4, tiles + (int64_t)RI * t + part * 4);
    cp_async_commit();
  }
  __device__ __forceinline__ void start(int lane) const {
    load(0, lane);
    load(1, lane);
  }
  __device__ __forceinline__ const int* at(int k) const {
    if (k % 8 == 0) {
      cp_async_wait<1>(); // batch k / 8 has landed
      __syncwarp();
    }
    return buf + ((k / 8) & 1) * 8 * RI + (k % 8) * RI;
  }
  __device__ __forceinline__ void done(int k, int lane) const {
    if (k % 8 == 7) {
      __syncwarp();
      load(k / 8 + 2, lane);
    }
  }
  __device__ __forceinline__ void drain() const { cp_async_wait<0>(); }
};

// Persistent tile kernels grab tiles from a global counter.  The last CTA to
// finish puts the counter (and the exit count) back to zero, so every launch
// -- including a replay of a captured CUDA graph with frozen arguments --
// starts from tile 0.  Called by all `nconsumers` consumer threads after their
// last tile (the producer warp has grabbed its last tile before the consumers
// see the end marker).
__device__ __forceinline__ void tile_counter_release(int* next_tile, int* done, int nconsumers, int tid) {
  named_bar(1, nconsumers);
  if (tid == 0 && atomicAdd(done, 1) == (int)gridDim.x - 1) { // the launch boundary orders these for the next launch
    *next_tile = 0;
    *done = 0;
  }
}

} // namespace loam_gpu
