// capi.cu -- extern "C" boundary (include/loam_gpu.h) over the engine.
//
// Error convention: loam::Error (common.hpp:36-49) -> int code 1 + ErrorKind
// with a thread-local message; CUDA failures -> LOAM_GPU_ERR_CUDA.  No CPU
// fallback: compute entry points fail with LOAM_GPU_ERR_NO_DEVICE when no
// sm_100 device is usable.
#include <atomic>
#include <map>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"
#include "plan.cuh"
#include "solver.cuh"
#include "fem.cuh"
#include "mesh.cuh"

using namespace loam_gpu;

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_msg.clear();
    return 0;
  } catch (const Error& e) {
    g_msg = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_msg = e.what();
    return LOAM_ERR(InvalidArgument);
  }
}

bool device_ok() {
  static const bool ok = [] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return false;
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major == 10) {
      // plan and staging buffers come from the stream-ordered pool: keep freed
      // blocks cached instead of returning them to the driver at every
      // synchronisation (the host calling convention synchronises per call)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
    }
    return major == 10;
  }();
  return ok;
}

void require_device() {
  require(device_ok(), LOAM_GPU_ERR_NO_DEVICE,
          "no usable sm_100 (B200) device: the loam_gpu engine has no CPU fallback");
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Device copies of the immutable objects of the host calling convention.  In
// the reference a Map is a shared_ptr<const Map> (topology.hpp:68) and a
// Sparsity is never modified after build_sparsity (data.hpp:116-179), so an
// object id names its content: execute_host uploads a Map / Sparsity once per
// (id, host pointer, size) and keeps it resident, like the C++ facade's
// Map/Sparsity objects do.  Dats (mutable, data.hpp:49-52) are copied every
// call.  loam_gpu_plan_cache_clear() drops these copies too.
struct Resident {
  const void* host = nullptr;
  size_t bytes = 0;
  void* dev = nullptr;
};
std::mutex g_res_mutex;
std::map<std::pair<int, uint64_t>, Resident> g_resident;

void* resident_copy(int kind, uint64_t id, const void* host, size_t bytes, cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_res_mutex);
  Resident& r = g_resident[{kind, id}];
  if (r.dev && r.host == host && r.bytes == bytes) return r.dev;
  if (r.dev) {
    LG_CUDA(cudaStreamSynchronize(s));
    LG_CUDA(cudaFree(r.dev));
    r.dev = nullptr;
  }
  LG_CUDA(cudaMalloc(&r.dev, bytes ? bytes : 1));
  if (bytes) LG_CUDA(cudaMemcpyAsync(r.dev, host, bytes, cudaMemcpyHostToDevice, s));
  r.host = host;
  r.bytes = bytes;
  return r.dev;
}

void resident_release(uint64_t id) {
  std::lock_guard<std::mutex> g(g_res_mutex);
  for (auto it = g_resident.begin(); it != g_resident.end();) {
    if (it->first.second == id) {
      if (it->second.dev) {
        cudaDeviceSynchronize(); // a queued call may still read it
        cudaFree(it->second.dev);
      }
      it = g_resident.erase(it);
    } else {
      ++it;
    }
  }
}

void resident_clear() {
  std::lock_guard<std::mutex> g(g_res_mutex);
  for (auto& [k, r] : g_resident)
    if (r.dev) cudaFree(r.dev);
  g_resident.clear();
}

} // namespace

extern "C" {

const char* loam_gpu_last_error(void) { return g_msg.c_str(); }
const char* loam_gpu_version(void) { return "loam_gpu 0.1 (sm_100a)"; }
int loam_gpu_device_ok(void) { return device_ok() ? 1 : 0; }

int loam_gpu_set_option(int option, int value) {
  return guarded([&] {
    switch (option) {
    case LOAM_OPT_INC_STRATEGY:
      require(value >= 0 && value <= 6, LOAM_ERR(InvalidArgument), "strategy must be 0..6");
      options().inc_strategy = value;
      break;
    case LOAM_OPT_CHECK_SPARSITY: options().check_sparsity = value ? 1 : 0; break;
    case LOAM_OPT_LOCALITY: options().locality = value ? 1 : 0; break;
    case LOAM_OPT_TEST_KERNELS: options().test_kernels = value ? 1 : 0; break;
    case LOAM_OPT_DETERMINISTIC:
      if (options().deterministic != (value ? 1 : 0)) plan_cache_clear(); // plans depend on it
      options().deterministic = value ? 1 : 0;
      break;
    default: fail(LOAM_ERR(InvalidArgument), "unknown option");
    }
  });
}

int loam_gpu_get_option(int option) {
  switch (option) {
  case LOAM_OPT_INC_STRATEGY: return options().inc_strategy;
  case LOAM_OPT_CHECK_SPARSITY: return options().check_sparsity;
  case LOAM_OPT_LOCALITY: return options().locality;
  case LOAM_OPT_TEST_KERNELS: return options().test_kernels;
  case LOAM_OPT_DETERMINISTIC: return options().deterministic;
  default: return -1;
  }
}

int loam_gpu_plan_cache_clear(void) {
  return guarded([] {
    plan_cache_clear();
    resident_clear();
  });
}

uint64_t loam_gpu_new_id(void) {
  static std::atomic<uint64_t> next{1};
  return next++;
}

int loam_gpu_release_id(uint64_t id) {
  if (id == 0) return 0;
  return guarded([&] {
    plan_cache_release(id);
    resident_release(id);
  });
}

int64_t loam_gpu_launch_count(void) { return g_launches.load(); }

int loam_gpu_kernel_signature(const char* name, int32_t* buf, int cap) {
  const KernelInfo* k = name ? find_kernel(name) : nullptr;
  if (!k) {
    g_msg = std::string("kernel ") + (name ? name : "(null)") + " is not registered";
    return -LOAM_ERR(InvalidArgument);
  }
  int w = 0;
  for (const auto& ext : k->extents) {
    if (w < cap) buf[w] = (int32_t)ext.size();
    ++w;
    for (int x : ext) {
      if (w < cap) buf[w] = x;
      ++w;
    }
  }
  return (int)k->extents.size();
}

const char* loam_gpu_kernel_names(void) { return kernel_names().c_str(); }

int loam_gpu_validate(const loam_kernel_desc* kernel, int32_t n, uint64_t iter, const loam_arg_desc* args,
                      int nargs) {
  return guarded([&] { validate(kernel, n, iter, args, nargs); });
}

int loam_gpu_execute(const loam_kernel_desc* kernel, int32_t n, uint64_t iter, const loam_arg_desc* args,
                     int nargs, void* stream) {
  return guarded([&] {
    require_device();
    execute(kernel, n, iter, args, nargs, as_stream(stream));
  });
}

int loam_gpu_execute_blocks(const loam_loop_desc* loops, int nloops, void* stream) {
  return guarded([&] {
    require_device();
    std::vector<LoopDesc> l((size_t)std::max(nloops, 0));
    for (int i = 0; i < nloops; ++i)
      l[i] = LoopDesc{loops[i].kernel, loops[i].iterset_size, loops[i].iterset_id, loops[i].args, loops[i].nargs};
    execute_blocks(l.data(), nloops, as_stream(stream));
  });
}

// Host-memory calling convention of the reference: every pointer is host
// memory.  Uploads maps, patterns and the data the loop reads, runs, downloads
// every written object, and returns with the results visible on the host.
namespace {
// The loops of one host-convention call: every loop validated first (nothing
// is copied for an illegal loop), one device copy per host array across the
// loops, the loops run (one loop: execute; several: execute_blocks), every
// written object downloaded.
void run_host_loops(const loam_loop_desc* loops, int nloops, cudaStream_t s) {
  for (int l = 0; l < nloops; ++l)
    validate(loops[l].kernel, loops[l].iterset_size, loops[l].iterset_id, loops[l].args, loops[l].nargs);
  std::vector<DevBuf<char>> bufs;
  std::vector<std::pair<const void*, void*>> uploaded; // one copy per host array
  auto up = [&](const void* host, size_t bytes) -> void* {
    for (auto& [h, d] : uploaded)
      if (h == host) return d;
    bufs.emplace_back(bytes ? bytes : 1, s);
    if (bytes) LG_CUDA(cudaMemcpyAsync(bufs.back().get(), host, bytes, cudaMemcpyHostToDevice, s));
    uploaded.emplace_back(host, bufs.back().get());
    return bufs.back().get();
  };
  // immutable objects with an id stay resident; anonymous ones (id 0) are copied per call
  auto keep = [&](int kind, uint64_t id, const void* host, size_t bytes) -> void* {
    return id ? resident_copy(kind, id, host, bytes, s) : up(host, bytes);
  };
  auto map_up = [&](const loam_map_desc* m, loam_map_desc& d) {
    d = *m;
    d.values = static_cast<const int32_t*>(
        keep(0, m->id, m->values, sizeof(int32_t) * (size_t)m->source_size * m->arity));
    if (m->expand_dim > 1 && m->node_values)
      d.node_values = static_cast<const int32_t*>(
          keep(1, m->id, m->node_values, sizeof(int32_t) * (size_t)m->source_size * m->node_arity));
  };
  struct DevLoop {
    std::vector<loam_arg_desc> dargs;
    std::vector<loam_map_desc> dmaps;
    std::vector<loam_sparsity_desc> dsp;
  };
  std::vector<DevLoop> dl((size_t)nloops);
  std::vector<std::pair<const void*, void*>> written; // host object -> its device copy (one per object)
  for (int l = 0; l < nloops; ++l) {
    const loam_arg_desc* args = loops[l].args;
    const int nargs = loops[l].nargs;
    DevLoop& D = dl[l];
    D.dargs.assign(args, args + nargs);
    D.dmaps.resize(2 * (size_t)nargs);
    D.dsp.resize((size_t)nargs);
    for (int q = 0; q < nargs; ++q) {
      const loam_arg_desc& a = args[q];
      loam_arg_desc& d = D.dargs[q];
      if (a.map) { map_up(a.map, D.dmaps[2 * q]); d.map = &D.dmaps[2 * q]; }
      if (a.col_map) { map_up(a.col_map, D.dmaps[2 * q + 1]); d.col_map = &D.dmaps[2 * q + 1]; }
      size_t count;
      if (a.kind == LOAM_ARG_MAT) {
        const loam_sparsity_desc* sp = a.sparsity;
        D.dsp[q] = *sp;
        D.dsp[q].row_ptr = static_cast<const int64_t*>(
            keep(2, sp->id, sp->row_ptr, sizeof(int64_t) * ((size_t)sp->nrows + 1)));
        D.dsp[q].col_idx = static_cast<const int32_t*>(keep(3, sp->id, sp->col_idx, sizeof(int32_t) * (size_t)sp->nnz));
        d.sparsity = &D.dsp[q];
        count = (size_t)sp->nnz;
      } else if (a.kind == LOAM_ARG_DAT) {
        count = (size_t)a.set_size * a.dim;
      } else {
        count = (size_t)a.dim;
      }
      const bool needs_old = a.access == LOAM_READ || a.access == LOAM_RW ||
                             (a.access == LOAM_INC && !(a.flags & LOAM_ARG_ZERO)) ||
                             (a.kind != LOAM_ARG_DAT && a.access == LOAM_WRITE);
      void* prior = nullptr; // an object an earlier loop of the call wrote: keep working on that copy
      for (auto& [h, dv] : written)
        if (h == a.data) prior = dv;
      if (prior) {
        d.data = static_cast<double*>(prior);
        if (!needs_old) d.flags &= ~LOAM_ARG_ZERO;
      } else if (needs_old) {
        d.data = static_cast<double*>(up(a.data, sizeof(double) * count));
      } else {
        bufs.emplace_back(count ? sizeof(double) * count : 1, s);
        d.data = reinterpret_cast<double*>(bufs.back().get());
        if (a.kind == LOAM_ARG_DAT && a.access == LOAM_WRITE && a.map) {
          // indirect WRITE leaves untouched entries as they were (test_parloop.cpp:182-200)
          LG_CUDA(cudaMemcpyAsync(d.data, a.data, sizeof(double) * count, cudaMemcpyHostToDevice, s));
        }
      }
      if (a.access != LOAM_READ && !prior) written.emplace_back(a.data, d.data);
    }
  }
  if (nloops == 1) {
    execute(loops[0].kernel, loops[0].iterset_size, loops[0].iterset_id, dl[0].dargs.data(), loops[0].nargs, s);
  } else {
    std::vector<LoopDesc> ld((size_t)nloops);
    for (int l = 0; l < nloops; ++l)
      ld[l] = LoopDesc{loops[l].kernel, loops[l].iterset_size, loops[l].iterset_id, dl[l].dargs.data(), loops[l].nargs};
    execute_blocks(ld.data(), nloops, s);
  }
  for (int l = 0; l < nloops; ++l)
    for (int q = 0; q < loops[l].nargs; ++q) {
      const loam_arg_desc& a = loops[l].args[q];
      if (a.access == LOAM_READ) continue;
      const size_t count = a.kind == LOAM_ARG_MAT ? (size_t)a.sparsity->nnz
                           : a.kind == LOAM_ARG_DAT ? (size_t)a.set_size * a.dim : (size_t)a.dim;
      if (count)
        LG_CUDA(cudaMemcpyAsync(a.data, dl[l].dargs[q].data, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    }
  LG_CUDA(cudaStreamSynchronize(s));
}
} // namespace

int loam_gpu_execute_host(const loam_kernel_desc* kernel, int32_t n, uint64_t iter,
                          const loam_arg_desc* args, int nargs, void* stream) {
  return guarded([&] {
    require_device();
    const loam_loop_desc one{kernel, n, iter, args, nargs};
    run_host_loops(&one, 1, as_stream(stream));
  });
}

// fem::assemble_blocks (fem/assemble.hpp:439-448) under the host-memory
// calling convention: the loops of loam_gpu_execute_blocks over host data.
int loam_gpu_execute_blocks_host(const loam_loop_desc* loops, int nloops, void* stream) {
  return guarded([&] {
    require_device();
    require(nloops >= 0 && (nloops == 0 || loops != nullptr), LOAM_ERR(InvalidArgument), "block loops without a list");
    if (nloops == 0) return;
    run_host_loops(loops, nloops, as_stream(stream));
  });
}

namespace {
// Copy engines of the batched host calling convention (created once).
struct CopyStreams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  CopyStreams() {
    LG_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    LG_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
  }
};
CopyStreams& copy_streams() {
  static CopyStreams c;
  return c;
}
size_t arg_count(const loam_arg_desc& a) {
  return a.kind == LOAM_ARG_MAT ? (size_t)a.sparsity->nnz
         : a.kind == LOAM_ARG_DAT ? (size_t)a.set_size * a.dim : (size_t)a.dim;
}
bool arg_needs_old(const loam_arg_desc& a) {
  return a.access == LOAM_READ || a.access == LOAM_RW || (a.access == LOAM_INC && !(a.flags & LOAM_ARG_ZERO)) ||
         (a.access == LOAM_WRITE && (a.kind != LOAM_ARG_DAT || a.map));
}
} // namespace

int loam_gpu_execute_host_batch(const loam_kernel_desc* kernel, int32_t n, uint64_t iter,
                                const loam_arg_desc* const* args, int nargs, int nsteps, void* stream) {
  return guarded([&] {
    require_device();
    require(nsteps >= 0 && (nsteps == 0 || args != nullptr), LOAM_ERR(InvalidArgument), "batch without steps");
    for (int k = 0; k < nsteps; ++k) validate(kernel, n, iter, args[k], nargs); // nothing copied if illegal
    if (nsteps == 0) return;
    cudaStream_t s = as_stream(stream);
    CopyStreams& cs = copy_streams();
    // device copies of the immutable objects (resident by id, as execute_host)
    const loam_arg_desc* a0 = args[0];
    std::vector<loam_map_desc> dmaps(2 * nargs);
    std::vector<loam_sparsity_desc> dsp(nargs);
    auto keep = [&](int kind, uint64_t id, const void* host, size_t bytes) -> void* {
      require(id != 0, LOAM_ERR(InvalidArgument), "batched host execution needs id'd maps and sparsities");
      return resident_copy(kind, id, host, bytes, s);
    };
    auto map_up = [&](const loam_map_desc* m, loam_map_desc& d) {
      d = *m;
      d.values = static_cast<const int32_t*>(
          keep(0, m->id, m->values, sizeof(int32_t) * (size_t)m->source_size * m->arity));
      if (m->expand_dim > 1 && m->node_values)
        d.node_values = static_cast<const int32_t*>(
            keep(1, m->id, m->node_values, sizeof(int32_t) * (size_t)m->source_size * m->node_arity));
    };
    for (int q = 0; q < nargs; ++q) {
      const loam_arg_desc& a = a0[q];
      if (a.map) map_up(a.map, dmaps[2 * q]);
      if (a.col_map) map_up(a.col_map, dmaps[2 * q + 1]);
      if (a.kind == LOAM_ARG_MAT) {
        dsp[q] = *a.sparsity;
        dsp[q].row_ptr = static_cast<const int64_t*>(
            keep(2, a.sparsity->id, a.sparsity->row_ptr, sizeof(int64_t) * ((size_t)a.sparsity->nrows + 1)));
        dsp[q].col_idx = static_cast<const int32_t*>(
            keep(3, a.sparsity->id, a.sparsity->col_idx, sizeof(int32_t) * (size_t)a.sparsity->nnz));
      }
    }
    for (int k = 1; k < nsteps; ++k) // one loop shape: the same objects in every step
      for (int q = 0; q < nargs; ++q)
        require(args[k][q].kind == a0[q].kind && args[k][q].access == a0[q].access &&
                    (!a0[q].map || (args[k][q].map && args[k][q].map->id == a0[q].map->id)) &&
                    (a0[q].kind != LOAM_ARG_MAT || args[k][q].sparsity->id == a0[q].sparsity->id) &&
                    arg_count(args[k][q]) == arg_count(a0[q]),
                LOAM_ERR(InvalidArgument), "batched steps must share the loop shape");
    // two device buffer sets; a set is reused once its previous step's downloads finished
    std::vector<DevBuf<double>> bufs[2];
    // Declared after the buffers, so destroyed first -- on success AND when a
    // step throws: both copy streams and `s` are drained before the buffers
    // are freed (stream-ordered on s) and before the caller's host buffers
    // are released, then the events are destroyed.
    struct Guard {
      CopyStreams& cs;
      cudaStream_t s;
      cudaEvent_t ev[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
      ~Guard() {
        cudaStreamSynchronize(cs.h2d);
        cudaStreamSynchronize(cs.d2h);
        cudaStreamSynchronize(s);
        for (auto& row : ev)
          for (auto& e : row)
            if (e) cudaEventDestroy(e);
      }
    } guard{cs, s};
    cudaEvent_t* in_ready = guard.ev[0];
    cudaEvent_t* done = guard.ev[1];
    cudaEvent_t* freed = guard.ev[2];
    for (int b = 0; b < 2; ++b) {
      for (int q = 0; q < nargs; ++q) bufs[b].emplace_back(std::max<size_t>(arg_count(a0[q]), 1), s);
      LG_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
      LG_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
      LG_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    }
    LG_CUDA(cudaEventRecord(freed[0], s)); // buffers allocated on s
    LG_CUDA(cudaEventRecord(freed[1], s));
    std::vector<loam_arg_desc> dargs(nargs);
    for (int k = 0; k < nsteps; ++k) {
      const int b = k & 1;
      const loam_arg_desc* a = args[k];
      LG_CUDA(cudaStreamWaitEvent(cs.h2d, freed[b], 0));
      for (int q = 0; q < nargs; ++q)
        if (arg_needs_old(a[q]) && arg_count(a[q]))
          LG_CUDA(cudaMemcpyAsync(bufs[b][q].get(), a[q].data, sizeof(double) * arg_count(a[q]),
                                  cudaMemcpyHostToDevice, cs.h2d));
      LG_CUDA(cudaEventRecord(in_ready[b], cs.h2d));
      LG_CUDA(cudaStreamWaitEvent(s, in_ready[b], 0));
      for (int q = 0; q < nargs; ++q) {
        dargs[q] = a[q];
        dargs[q].data = bufs[b][q].get();
        if (a[q].map) dargs[q].map = &dmaps[2 * q];
        if (a[q].col_map) dargs[q].col_map = &dmaps[2 * q + 1];
        if (a[q].kind == LOAM_ARG_MAT) dargs[q].sparsity = &dsp[q];
      }
      execute(kernel, n, iter, dargs.data(), nargs, s);
      LG_CUDA(cudaEventRecord(done[b], s));
      LG_CUDA(cudaStreamWaitEvent(cs.d2h, done[b], 0));
      for (int q = 0; q < nargs; ++q)
        if (a[q].access != LOAM_READ && arg_count(a[q]))
          LG_CUDA(cudaMemcpyAsync(a[q].data, bufs[b][q].get(), sizeof(double) * arg_count(a[q]),
                                  cudaMemcpyDeviceToHost, cs.d2h));
      LG_CUDA(cudaEventRecord(freed[b], cs.d2h));
    }
    LG_CUDA(cudaStreamSynchronize(cs.d2h));
    LG_CUDA(cudaStreamSynchronize(s));
  });
}

int loam_gpu_spmv(const loam_sparsity_desc* sparsity, const double* values, const double* x, int64_t x_len,
                  double* y, void* stream) {
  return guarded([&] {
    require_device();
    require(sparsity != nullptr, LOAM_ERR(InvalidArgument), "spmv without a sparsity");
    spmv(single_block(sparsity, values), x, x_len, y, false, as_stream(stream));
  });
}

namespace {
BlockOperator block_op(const loam_block_mat* op) {
  require(op != nullptr, LOAM_ERR(InvalidArgument), "null block operator");
  BlockOperator B;
  for (int i = 0; i < 2; ++i) {
    B.row_sizes[i] = op->row_sizes[i];
    B.col_sizes[i] = op->col_sizes[i];
    for (int j = 0; j < 2; ++j) {
      B.sparsity[i][j] = op->sparsity[i][j];
      B.values[i][j] = op->values[i][j];
    }
  }
  return B;
}
} // namespace

int loam_gpu_block_spmv(const loam_block_mat* op, const double* x, int64_t x_len, double* y, void* stream) {
  return guarded([&] {
    require_device();
    spmv(block_op(op), x, x_len, y, true, as_stream(stream));
  });
}

int loam_gpu_cg_solve(const loam_sparsity_desc* sparsity, const double* values, const double* b, int64_t b_len,
                      double* x, double rtol, double atol, int32_t maxit, int32_t jacobi, loam_solve_report* report,
                      void* stream) {
  return guarded([&] {
    require_device();
    require(sparsity != nullptr && report != nullptr, LOAM_ERR(InvalidArgument), "cg without matrix or report");
    *report = cg_solve(single_block(sparsity, values), b, b_len, x, rtol, atol, maxit, jacobi != 0, false,
                       as_stream(stream));
  });
}

int loam_gpu_cg_solve_block(const loam_block_mat* op, const double* b, int64_t b_len, double* x, double rtol,
                            double atol, int32_t maxit, int32_t jacobi, loam_solve_report* report, void* stream) {
  return guarded([&] {
    require_device();
    require(report != nullptr, LOAM_ERR(InvalidArgument), "cg without a report");
    *report = cg_solve(block_op(op), b, b_len, x, rtol, atol, maxit, jacobi != 0, true, as_stream(stream));
  });
}

int loam_gpu_map_check(const loam_map_desc* map, void* stream) {
  return guarded([&] {
    require_device();
    map_check(map, as_stream(stream));
  });
}

int loam_gpu_build_sparsity(const loam_map_desc* row_map, const loam_map_desc* col_map, int row_dim,
                            int col_dim, int64_t** row_ptr, int32_t** col_idx, int64_t* nnz, void* stream) {
  return guarded([&] {
    require_device();
    require(row_dim >= 1 && col_dim >= 1, LOAM_ERR(InvalidArgument), "dims must be positive");
    require(row_map->source_size == col_map->source_size &&
                (row_map->source_id == 0 || col_map->source_id == 0 || row_map->source_id == col_map->source_id),
            LOAM_ERR(SourceMismatch), "row and column maps must share their source set");
    MapView r{row_map->values, row_map->source_size, row_map->arity, row_map->target_size};
    MapView c{col_map->values, col_map->source_size, col_map->arity, col_map->target_size};
    build_sparsity_dev(r, c, row_dim, col_dim, row_ptr, col_idx, nnz, as_stream(stream));
    LG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  });
}

int loam_gpu_color_iteration(int32_t n, uint64_t iter, const loam_map_desc* maps, int nmaps, int32_t* colors,
                             int32_t* num_colors, void* stream) {
  return guarded([&] {
    require_device();
    for (int i = 0; i < nmaps; ++i)
      require(maps[i].source_id == 0 || iter == 0 || maps[i].source_id == iter, LOAM_ERR(SourceMismatch),
              "conflict map source differs from iteration set");
    color_iteration(n, maps, nmaps, colors, num_colors, as_stream(stream));
  });
}

int loam_gpu_malloc(void** ptr, size_t bytes) {
  return guarded([&] {
    require_device();
    LG_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
  });
}
int loam_gpu_free(void* ptr) {
  return guarded([&] { LG_CUDA(cudaFree(ptr)); });
}
int loam_gpu_host_alloc(void** ptr, size_t bytes) {
  return guarded([&] {
    require_device();
    LG_CUDA(cudaMallocHost(ptr, bytes ? bytes : 1));
  });
}
int loam_gpu_host_free(void* ptr) {
  return guarded([&] { LG_CUDA(cudaFreeHost(ptr)); });
}
int loam_gpu_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] { LG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream))); });
}
int loam_gpu_memset(void* dst, int value, size_t bytes, void* stream) {
  return guarded([&] { LG_CUDA(cudaMemsetAsync(dst, value, bytes, as_stream(stream))); });
}
int loam_gpu_stream_sync(void* stream) {
  return guarded([&] { LG_CUDA(cudaStreamSynchronize(as_stream(stream))); });
}

} // extern "C"

// ---- around the assembly loop (fem.cu) -----------------------------------
extern "C" {

int loam_gpu_apply_dirichlet(const loam_sparsity_desc* sparsity, double* values, double* rhs, const int32_t* nodes,
                             int32_t nnodes, const double* node_values, double constant, void* stream) {
  return guarded([&] {
    require_device();
    apply_dirichlet(sparsity, values, rhs, nodes, nnodes, node_values, constant, as_stream(stream));
  });
}

int loam_gpu_bc_apply(double* dat, int32_t set_size, const int32_t* nodes, int32_t nnodes, const double* node_values,
                      double constant, void* stream) {
  return guarded([&] {
    require_device();
    bc_apply(dat, set_size, nodes, nnodes, node_values, constant, as_stream(stream));
  });
}

int loam_gpu_pointwise(double* out, int64_t n, int32_t op, const loam_pw_instr* program, int32_t nprogram,
                       const double* const* fields, int32_t nfields, void* stream) {
  return guarded([&] {
    pw_check(program, nprogram, nfields); // program errors are reported without a device
    require_device();
    pointwise(out, n, op, program, nprogram, fields, nfields, as_stream(stream));
  });
}

int loam_gpu_reduce_dev(const double* x, int64_t n, int32_t kind, double* result_dev, void* stream) {
  return guarded([&] {
    require_device();
    require(result_dev != nullptr, LOAM_ERR(InvalidArgument), "reduce without a result");
    reduce(x, n, kind, result_dev, as_stream(stream));
  });
}

int loam_gpu_bc_apply_dev(double* dat, int32_t set_size, const int32_t* nodes, int32_t nnodes,
                          const double* value_dev, void* stream) {
  return guarded([&] {
    require_device();
    require(value_dev != nullptr, LOAM_ERR(InvalidArgument), "bc apply without a device value");
    bc_apply(dat, set_size, nodes, nnodes, nullptr, 0.0, as_stream(stream), value_dev);
  });
}

int loam_gpu_wave_clock(double* state_dev, double dt, double first_period, int32_t phase, void* stream) {
  return guarded([&] {
    require_device();
    wave_clock(state_dev, dt, first_period, phase, as_stream(stream));
  });
}

int loam_gpu_reduce(const double* x, int64_t n, int32_t kind, double* result, void* stream) {
  return guarded([&] {
    require_device();
    require(result != nullptr, LOAM_ERR(InvalidArgument), "reduce without a result");
    const cudaStream_t s = as_stream(stream);
    DevBuf<double> r(1, s);
    reduce(x, n, kind, r.get(), s);
    LG_CUDA(cudaMemcpyAsync(result, r.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    LG_CUDA(cudaStreamSynchronize(s));
  });
}

} // extern "C"

// ---- mesh-side builders (mesh.cu) ------------------------------------------
extern "C" {

int loam_gpu_p2_cell_node_map_dev(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv, int32_t* cn,
                                  int32_t* nnodes, void* stream) {
  return guarded([&] {
    require_device();
    require(nnodes != nullptr, LOAM_ERR(InvalidArgument), "null node count");
    *nnodes = p2_cell_node_map_dev(cv, ncells, nverts, gdim, cn, as_stream(stream));
    LG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  });
}

int loam_gpu_exterior_facets(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv,
                             int32_t** facet_vertices, int32_t** facet_cell, int32_t* nfacets, void* stream) {
  return guarded([&] {
    require_device();
    require(facet_vertices && facet_cell && nfacets, LOAM_ERR(InvalidArgument), "null output");
    *nfacets = exterior_facets_dev(cv, ncells, nverts, gdim, facet_vertices, facet_cell, as_stream(stream));
  });
}

int loam_gpu_wave_step(const loam_kernel_desc* kernel, int32_t n, uint64_t iter, const loam_arg_desc* args,
                       int nargs, const double* p_in, const double* phi_in, double* p_out, double* phi_out,
                       const double* p_constant, const uint8_t* bc_mask, double half_dt, double* state,
                       void* stream) {
  return guarded([&] {
    require_device();
    require(p_in && phi_in && p_out && phi_out && p_constant && bc_mask && state, LOAM_ERR(InvalidArgument),
            "null field");
    require(p_out != p_in && phi_out != phi_in && p_out != phi_in && phi_out != p_in, LOAM_ERR(InvalidArgument),
            "wave step: outputs must not alias the inputs");
    wave_step(kernel, n, iter, args, nargs, p_in, phi_in, p_out, phi_out, p_constant, bc_mask, half_dt, state,
              as_stream(stream));
  });
}

int loam_gpu_rcm_order(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, int32_t* order, void* stream) {
  return guarded([&] {
    require_device();
    require(n == 0 || (row_ptr && col_idx && order), LOAM_ERR(InvalidArgument), "null adjacency or output");
    rcm_order_dev(n, row_ptr, col_idx, order, as_stream(stream));
  });
}

int loam_gpu_vertex_adjacency(int32_t ncells, int32_t nverts, int32_t gdim, const int32_t* cv, int64_t** row_ptr,
                              int32_t** col_idx, int64_t* nnz, void* stream) {
  return guarded([&] {
    require_device();
    require(row_ptr && col_idx && nnz, LOAM_ERR(InvalidArgument), "null output");
    require(gdim == 2 || gdim == 3, LOAM_ERR(InvalidArgument), "gdim must be 2 or 3");
    *nnz = vertex_adjacency_dev(cv, ncells, nverts, gdim, row_ptr, col_idx, as_stream(stream));
  });
}

int loam_gpu_renumber_vertices(int32_t nverts, int32_t gdim, const double* coords, int32_t ncells, const int32_t* cv,
                               const int32_t* perm, double* coords_out, int32_t* cv_out, void* stream) {
  return guarded([&] {
    require_device();
    require(gdim == 2 || gdim == 3, LOAM_ERR(InvalidArgument), "gdim must be 2 or 3");
    renumber_vertices_dev(nverts, gdim, coords, ncells, cv, perm, coords_out, cv_out, as_stream(stream));
  });
}

} // extern "C"
