// loam_gpu_ref.hpp -- adapter from the REFERENCE's own objects to the B200
// engine (the drop-in seen from the reference's side).
//
// Include after the reference headers are on the include path
// (-I<reference>/proj/include) and link libloam_gpu.so.  Nothing here is a
// copy of the reference: it reads the reference's public objects
// (loam::Parloop, Set/Map/Dat/Mat/Global, fem::Form, MixedForm) and turns them
// into the C-ABI descriptors of include/loam_gpu.h, host pointers straight
// into the reference's own storage (std::vector<int> map values,
// std::vector<Real> Dat / Mat values, std::vector<long> row offsets).
//
//   loam_gpu_ref::execute(loop, threads)      replaces loam::execute            parloop.hpp:191
//   loam_gpu_ref::validate(loop)              = loam::validate (the reference's) parloop.hpp:89
//   loam_gpu_ref::build_sparsity(r, c, rd, cd) replaces loam::build_sparsity    data.hpp:149-179
//   loam_gpu_ref::fem::assemble_matrix(form)  replaces fem::assemble_matrix     assemble.hpp:85-104
//   loam_gpu_ref::fem::assemble_vector(form)  replaces fem::assemble_vector     assemble.hpp:108-135
//   loam_gpu_ref::fem::assemble_blocks(mixed) replaces fem::assemble_blocks     assemble.hpp:439-448
//
// Kernels are dispatched on ir::Kernel::name (kernel.hpp:504-511): the
// reference's form compiler names its kernels "<kind>_p<deg>_<tri|tet>"
// (form.hpp:214-222) and the B200 registry uses the same names.  Literals
// the reference bakes into a kernel's AST (Helmholtz kappa) are passed as
// `params`; the fem:: callers take them from the Form (Form::constant).  A
// kernel without a device implementation is an error -- never a CPU
// fallback -- exactly like the C ABI.
//
// Semantics kept: validate runs first and before any mutation (the
// reference's own loam::validate, so messages are identical); written Dats
// bump their version once (parloop.hpp:217 mutable_view); a Mat INC adds to
// the current values; results are in the reference objects on return
// (synchronous, like loam::execute).  `threads` is accepted and ignored.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "loam/fem/assemble.hpp"
#include "loam/parloop.hpp"
#include "loam_gpu.h"

namespace loam_gpu_ref {

static_assert(sizeof(long) == sizeof(int64_t), "reference row offsets (std::vector<long>) must be 64-bit");
static_assert(sizeof(int) == sizeof(int32_t), "reference map values (std::vector<int>) must be 32-bit");
static_assert(sizeof(loam::Real) == sizeof(double), "reference Real must be double");

namespace detail {

/// C-ABI return code -> the reference's exception (loam::Error, same kind).
inline void check(int code) {
  if (code == 0) return;
  const char* msg = loam_gpu_last_error();
  if (code >= 1 && code <= 1 + LOAM_KIND_InvalidArgument)
    throw loam::Error(static_cast<loam::ErrorKind>(code - 1), msg ? msg : "loam_gpu error");
  throw loam::Error(loam::ErrorKind::InvalidArgument, std::string("loam_gpu: ") + (msg ? msg : "device error"));
}

/// Object identities for the engine's plan cache.  The reference compares
/// objects by shared_ptr identity; here every live object gets a library id
/// (loam_gpu_new_id).  An entry remembers its object weakly: once the object
/// is gone its id is released (cached plans and resident copies evicted), so
/// a recycled heap address never inherits another object's plan.
class Ids {
public:
  template <class T>
  uint64_t of(const std::shared_ptr<T>& p) {
    if (!p) return 0;
    std::lock_guard<std::mutex> lk(mu_);
    sweep();
    const void* key = static_cast<const void*>(p.get());
    auto it = ids_.find(key);
    if (it != ids_.end() && !it->second.first.expired()) return it->second.second;
    if (it != ids_.end()) {
      loam_gpu_release_id(it->second.second);
      ids_.erase(it);
    }
    const uint64_t id = loam_gpu_new_id();
    ids_.emplace(key, std::make_pair(std::weak_ptr<const void>(std::shared_ptr<const void>(p)), id));
    return id;
  }

private:
  void sweep() {
    if (++calls_ % 64) return;
    for (auto it = ids_.begin(); it != ids_.end();) {
      if (it->second.first.expired()) {
        loam_gpu_release_id(it->second.second);
        it = ids_.erase(it);
      } else {
        ++it;
      }
    }
  }
  std::mutex mu_;
  std::unordered_map<const void*, std::pair<std::weak_ptr<const void>, uint64_t>> ids_;
  uint64_t calls_ = 0;
};

inline Ids& ids() {
  static Ids r;
  return r;
}

/// Patterns built through loam_gpu_ref::build_sparsity remember the maps and
/// dof dims they came from (loam_sparsity_desc provenance): a loop over
/// exactly those maps may then write a fresh Mat's rows without zero-filling.
struct Provenance {
  std::weak_ptr<const loam::Sparsity> sp;
  uint64_t row_map = 0, col_map = 0;
  int row_dim = 1, col_dim = 1;
};

inline std::mutex& prov_mutex() {
  static std::mutex m;
  return m;
}
inline std::unordered_map<const void*, Provenance>& provenance() {
  static std::unordered_map<const void*, Provenance> p;
  return p;
}

inline loam_map_desc map_desc(const loam::MapPtr& m) {
  loam_map_desc d{};
  d.values = m->values().data();
  d.source_size = m->source()->size();
  d.target_size = m->target()->size();
  d.arity = m->arity();
  d.source_id = ids().of(m->source());
  d.target_id = ids().of(m->target());
  d.id = ids().of(m);
  d.expand_dim = 0;
  return d;
}

inline loam_sparsity_desc sparsity_desc(const loam::SparsityPtr& sp) {
  loam_sparsity_desc d{};
  d.row_ptr = reinterpret_cast<const int64_t*>(sp->row_offsets().data());
  d.col_idx = sp->col_indices().data();
  d.nrows = sp->nrows();
  d.ncols = sp->ncols();
  d.nnz = sp->nnz();
  d.row_dim = 1;
  d.col_dim = 1;
  d.id = ids().of(sp);
  std::lock_guard<std::mutex> lk(prov_mutex());
  auto it = provenance().find(sp.get());
  if (it != provenance().end() && !it->second.sp.expired()) {
    d.pattern_row_map = it->second.row_map;
    d.pattern_col_map = it->second.col_map;
    d.pattern_row_dim = it->second.row_dim;
    d.pattern_col_dim = it->second.col_dim;
  }
  return d;
}

/// Descriptors of one Parloop over the reference's host storage.  `fresh`
/// lists args whose target the caller just created zero-initialised
/// (make_dat / make_mat, data.hpp:37-39,185-187): LOAM_ARG_ZERO, no upload.
struct Descs {
  std::vector<loam_map_desc> maps;
  std::vector<loam_sparsity_desc> sps;
  std::vector<loam_arg_desc> args;
};

inline void describe(const loam::Parloop& loop, const std::vector<bool>& fresh, Descs& out) {
  const size_t n = loop.args.size();
  out.maps.assign(2 * n, loam_map_desc{});
  out.sps.assign(n, loam_sparsity_desc{});
  out.args.assign(n, loam_arg_desc{});
  for (size_t k = 0; k < n; ++k) {
    const loam::Arg& a = loop.args[k];
    loam_arg_desc& d = out.args[k];
    d.access = static_cast<int32_t>(a.access);
    d.flags = (k < fresh.size() && fresh[k]) ? LOAM_ARG_ZERO : 0;
    if (a.is_dat()) {
      d.kind = LOAM_ARG_DAT;
      // written Dats: one mutable_view per execute (version bump, parloop.hpp:217)
      d.data = loam::detail::writes(a.access) ? a.dat->mutable_view().data()
                                              : const_cast<double*>(a.dat->view().data());
      d.dim = a.dat->dim();
      d.set_size = a.dat->set()->size();
      d.set_id = ids().of(a.dat->set());
      d.obj_id = ids().of(a.dat);
      if (!a.direct()) {
        out.maps[2 * k] = map_desc(a.maps[0]);
        d.map = &out.maps[2 * k];
      }
    } else if (a.is_mat()) {
      d.kind = LOAM_ARG_MAT;
      d.data = a.mat->values().data();
      d.obj_id = ids().of(a.mat);
      out.maps[2 * k] = map_desc(a.maps[0]);
      out.maps[2 * k + 1] = map_desc(a.maps[1]);
      d.map = &out.maps[2 * k];
      d.col_map = &out.maps[2 * k + 1];
      out.sps[k] = sparsity_desc(a.mat->sparsity());
      d.sparsity = &out.sps[k];
    } else {
      d.kind = LOAM_ARG_GLOBAL;
      d.data = a.global->mutable_view().data();
      d.dim = a.global->dim();
      d.obj_id = ids().of(a.global);
    }
  }
}

inline void execute_impl(const loam::Parloop& loop, const std::vector<double>& params,
                         const std::vector<bool>& fresh) {
  loam::validate(loop); // the reference's own checks and messages, before any mutation
  Descs ds;
  describe(loop, fresh, ds);
  loam_kernel_desc kd{loop.kernel->name.c_str(), params.empty() ? nullptr : params.data(),
                      static_cast<int32_t>(params.size())};
  check(loam_gpu_execute_host(&kd, loop.iterset->size(), ids().of(loop.iterset), ds.args.data(),
                              static_cast<int>(ds.args.size()), nullptr));
}

} // namespace detail

/// loam::validate (parloop.hpp:89-146): the reference's own function.
inline void validate(const loam::Parloop& loop) { loam::validate(loop); }

/// loam::execute (parloop.hpp:191) on the B200.  `params` = the literals of
/// the kernel (e.g. {kappa} for helmholtz_*); empty for kernels without any.
inline void execute(const loam::Parloop& loop, int threads = 1, const std::vector<double>& params = {}) {
  loam::require(threads >= 1, loam::ErrorKind::InvalidArgument, "thread count must be positive");
  detail::execute_impl(loop, params, {});
}

/// loam::build_sparsity (data.hpp:149-179) on the device: bit-exact, returned
/// as the reference's own Sparsity object.
inline loam::SparsityPtr build_sparsity(const loam::MapPtr& row_map, const loam::MapPtr& col_map, int row_dim = 1,
                                        int col_dim = 1) {
  loam::require(row_map->source() == col_map->source(), loam::ErrorKind::SourceMismatch,
                "row and column maps must share their source set");
  const loam_map_desc rh = detail::map_desc(row_map), ch = detail::map_desc(col_map);
  // device copies of the two maps (the engine's build works on device memory)
  auto upload = [](const loam_map_desc& h, int32_t** dev) {
    const size_t bytes = sizeof(int32_t) * (size_t)h.source_size * h.arity;
    detail::check(loam_gpu_malloc(reinterpret_cast<void**>(dev), bytes ? bytes : 4));
    if (bytes) detail::check(loam_gpu_memcpy(*dev, h.values, bytes, nullptr));
  };
  int32_t *dr = nullptr, *dc = nullptr;
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  int64_t nnz = 0;
  std::vector<long> offsets;
  std::vector<int> cols;
  try {
    upload(rh, &dr);
    if (col_map == row_map) dc = dr;
    else upload(ch, &dc);
    loam_map_desc rd = rh, cd = ch;
    rd.values = dr;
    cd.values = dc;
    rd.id = cd.id = 0; // device copies: not the host objects' resident copies
    if (col_map == row_map) cd = rd;
    detail::check(loam_gpu_build_sparsity(&rd, &cd, row_dim, col_dim, &rp, &ci, &nnz, nullptr));
    const int nrows = row_map->target()->size() * row_dim;
    offsets.resize((size_t)nrows + 1);
    cols.resize((size_t)nnz);
    detail::check(loam_gpu_memcpy(offsets.data(), rp, sizeof(int64_t) * offsets.size(), nullptr));
    if (nnz) detail::check(loam_gpu_memcpy(cols.data(), ci, sizeof(int32_t) * (size_t)nnz, nullptr));
    detail::check(loam_gpu_stream_sync(nullptr));
  } catch (...) {
    if (rp) loam_gpu_free(rp);
    if (ci) loam_gpu_free(ci);
    if (dc && dc != dr) loam_gpu_free(dc);
    if (dr) loam_gpu_free(dr);
    throw;
  }
  loam_gpu_free(rp);
  loam_gpu_free(ci);
  if (dc != dr) loam_gpu_free(dc);
  loam_gpu_free(dr);
  auto sp = std::make_shared<const loam::Sparsity>(row_map->target()->size() * row_dim,
                                                   col_map->target()->size() * col_dim, std::move(offsets),
                                                   std::move(cols));
  {
    std::lock_guard<std::mutex> lk(detail::prov_mutex());
    auto& prov = detail::provenance();
    for (auto it = prov.begin(); it != prov.end();) // drop dead patterns
      it = it->second.sp.expired() ? prov.erase(it) : std::next(it);
    prov[sp.get()] = detail::Provenance{sp, rh.id, ch.id, row_dim, col_dim};
  }
  return sp;
}

namespace fem {

namespace detail {

/// The kernel name the reference's form compiler gives `form`
/// (form.hpp:214-222) and the literals its AST bakes in.
inline loam::ir::KernelPtr kernel_of(const loam::fem::Form& form, std::vector<double>& params) {
  using loam::fem::FormKind;
  const auto& mesh = *form.test->mesh;
  std::string name;
  switch (form.kind) {
  case FormKind::Mass: name = form.bilinear() ? "mass" : "mass_action"; break;
  case FormKind::Stiffness: name = form.bilinear() ? "stiffness" : "stiffness_action"; break;
  case FormKind::Helmholtz: name = "helmholtz"; break;
  case FormKind::Source: name = "source"; break;
  default:
    loam::fail(loam::ErrorKind::UnsupportedForm, "facet forms have no device implementation");
  }
  name += "_p" + std::to_string(form.test->element.degree) + (mesh.dim == 2 ? "_tri" : "_tet");
  params.clear();
  if (form.kind == FormKind::Helmholtz) params.push_back(form.constant);
  // the device kernel is looked up by name; the AST is not needed on this path
  auto k = std::make_shared<loam::ir::Kernel>();
  k->name = name;
  int32_t buf[64];
  const int np = loam_gpu_kernel_signature(name.c_str(), buf, 64);
  loam_gpu_ref::detail::check(np < 0 ? -np : 0);
  for (int p = 0, o = 0; p < np; ++p) { // staged extents: the registry's = the reference's
    const int rank = buf[o++];
    std::vector<int> ext(buf + o, buf + o + rank);
    o += rank;
    k->host_params.push_back(loam::ir::Param{"p" + std::to_string(p), std::move(ext)});
  }
  return k;
}

} // namespace detail

/// fem::assemble_matrix (assemble.hpp:85-104) on the B200: sparsity built on
/// the device, the cell loop executed by the engine, Dirichlet rows as the
/// reference applies them.
inline loam::MatPtr assemble_matrix(const loam::fem::Form& form, const std::vector<loam::fem::DirichletBC>& bcs = {},
                                    int threads = 1) {
  loam::require(form.bilinear(), loam::ErrorKind::UnsupportedForm, "matrix assembly needs a bilinear form");
  loam::require(threads >= 1, loam::ErrorKind::InvalidArgument, "thread count must be positive");
  auto sparsity = loam_gpu_ref::build_sparsity(form.test->cell_node_map, form.trial->cell_node_map);
  auto mat = loam::make_mat(std::move(sparsity), "assembled");
  std::vector<double> params;
  loam::Parloop loop;
  loop.kernel = detail::kernel_of(form, params);
  loop.iterset = form.test->mesh->cells;
  loop.args.push_back(loam::arg(mat, loam::Access::INC, form.test->cell_node_map, form.trial->cell_node_map));
  loop.args.push_back(loam::arg(form.test->mesh->coordinates, loam::Access::READ, form.test->mesh->cell_vertex_map));
  if (form.coefficient)
    loop.args.push_back(
        loam::arg(form.coefficient->dat, loam::Access::READ, form.coefficient->space->cell_node_map));
  loam_gpu_ref::detail::execute_impl(loop, params, {true}); // the Mat is fresh (make_mat zero-fills)
  for (const auto& bc : bcs) loam::fem::apply_dirichlet_rows(*mat, bc);
  return mat;
}

/// fem::assemble_vector (assemble.hpp:108-135) for cell forms on the B200.  A
/// constant source density is interpolated into a constant coefficient (the
/// same integral, rounding aside).  Facet sources have no device kernel.
inline loam::DatPtr assemble_vector(const loam::fem::Form& form, const std::vector<loam::fem::DirichletBC>& bcs = {},
                                    int threads = 1) {
  loam::require(!form.bilinear(), loam::ErrorKind::UnsupportedForm, "vector assembly needs a linear form");
  loam::require(threads >= 1, loam::ErrorKind::InvalidArgument, "thread count must be positive");
  auto out = loam::make_dat(form.test->node_set, 1, "assembled");
  std::vector<double> params;
  loam::Parloop loop;
  loop.kernel = detail::kernel_of(form, params);
  loop.iterset = form.test->mesh->cells;
  loop.args.push_back(loam::arg(out, loam::Access::INC, form.test->cell_node_map));
  loop.args.push_back(loam::arg(form.test->mesh->coordinates, loam::Access::READ, form.test->mesh->cell_vertex_map));
  if (form.coefficient) {
    loop.args.push_back(
        loam::arg(form.coefficient->dat, loam::Access::READ, form.coefficient->space->cell_node_map));
  } else if (form.kind == loam::fem::FormKind::Source) {
    auto c = loam::make_dat(form.test->node_set, 1, "density");
    auto v = c->mutable_view();
    std::fill(v.begin(), v.end(), form.constant);
    loop.args.push_back(loam::arg(c, loam::Access::READ, form.test->cell_node_map));
  }
  loam_gpu_ref::detail::execute_impl(loop, params, {true});
  for (const auto& bc : bcs) bc.apply(*out);
  return out;
}

/// fem::assemble_blocks (assemble.hpp:439-448): the nested 2x2 BlockMat
/// (solver.hpp:21-28), every present block assembled on the B200.
inline loam::BlockMat assemble_blocks(const loam::fem::MixedForm& mixed, int threads = 1) {
  auto blocks = loam::fem::split_mixed(mixed);
  loam::BlockMat out;
  for (int i = 0; i < 2; ++i) out.row_sizes[i] = mixed.test[i]->node_set->size();
  for (int j = 0; j < 2; ++j) out.col_sizes[j] = mixed.trial[j]->node_set->size();
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      if (blocks[i][j]) out.blocks[i][j] = loam_gpu_ref::fem::assemble_matrix(*blocks[i][j], {}, threads);
  return out;
}

} // namespace fem

} // namespace loam_gpu_ref
