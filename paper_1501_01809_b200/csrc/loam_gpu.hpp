// loam_gpu.hpp -- C++ drop-in facade of the reference operator surface.
//
// Mirrors /root/reference/proj/include/loam (C++20 header-only) for the
// par_loop path, over the C ABI of include/loam_gpu.h:
//   Set / Map / make_set / make_map                topology.hpp:15-74
//   Coloring / color_iteration                     topology.hpp:76-125
//   Access / Dat / Global / Sparsity / Mat         data.hpp:15-234
//   build_sparsity                                 data.hpp:149-179
//   Arg / arg() / Parloop / validate / execute     parloop.hpp:17-384
//   Error / ErrorKind                              common.hpp:10-49
// Porting code from the reference means replacing `loam::` by `loam_gpu::`
// and the AST kernel by a registry kernel (kernel.hpp:504-511 -> Kernel{name,
// params}); every call keeps its arguments, meaning and error kinds.  Objects
// own DEVICE storage (cudaMalloc); view()/mutable_view() expose a host mirror
// that is synchronised on demand, so the reference's host-side idioms work.
#pragma once
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "loam_gpu.h"

namespace loam_gpu {

using Real = double;

enum class ErrorKind {
  IndexOutOfRange, ArityMismatch, SourceMismatch, AsymmetricAdjacency, IllegalAccess,
  MapSourceMismatch, ShapeMismatch, UnboundIdentifier, NonDividingFactor, OutsideSparsity,
  EmptyPartials, DimensionMismatch, InvalidSubdivision, ParseError, NonManifold, CellMismatch,
  UnsupportedForm, MissingDiagonal, SpaceMismatch, IndefiniteBreakdown, InstabilityDetected,
  InvalidArgument,
  CudaError = 99, NoDevice = 100
};

class Error : public std::runtime_error {
public:
  Error(ErrorKind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

private:
  ErrorKind kind_;
};

inline void check(int code) {
  if (code == 0) return;
  const ErrorKind k = code == LOAM_GPU_ERR_CUDA ? ErrorKind::CudaError
                      : code == LOAM_GPU_ERR_NO_DEVICE ? ErrorKind::NoDevice
                                                       : static_cast<ErrorKind>(code - 1);
  throw Error(k, loam_gpu_last_error());
}
inline void require(bool c, ErrorKind k, const std::string& m) {
  if (!c) throw Error(k, m);
}

namespace detail {
// Identities come from the library so they are unique across every client
// of it in the process (plans and resident copies are cached by id).
inline uint64_t next_id() { return loam_gpu_new_id(); }
template <class T>
struct DeviceArray { // owned device buffer + lazily synchronised host mirror
  T* dev = nullptr;
  size_t n = 0;
  mutable std::vector<T> host;
  mutable bool host_valid = false, dev_stale = false;
  explicit DeviceArray(size_t count, bool zero = true) : n(count) {
    check(loam_gpu_malloc(reinterpret_cast<void**>(&dev), sizeof(T) * (n ? n : 1)));
    if (zero) check(loam_gpu_memset(dev, 0, sizeof(T) * (n ? n : 1), nullptr));
  }
  ~DeviceArray() { loam_gpu_free(dev); }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  void upload(const T* src) {
    check(loam_gpu_memcpy(dev, src, sizeof(T) * n, nullptr));
    check(loam_gpu_stream_sync(nullptr));
    host_valid = false;
  }
  const std::vector<T>& download() const {
    if (!host_valid) {
      host.resize(n);
      check(loam_gpu_memcpy(host.data(), dev, sizeof(T) * n, nullptr));
      check(loam_gpu_stream_sync(nullptr));
      host_valid = true;
    }
    return host;
  }
  T* device() { // push host edits (mutable_view) before device use
    if (dev_stale) {
      check(loam_gpu_memcpy(dev, host.data(), sizeof(T) * n, nullptr));
      dev_stale = false;
    }
    return dev;
  }
};
} // namespace detail

// ---------------------------------------------------------------- topology
class Set { // topology.hpp:15-26
public:
  explicit Set(int size, std::string name = "set") : size_(size), name_(std::move(name)) {
    require(size >= 0, ErrorKind::InvalidArgument, "Set size must be non-negative");
  }
  int size() const { return size_; }
  const std::string& name() const { return name_; }
  uint64_t id() const { return id_; }

private:
  int size_;
  std::string name_;
  uint64_t id_ = detail::next_id();
};
using SetPtr = std::shared_ptr<const Set>;
inline SetPtr make_set(int size, std::string name = "set") { return std::make_shared<const Set>(size, std::move(name)); }

class Map { // topology.hpp:36-66 (validated on construction, on the device)
public:
  Map(SetPtr source, SetPtr target, int arity, std::vector<int> values, std::string name = "map")
      : source_(std::move(source)), target_(std::move(target)), arity_(arity), values_(std::move(values)),
        name_(std::move(name)), dev_(values_.size()) {
    require(arity_ > 0, ErrorKind::InvalidArgument, "Map arity must be positive");
    require((long)values_.size() == (long)source_->size() * arity_, ErrorKind::ArityMismatch,
            name_ + ": value table length != source size * arity");
    dev_.upload(values_.data());
    loam_map_desc d = desc();
    if (!values_.empty()) check(loam_gpu_map_check(&d, nullptr));
  }
  const SetPtr& source() const { return source_; }
  const SetPtr& target() const { return target_; }
  int arity() const { return arity_; }
  const std::string& name() const { return name_; }
  ~Map() { loam_gpu_release_id(id_); } // evict the plans cached for this map
  uint64_t id() const { return id_; }
  Map(const Map&) = delete;
  Map& operator=(const Map&) = delete;
  const int* row(int e) const { return values_.data() + static_cast<long>(e) * arity_; }
  const std::vector<int>& values() const { return values_; }
  loam_map_desc desc() const {
    loam_map_desc d{};
    d.values = dev_.dev;
    d.source_size = source_->size();
    d.target_size = target_->size();
    d.arity = arity_;
    d.source_id = source_->id();
    d.target_id = target_->id();
    d.id = id_;
    if (node_) { // a dof-expanded map declares the node map it expands
      const loam_map_desc n = node_->desc();
      d.expand_dim = expand_dim_;
      d.node_values = n.values;
      d.node_arity = n.arity;
      d.node_target_size = n.target_size;
      d.node_id = n.id;
    }
    return d;
  }
  /// (make_expanded_map) the node map this map expands by `dim` dofs per node
  void declare_node_map(std::shared_ptr<const Map> node, int dim) const {
    node_ = std::move(node);
    expand_dim_ = dim;
  }
  const std::shared_ptr<const Map>& node_map() const { return node_; }
  int expand_dim() const { return expand_dim_; }

private:
  SetPtr source_, target_;
  int arity_;
  std::vector<int> values_;
  std::string name_;
  detail::DeviceArray<int32_t> dev_;
  uint64_t id_ = detail::next_id();
  mutable std::shared_ptr<const Map> node_;
  mutable int expand_dim_ = 0;
};
using MapPtr = std::shared_ptr<const Map>;
inline MapPtr make_map(SetPtr source, SetPtr target, int arity, std::vector<int> values, std::string name = "map") {
  return std::make_shared<const Map>(std::move(source), std::move(target), arity, std::move(values), std::move(name));
}

/// The dof-expanded map a vector-valued Mat needs (entries dim * node + d, the
/// layout fem spaces with value_dim > 1 use), declaring its node map
/// so the device works on the 1/dim-size node map.
inline MapPtr make_expanded_map(const MapPtr& node_map, int dim, SetPtr dofs = nullptr, std::string name = "dof_map") {
  require(dim >= 1, ErrorKind::InvalidArgument, "dof expansion must be positive");
  if (!dofs) dofs = make_set(node_map->target()->size() * dim, name + "_dofs");
  const std::vector<int>& v = node_map->values();
  std::vector<int> exp(v.size() * (size_t)dim);
  for (size_t i = 0; i < v.size(); ++i)
    for (int d = 0; d < dim; ++d) exp[i * dim + d] = v[i] * dim + d;
  auto m = make_map(node_map->source(), std::move(dofs), node_map->arity() * dim, std::move(exp), std::move(name));
  m->declare_node_map(node_map, dim);
  return m;
}

struct Coloring { // topology.hpp:78-81
  std::vector<int> colors;
  int num_colors = 0;
};
inline Coloring color_iteration(const SetPtr& iter, const std::vector<MapPtr>& conflict_maps) {
  std::vector<loam_map_desc> d;
  for (const auto& m : conflict_maps) {
    require(m->source() == iter, ErrorKind::SourceMismatch,
            "conflict map " + m->name() + " source differs from iteration set");
    d.push_back(m->desc());
  }
  detail::DeviceArray<int32_t> colors(iter->size(), false);
  int32_t nc = 0;
  check(loam_gpu_color_iteration(iter->size(), iter->id(), d.data(), (int)d.size(), colors.dev, &nc, nullptr));
  Coloring c;
  const auto& h = colors.download();
  c.colors.assign(h.begin(), h.end());
  c.num_colors = nc;
  return c;
}

// ---------------------------------------------------------------- data
enum class Access { READ, WRITE, RW, INC, SUM, MIN, MAX }; // data.hpp:17

class Dat { // data.hpp:35-60
public:
  Dat(SetPtr set, int dim, std::string name = "dat")
      : set_(std::move(set)), dim_(dim), name_(std::move(name)), data_((size_t)set_->size() * dim) {
    require(dim > 0, ErrorKind::InvalidArgument, "Dat dim must be positive");
  }
  const SetPtr& set() const { return set_; }
  int dim() const { return dim_; }
  const std::string& name() const { return name_; }
  std::uint64_t version() const { return version_; }
  std::span<const Real> view() const {
    const auto& h = data_.download();
    return {h.data(), h.size()};
  }
  std::span<Real> mutable_view() { // host edits are pushed before the next device use
    ++version_;
    data_.download();
    data_.dev_stale = true;
    zero_ = false;
    return {data_.host.data(), data_.host.size()};
  }
  // device access for execute
  double* device_data() { return data_.device(); }
  void touched_by_device() {
    ++version_;
    data_.host_valid = false;
    zero_ = false;
  }
  bool known_zero() const { return zero_; }
  uint64_t id() const { return id_; }

private:
  SetPtr set_;
  int dim_;
  std::string name_;
  detail::DeviceArray<double> data_;
  std::uint64_t version_ = 0;
  bool zero_ = true;
  uint64_t id_ = detail::next_id();
};
using DatPtr = std::shared_ptr<Dat>;
inline DatPtr make_dat(SetPtr set, int dim, std::string name = "dat") {
  return std::make_shared<Dat>(std::move(set), dim, std::move(name));
}

class Global { // data.hpp:69-87
public:
  explicit Global(int dim, std::string name = "global") : dim_(dim), name_(std::move(name)), data_(dim) {
    require(dim > 0, ErrorKind::InvalidArgument, "Global dim must be positive");
  }
  int dim() const { return dim_; }
  std::span<const Real> view() const {
    const auto& h = data_.download();
    return {h.data(), h.size()};
  }
  std::span<Real> mutable_view() {
    data_.download();
    data_.dev_stale = true;
    return {data_.host.data(), data_.host.size()};
  }
  double* device_data() { return data_.device(); }
  void touched_by_device() { data_.host_valid = false; }
  uint64_t id() const { return id_; }

private:
  int dim_;
  std::string name_;
  detail::DeviceArray<double> data_;
  uint64_t id_ = detail::next_id();
};
using GlobalPtr = std::shared_ptr<Global>;
inline GlobalPtr make_global(int dim, std::string name = "global") { return std::make_shared<Global>(dim, std::move(name)); }

class Sparsity { // data.hpp:116-142 (device CSR)
public:
  Sparsity(int nrows, int ncols, int64_t* row_ptr, int32_t* col_idx, int64_t nnz, int rd, int cd,
           uint64_t row_map_id = 0, uint64_t col_map_id = 0)
      : nrows_(nrows), ncols_(ncols), rp_(row_ptr), ci_(col_idx), nnz_(nnz), rd_(rd), cd_(cd),
        row_map_id_(row_map_id), col_map_id_(col_map_id) {}
  ~Sparsity() {
    loam_gpu_release_id(id_);
    loam_gpu_free(rp_);
    loam_gpu_free(ci_);
  }
  Sparsity(const Sparsity&) = delete;
  Sparsity& operator=(const Sparsity&) = delete;
  int nrows() const { return nrows_; }
  int ncols() const { return ncols_; }
  long nnz() const { return (long)nnz_; }
  const std::vector<long>& row_offsets() const {
    sync();
    return hrp_;
  }
  const std::vector<int>& col_indices() const {
    sync();
    return hci_;
  }
  long find(int row, int col) const { // data.hpp:129-136
    if (row < 0 || row >= nrows_) return -1;
    sync();
    auto first = hci_.begin() + hrp_[row], last = hci_.begin() + hrp_[row + 1];
    auto it = std::lower_bound(first, last, col);
    return (it == last || *it != col) ? -1 : it - hci_.begin();
  }
  loam_sparsity_desc desc() const {
    // provenance: the maps build_sparsity was given (loam_gpu.h)
    return loam_sparsity_desc{rp_, ci_, nrows_, ncols_, nnz_, rd_, cd_, id_, row_map_id_, col_map_id_, rd_, cd_};
  }

private:
  void sync() const {
    if (synced_) return;
    std::vector<int64_t> r(nrows_ + 1);
    hci_.resize(nnz_);
    check(loam_gpu_memcpy(r.data(), rp_, sizeof(int64_t) * r.size(), nullptr));
    if (nnz_) check(loam_gpu_memcpy(hci_.data(), ci_, sizeof(int32_t) * nnz_, nullptr));
    check(loam_gpu_stream_sync(nullptr));
    hrp_.assign(r.begin(), r.end());
    synced_ = true;
  }
  int nrows_, ncols_;
  int64_t* rp_;
  int32_t* ci_;
  int64_t nnz_;
  int rd_, cd_;
  uint64_t row_map_id_, col_map_id_;
  uint64_t id_ = detail::next_id();
  mutable bool synced_ = false;
  mutable std::vector<long> hrp_;
  mutable std::vector<int> hci_;
};
using SparsityPtr = std::shared_ptr<const Sparsity>;

// data.hpp:149-179, built on the device (bit-exact).
inline SparsityPtr build_sparsity(const MapPtr& row_map, const MapPtr& col_map, int row_dim = 1, int col_dim = 1) {
  require(row_map->source() == col_map->source(), ErrorKind::SourceMismatch,
          "row and column maps must share their source set");
  loam_map_desc r = row_map->desc(), c = col_map->desc();
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  int64_t nnz = 0;
  check(loam_gpu_build_sparsity(&r, &c, row_dim, col_dim, &rp, &ci, &nnz, nullptr));
  return std::make_shared<const Sparsity>(row_map->target()->size() * row_dim, col_map->target()->size() * col_dim, rp,
                                          ci, nnz, row_dim, col_dim, row_map->id(), col_map->id());
}

class Mat { // data.hpp:183-228
public:
  explicit Mat(SparsityPtr sparsity, std::string name = "mat")
      : sparsity_(std::move(sparsity)), name_(std::move(name)), values_(sparsity_->nnz(), false) {}
  const SparsityPtr& sparsity() const { return sparsity_; }
  int nrows() const { return sparsity_->nrows(); }
  int ncols() const { return sparsity_->ncols(); }
  const std::vector<Real>& values() const {
    materialize();
    return values_.download();
  }
  Real at(int row, int col) const {
    const long pos = sparsity_->find(row, col);
    return pos < 0 ? 0.0 : values()[pos];
  }
  void zero() { zero_ = stale_ = true; } // lazily: the next INC treats the values as zeros
  double* device_data() {
    materialize();
    return values_.device();
  }
  double* device_data_for_zero_inc() { return values_.dev; } // contents ignored (LOAM_ARG_ZERO)
  void touched_by_device() {
    values_.host_valid = false;
    zero_ = stale_ = false;
  }
  bool known_zero() const { return zero_; }
  uint64_t id() const { return id_; }
  const double* device_values() const { // current values on the device (for spmv / cg)
    materialize();
    return values_.device();
  }

  /// data.hpp:205-222: add (INC) or overwrite (WRITE) a dense local block at
  /// rows x cols -- the reference's host-side setter; every (row, col) pair
  /// must lie inside the sparsity.
  void addto(std::span<const int> rows, std::span<const int> cols, std::span<const Real> block,
             Access mode = Access::INC) {
    require(mode == Access::INC || mode == Access::WRITE, ErrorKind::IllegalAccess,
            "Mats are write-only: only WRITE and INC are permitted");
    require(block.size() == rows.size() * cols.size(), ErrorKind::ShapeMismatch,
            "block shape does not match rows x cols");
    materialize();
    values_.download();
    for (size_t i = 0; i < rows.size(); ++i)
      for (size_t j = 0; j < cols.size(); ++j) {
        const long pos = sparsity_->find(rows[i], cols[j]);
        require(pos >= 0, ErrorKind::OutsideSparsity,
                name_ + ": entry (" + std::to_string(rows[i]) + ", " + std::to_string(cols[j]) + ") outside sparsity");
        if (mode == Access::INC) values_.host[pos] += block[i * cols.size() + j];
        else values_.host[pos] = block[i * cols.size() + j];
      }
    values_.dev_stale = true;
    zero_ = false;
  }

private:
  void materialize() const {
    if (stale_) {
      check(loam_gpu_memset(values_.dev, 0, sizeof(double) * (values_.n ? values_.n : 1), nullptr));
      values_.host_valid = false;
      stale_ = false;
    }
  }
  SparsityPtr sparsity_;
  std::string name_;
  mutable detail::DeviceArray<double> values_;
  bool zero_ = true;
  mutable bool stale_ = true; // make_mat: zero-filled on first materialisation
  uint64_t id_ = detail::next_id();
};
using MatPtr = std::shared_ptr<Mat>;
inline MatPtr make_mat(SparsityPtr sparsity, std::string name = "mat") {
  return std::make_shared<Mat>(std::move(sparsity), std::move(name));
}

// ---------------------------------------------------------------- par_loop
struct Kernel { // ir::Kernel (kernel.hpp:504-511) -> registry key + baked literals
  std::string name;
  std::vector<double> params;
};
using KernelPtr = std::shared_ptr<const Kernel>;
inline KernelPtr kernel(std::string name, std::vector<double> params = {}) {
  return std::make_shared<const Kernel>(Kernel{std::move(name), std::move(params)});
}

struct Arg { // parloop.hpp:17-28
  DatPtr dat;
  MatPtr mat;
  GlobalPtr global;
  Access access = Access::READ;
  std::vector<MapPtr> maps;
};
inline Arg arg(DatPtr dat, Access access, MapPtr map = nullptr) {
  Arg a;
  a.dat = std::move(dat);
  a.access = access;
  if (map) a.maps.push_back(std::move(map));
  return a;
}
inline Arg arg(MatPtr mat, Access access, MapPtr row_map, MapPtr col_map) {
  Arg a;
  a.mat = std::move(mat);
  a.access = access;
  a.maps = {std::move(row_map), std::move(col_map)};
  return a;
}
inline Arg arg(GlobalPtr global, Access access) {
  Arg a;
  a.global = std::move(global);
  a.access = access;
  return a;
}

struct Parloop { // parloop.hpp:55-59
  KernelPtr kernel;
  SetPtr iterset;
  std::vector<Arg> args;
};

namespace detail {
struct Descs {
  std::vector<loam_arg_desc> args;
  std::vector<loam_map_desc> maps;
  std::vector<loam_sparsity_desc> sps;
  loam_kernel_desc kd{};
};
inline void build(const Parloop& loop, Descs& D, bool for_execute) {
  require(loop.kernel != nullptr, ErrorKind::InvalidArgument, "parloop without kernel");
  require(loop.iterset != nullptr, ErrorKind::InvalidArgument, "parloop without iteration set");
  const size_t n = loop.args.size();
  D.args.assign(n, loam_arg_desc{});
  D.maps.assign(2 * n, loam_map_desc{});
  D.sps.assign(n, loam_sparsity_desc{});
  for (size_t k = 0; k < n; ++k) {
    const Arg& a = loop.args[k];
    loam_arg_desc& d = D.args[k];
    d.access = static_cast<int32_t>(a.access);
    const int kinds = int(a.dat != nullptr) + int(a.mat != nullptr) + int(a.global != nullptr);
    require(kinds == 1, ErrorKind::InvalidArgument, "argument must target exactly one object");
    if (a.dat) {
      d.kind = LOAM_ARG_DAT;
      d.dim = a.dat->dim();
      d.set_size = a.dat->set()->size();
      d.set_id = a.dat->set()->id();
      d.obj_id = a.dat->id();
      require(a.maps.size() <= 1, ErrorKind::InvalidArgument, "Dat argument with several maps");
      if (for_execute) {
        d.data = a.dat->device_data();
        if (a.access == Access::INC && a.dat->known_zero()) d.flags = LOAM_ARG_ZERO;
      }
      if (!a.maps.empty()) {
        D.maps[2 * k] = a.maps[0]->desc();
        d.map = &D.maps[2 * k];
      }
    } else if (a.mat) {
      d.kind = LOAM_ARG_MAT;
      d.obj_id = a.mat->id();
      require(a.maps.size() == 2, ErrorKind::InvalidArgument, "Mat argument requires row and column maps");
      if (for_execute) {
        if (a.mat->known_zero()) {
          d.flags = LOAM_ARG_ZERO;
          d.data = a.mat->device_data_for_zero_inc();
        } else {
          d.data = a.mat->device_data();
        }
      }
      D.maps[2 * k] = a.maps[0]->desc();
      D.maps[2 * k + 1] = a.maps[1]->desc();
      D.sps[k] = a.mat->sparsity()->desc();
      d.map = &D.maps[2 * k];
      d.col_map = &D.maps[2 * k + 1];
      d.sparsity = &D.sps[k];
    } else {
      d.kind = LOAM_ARG_GLOBAL;
      d.dim = a.global->dim();
      d.obj_id = a.global->id();
      if (for_execute) d.data = a.global->device_data();
    }
  }
  D.kd = loam_kernel_desc{loop.kernel->name.c_str(), loop.kernel->params.data(),
                          (int32_t)loop.kernel->params.size()};
}
} // namespace detail

// parloop.hpp:89-146
inline void validate(const Parloop& loop) {
  detail::Descs D;
  detail::build(loop, D, false);
  check(loam_gpu_validate(&D.kd, loop.iterset->size(), loop.iterset->id(), D.args.data(), (int)D.args.size()));
}

// parloop.hpp:191.  `threads` is accepted for drop-in compatibility; results are
// visible on return, as in the reference (the call synchronises the stream).
inline void execute(const Parloop& loop, int threads = 1) {
  require(threads >= 1, ErrorKind::InvalidArgument, "thread count must be positive");
  detail::Descs D;
  detail::build(loop, D, true);
  check(loam_gpu_execute(&D.kd, loop.iterset->size(), loop.iterset->id(), D.args.data(), (int)D.args.size(), nullptr));
  check(loam_gpu_stream_sync(nullptr));
  for (const Arg& a : loop.args) {
    if (a.access == Access::READ) continue;
    if (a.dat) a.dat->touched_by_device();
    if (a.mat) a.mat->touched_by_device();
    if (a.global) a.global->touched_by_device();
  }
}

// fem::assemble_blocks (fem/assemble.hpp:439-448) issues one par_loop per block
// of a nested BlockMat; execute_blocks takes those loops together: all are
// validated before anything is written, then they run in order -- the
// Taylor-Hood Stokes triple (stokes_a / stokes_b / stokes_bt over one cell set
// and one pair of maps) as ONE launch.  Results visible on return.
inline void execute_blocks(const std::vector<Parloop>& loops, int threads = 1) {
  require(threads >= 1, ErrorKind::InvalidArgument, "thread count must be positive");
  std::vector<detail::Descs> D(loops.size());
  std::vector<loam_loop_desc> L(loops.size());
  for (size_t i = 0; i < loops.size(); ++i) {
    detail::build(loops[i], D[i], true);
    L[i] = loam_loop_desc{&D[i].kd, loops[i].iterset->size(), loops[i].iterset->id(), D[i].args.data(),
                          (int32_t)D[i].args.size()};
  }
  check(loam_gpu_execute_blocks(L.data(), (int)L.size(), nullptr));
  check(loam_gpu_stream_sync(nullptr));
  for (const Parloop& loop : loops)
    for (const Arg& a : loop.args) {
      if (a.access == Access::READ) continue;
      if (a.dat) a.dat->touched_by_device();
      if (a.mat) a.mat->touched_by_device();
      if (a.global) a.global->touched_by_device();
    }
}

// ---------------------------------------------------------------- matrix consumers
namespace detail {
inline DeviceArray<double>* to_device(std::span<const Real> v, std::unique_ptr<DeviceArray<double>>& keep) {
  keep = std::make_unique<DeviceArray<double>>(v.size(), false);
  if (!v.empty()) keep->upload(v.data());
  return keep.get();
}
inline std::vector<Real> to_host(const DeviceArray<double>& d, size_t n) {
  const auto& h = d.download();
  return std::vector<Real>(h.begin(), h.begin() + n);
}
} // namespace detail

/// y = A x by CSR traversal (data.hpp:236-250), bitwise equal to the reference.
inline std::vector<Real> mat_spmv(const Mat& mat, std::span<const Real> x) {
  std::unique_ptr<detail::DeviceArray<double>> dx;
  detail::to_device(x, dx);
  detail::DeviceArray<double> y(mat.nrows(), false);
  const loam_sparsity_desc sp = mat.sparsity()->desc();
  check(loam_gpu_spmv(&sp, mat.device_values(), dx->dev, (int64_t)x.size(), y.dev, nullptr));
  check(loam_gpu_stream_sync(nullptr));
  return detail::to_host(y, mat.nrows());
}

/// solver.hpp:21-28: 2x2 table of blocks; missing entries are zero blocks.
struct BlockMat {
  std::array<std::array<MatPtr, 2>, 2> blocks{};
  std::array<int, 2> row_sizes{};
  std::array<int, 2> col_sizes{};
  int nrows() const { return row_sizes[0] + row_sizes[1]; }
  int ncols() const { return col_sizes[0] + col_sizes[1]; }
};

namespace detail {
struct BlockDesc {
  loam_block_mat op{};
  loam_sparsity_desc sp[2][2]{};
  explicit BlockDesc(const BlockMat& B) {
    for (int i = 0; i < 2; ++i) {
      op.row_sizes[i] = B.row_sizes[i];
      op.col_sizes[i] = B.col_sizes[i];
      for (int j = 0; j < 2; ++j)
        if (const MatPtr& m = B.blocks[i][j]) {
          sp[i][j] = m->sparsity()->desc();
          op.sparsity[i][j] = &sp[i][j];
          op.values[i][j] = m->device_values();
        }
    }
  }
};
} // namespace detail

/// solver.hpp:33-58, bitwise equal to the reference.
inline std::vector<Real> block_spmv(const BlockMat& op, std::span<const Real> x) {
  detail::BlockDesc D(op);
  std::unique_ptr<detail::DeviceArray<double>> dx;
  detail::to_device(x, dx);
  detail::DeviceArray<double> y(op.nrows(), false);
  check(loam_gpu_block_spmv(&D.op, dx->dev, (int64_t)x.size(), y.dev, nullptr));
  check(loam_gpu_stream_sync(nullptr));
  return detail::to_host(y, op.nrows());
}

/// Reverse Cuthill-McKee (topology.hpp:131-178) on the device: r[new] = old,
/// bit-identical to the reference; IndexOutOfRange / AsymmetricAdjacency at
/// the first offending entry in list order.
inline std::vector<int> rcm_order(int n, const std::vector<std::vector<int>>& adjacency) {
  require(static_cast<int>(adjacency.size()) == n, ErrorKind::InvalidArgument, "adjacency list count != n");
  std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
  for (int u = 0; u < n; ++u) rp[u + 1] = rp[u] + static_cast<int64_t>(adjacency[u].size());
  std::vector<int32_t> ci;
  ci.reserve(static_cast<size_t>(rp[n]));
  for (const auto& a : adjacency) ci.insert(ci.end(), a.begin(), a.end());
  detail::DeviceArray<int64_t> drp(rp.size(), false);
  detail::DeviceArray<int32_t> dci(ci.size(), false), dout(static_cast<size_t>(n), false);
  drp.upload(rp.data());
  if (!ci.empty()) dci.upload(ci.data());
  check(loam_gpu_rcm_order(n, drp.dev, dci.dev, dout.dev, nullptr));
  const auto& h = dout.download();
  return std::vector<int>(h.begin(), h.begin() + n);
}

struct SolveReport { // solver.hpp:13-18
  int iterations = 0;
  Real final_residual_norm = 0.0;
  bool converged = false;
  enum class Reason { rtol, atol, maxit } reason = Reason::maxit;
};

enum class Preconditioner { None, Jacobi };

namespace detail {
inline SolveReport report_of(const loam_solve_report& r) {
  SolveReport s;
  s.iterations = r.iterations;
  s.final_residual_norm = r.final_residual_norm;
  s.converged = r.converged != 0;
  s.reason = r.reason == 0 ? SolveReport::Reason::rtol
                           : (r.reason == 1 ? SolveReport::Reason::atol : SolveReport::Reason::maxit);
  return s;
}
template <class Call>
std::pair<std::vector<Real>, SolveReport> cg_run(std::span<const Real> b, std::vector<Real> x0, Call&& call) {
  if (x0.empty()) x0.assign(b.size(), 0.0);
  require(x0.size() == b.size(), ErrorKind::DimensionMismatch, "x0 length != rhs length");
  std::unique_ptr<DeviceArray<double>> db, dx;
  to_device(b, db);
  to_device(std::span<const Real>(x0.data(), x0.size()), dx);
  loam_solve_report rep{};
  check(call(db->dev, dx->dev, &rep));
  check(loam_gpu_stream_sync(nullptr));
  dx->host_valid = false;
  return {to_host(*dx, b.size()), report_of(rep)};
}
} // namespace detail

/// Preconditioned CG (solver.hpp:170-188), the iteration on the device.
inline std::pair<std::vector<Real>, SolveReport> cg_solve(const Mat& mat, std::span<const Real> b,
                                                          std::vector<Real> x0 = {}, Real rtol = 1e-8,
                                                          Real atol = 1e-14, int maxit = 1000,
                                                          Preconditioner precond = Preconditioner::None) {
  const loam_sparsity_desc sp = mat.sparsity()->desc();
  return detail::cg_run(b, std::move(x0), [&](const double* db, double* dx, loam_solve_report* rep) {
    return loam_gpu_cg_solve(&sp, mat.device_values(), db, (int64_t)b.size(), dx, rtol, atol, maxit,
                             precond == Preconditioner::Jacobi ? 1 : 0, rep, nullptr);
  });
}

/// CG on a nested block operator over the flattened numbering (solver.hpp:190-207).
inline std::pair<std::vector<Real>, SolveReport> cg_solve(const BlockMat& op, std::span<const Real> b,
                                                          std::vector<Real> x0 = {}, Real rtol = 1e-8,
                                                          Real atol = 1e-14, int maxit = 1000,
                                                          Preconditioner precond = Preconditioner::None) {
  detail::BlockDesc D(op);
  return detail::cg_run(b, std::move(x0), [&](const double* db, double* dx, loam_solve_report* rep) {
    return loam_gpu_cg_solve_block(&D.op, db, (int64_t)b.size(), dx, rtol, atol, maxit,
                                   precond == Preconditioner::Jacobi ? 1 : 0, rep, nullptr);
  });
}

} // namespace loam_gpu
