"""Python mirror of the reference operator surface over the C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/loam): Set/Map (topology.hpp:15-74),
Dat/Global/Sparsity/Mat/build_sparsity (data.hpp:15-234), Arg/arg/Parloop/
validate/execute (parloop.hpp:17-384), color_iteration (topology.hpp:86-125).
Objects are DEVICE-resident (torch CUDA tensors are only the allocator);
every compute call goes through libloam_gpu.so -- there is no CPU path.
Errors raise capi.LoamError whose `.kind` is the reference ErrorKind name.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import capi


def _release(obj_id: int) -> None:
    """Evict a destroyed Map / Sparsity's cached plans (quietly at interpreter exit)."""
    try:
        capi.release_id(obj_id)
    except Exception:  # noqa: BLE001 -- module teardown: nothing left to evict
        pass
from .capi import INC, MAX, MIN, READ, RW, SUM, WRITE, LoamError

class _Ids:
    """Object identities come from the library (loam_gpu_new_id), unique across
    every client in the process (C++ facade, FFI bindings, this mirror)."""

    def __next__(self) -> int:
        return capi.new_id()


_ids = _Ids()


def _fail(kind: str, msg: str):
    raise LoamError(1 + capi.ERROR_KINDS.index(kind), msg)


def _require(cond: bool, kind: str, msg: str) -> None:
    if not cond:
        _fail(kind, msg)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Access:
    READ, WRITE, RW, INC, SUM, MIN, MAX = READ, WRITE, RW, INC, SUM, MIN, MAX


# --------------------------------------------------------------------------- topology


class Set:
    """topology.hpp:15-26: a count only."""

    def __init__(self, size: int, name: str = "set"):
        _require(size >= 0, "InvalidArgument", "Set size must be non-negative")
        self.size = int(size)
        self.name = name
        self.id = next(_ids)


def make_set(size: int, name: str = "set") -> Set:
    return Set(size, name)


class Map:
    """topology.hpp:36-66: int32 row-major [source.size x arity], validated on construction.

    `node_map`/`expand_dim` (extension): a dof-expanded map (entries dim*n+d,
    SURVEY A6) can declare the node map it expands so the device reads the
    smaller node map; see expanded_map().
    """

    def __init__(self, source: Set, target: Set, arity: int, values, name: str = "map",
                 node_map: "Map | None" = None, expand_dim: int = 0):
        _require(arity > 0, "InvalidArgument", "Map arity must be positive")
        vals = np.ascontiguousarray(np.asarray(values, dtype=np.int32).reshape(-1))
        _require(vals.size == source.size * arity, "ArityMismatch",
                 f"{name}: value table length != source size * arity")
        if vals.size:
            lo, hi = int(vals.min()), int(vals.max())
            bad = lo if lo < 0 else hi
            _require(lo >= 0 and hi < target.size, "IndexOutOfRange",
                     f"{name}: map entry {bad} outside target set of size {target.size}")
        self.source, self.target, self.arity, self.name = source, target, int(arity), name
        self.values = vals
        self.dev = torch.from_numpy(vals).cuda() if vals.size else torch.zeros(1, dtype=torch.int32, device="cuda")
        self.id = next(_ids)
        self.node_map = node_map
        self.expand_dim = expand_dim
        self._desc = None

    def row(self, e: int) -> np.ndarray:
        return self.values[e * self.arity:(e + 1) * self.arity]

    def node_level(self, dim: int = 1):
        """(identity, dof dim) at node level: a dof-expanded map stands for its node map."""
        if self.node_map is not None and self.expand_dim > 1:
            return self.node_map.id, dim * self.expand_dim
        return self.id, dim

    def __del__(self):
        try:
            _release(getattr(self, "id", 0))
        except Exception:  # noqa: BLE001 -- interpreter teardown: module globals already gone
            pass

    def desc(self) -> capi.MapDesc:
        if self._desc is None:
            d = capi.MapDesc()
            d.values = self.dev.data_ptr()
            d.source_size, d.target_size, d.arity = self.source.size, self.target.size, self.arity
            d.source_id, d.target_id, d.id = self.source.id, self.target.id, self.id
            if self.node_map is not None:
                d.expand_dim = self.expand_dim
                d.node_values = self.node_map.dev.data_ptr()
                d.node_arity = self.node_map.arity
                d.node_target_size = self.node_map.target.size
                d.node_id = self.node_map.id
            self._desc = d
        return self._desc


def make_map(source: Set, target: Set, arity: int, values, name: str = "map") -> Map:
    return Map(source, target, arity, values, name)


def expanded_map(node_map: Map, dim: int, target: Set | None = None, name: str = "dof_map") -> Map:
    """The dof-expanded Map a vector-valued Mat needs (entries dim*n+d)."""
    if target is None:
        target = Set(node_map.target.size * dim, name + "_dofs")
    v = node_map.values.reshape(-1, node_map.arity).astype(np.int64)
    exp = (v[:, :, None] * dim + np.arange(dim)[None, None, :]).reshape(-1).astype(np.int32)
    return Map(node_map.source, target, node_map.arity * dim, exp, name, node_map=node_map, expand_dim=dim)


def color_iteration(iterset: Set, conflict_maps: Sequence[Map]):
    """topology.hpp:86-125 on the device: returns (colors ndarray, num_colors)."""
    for m in conflict_maps:
        _require(m.source is iterset, "SourceMismatch",
                 f"conflict map {m.name} source differs from iteration set")
    n = iterset.size
    colors = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    descs = (capi.MapDesc * max(len(conflict_maps), 1))(*[m.desc() for m in conflict_maps])
    nc = C.c_int32(0)
    capi.check(capi.lib().loam_gpu_color_iteration(n, iterset.id, descs, len(conflict_maps),
                                                    colors.data_ptr(), C.byref(nc), _stream()))
    return colors[:n].cpu().numpy(), int(nc.value)


# --------------------------------------------------------------------------- data


class Dat:
    """data.hpp:35-60: fp64 AoS [set.size x dim] with a version counter."""

    def __init__(self, set_: Set, dim: int, name: str = "dat"):
        _require(dim > 0, "InvalidArgument", "Dat dim must be positive")
        self.set, self.dim, self.name = set_, int(dim), name
        self.data = torch.zeros(max(set_.size * dim, 1), dtype=torch.float64, device="cuda")
        self.version = 0
        self.id = next(_ids)
        self._zero = True    # logically zero-initialised (make_dat, data.hpp:37-39)
        self._stale = False  # zero() deferred: memory not cleared yet

    def _materialize(self) -> None:
        if self._stale:
            self.data.zero_()
            self._stale = False

    def view(self) -> np.ndarray:
        self._materialize()
        return self.data[: self.set.size * self.dim].cpu().numpy()

    def set_values(self, values) -> None:
        """mutable_view() + assignment: bumps the version (data.hpp:49-52)."""
        v = torch.as_tensor(np.asarray(values, dtype=np.float64).reshape(-1))
        _require(v.numel() == self.set.size * self.dim, "DimensionMismatch", "value count mismatch")
        self.version += 1
        self.data[: v.numel()].copy_(v.cuda())
        self._zero = self._stale = False

    def zero(self) -> None:
        """Lazy: the next INC through the device treats the Dat as zeros
        (LOAM_ARG_ZERO); the memory is cleared only if something reads it."""
        self.version += 1
        self._zero = self._stale = True


def make_dat(set_: Set, dim: int, name: str = "dat") -> Dat:
    return Dat(set_, dim, name)


class Global:
    """data.hpp:69-87."""

    def __init__(self, dim: int = 1, name: str = "global", init=None):
        if init is not None:
            init = list(init)
            dim = len(init)
        _require(dim > 0, "InvalidArgument", "Global dim must be positive")
        self.dim, self.name = int(dim), name
        self.data = torch.zeros(self.dim, dtype=torch.float64, device="cuda")
        if init is not None:
            self.data.copy_(torch.tensor(init, dtype=torch.float64))
        self.id = next(_ids)

    def view(self) -> np.ndarray:
        return self.data.cpu().numpy()

    def set_values(self, values) -> None:
        self.data.copy_(torch.as_tensor(np.asarray(values, dtype=np.float64)))


def make_global(dim: int = 1, name: str = "global") -> Global:
    return Global(dim, name)


class Sparsity:
    """data.hpp:116-142: CSR with int64 row offsets and int32 columns (device)."""

    def __init__(self, nrows: int, ncols: int, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                 row_dim: int = 1, col_dim: int = 1, built_from=None):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr, self.col_idx = row_ptr, col_idx
        self.row_dim, self.col_dim = row_dim, col_dim
        # node-level (row map id, row dim, col map id, col dim) it was built from
        self.built_from = built_from
        self.id = next(_ids)
        self._host = None
        self._desc = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[self.nrows].item())

    def host(self):
        if self._host is None:
            self._host = (self.row_ptr.cpu().numpy(), self.col_idx[: max(self.nnz, 0)].cpu().numpy())
        return self._host

    def find(self, row: int, col: int) -> int:
        """Position of (row, col) in the values array or -1 (data.hpp:129-136)."""
        if row < 0 or row >= self.nrows:
            return -1
        rp, ci = self.host()
        lo, hi = int(rp[row]), int(rp[row + 1])
        k = lo + int(np.searchsorted(ci[lo:hi], col))
        return k if k < hi and ci[k] == col else -1

    def desc(self) -> capi.SparsityDesc:
        if self._desc is None:
            d = capi.SparsityDesc()
            d.row_ptr, d.col_idx = self.row_ptr.data_ptr(), self.col_idx.data_ptr()
            d.nrows, d.ncols, d.nnz = self.nrows, self.ncols, self.nnz
            d.row_dim, d.col_dim, d.id = self.row_dim, self.col_dim, self.id
            if self.built_from is not None:
                d.pattern_row_map, d.pattern_row_dim, d.pattern_col_map, d.pattern_col_dim = self.built_from
            self._desc = d
        return self._desc

    def __del__(self):
        try:
            _release(getattr(self, "id", 0))
        except Exception:  # noqa: BLE001 -- interpreter teardown: module globals already gone
            pass


def build_sparsity(row_map: Map, col_map: Map, row_dim: int = 1, col_dim: int = 1) -> Sparsity:
    """data.hpp:149-179 on the device (bit-exact)."""
    rp, ci, nnz = C.c_void_p(), C.c_void_p(), C.c_int64()
    capi.check(capi.lib().loam_gpu_build_sparsity(row_map.desc(), col_map.desc(), row_dim, col_dim,
                                                   C.byref(rp), C.byref(ci), C.byref(nnz), _stream()))
    nrows = row_map.target.size * row_dim
    ncols = col_map.target.size * col_dim
    try:  # copy into torch-owned storage, release the library allocation
        row_ptr = torch.empty(nrows + 1, dtype=torch.int64, device="cuda")
        col_idx = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
        capi.check(capi.lib().loam_gpu_memcpy(row_ptr.data_ptr(), rp, 8 * (nrows + 1), _stream()))
        capi.check(capi.lib().loam_gpu_memcpy(col_idx.data_ptr(), ci, 4 * nnz.value, _stream()))
        capi.check(capi.lib().loam_gpu_stream_sync(_stream()))
    finally:
        capi.lib().loam_gpu_free(rp)
        capi.lib().loam_gpu_free(ci)
    return Sparsity(nrows, ncols, row_ptr, col_idx, row_dim, col_dim,
                    built_from=(*row_map.node_level(row_dim), *col_map.node_level(col_dim)))


class Mat:
    """data.hpp:183-228: fp64 values over a fixed sparsity, zero-initialised."""

    def __init__(self, sparsity: Sparsity, name: str = "mat"):
        self.sparsity, self.name = sparsity, name
        self.values = torch.zeros(max(sparsity.nnz, 1), dtype=torch.float64, device="cuda")
        self.id = next(_ids)
        self._zero = True    # make_mat zero-fills (data.hpp:185-187)
        self._stale = False

    def _materialize(self) -> None:
        if self._stale:
            self.values.zero_()
            self._stale = False

    @property
    def nrows(self):
        return self.sparsity.nrows

    @property
    def ncols(self):
        return self.sparsity.ncols

    def host_values(self) -> np.ndarray:
        self._materialize()
        return self.values[: self.sparsity.nnz].cpu().numpy()

    def at(self, row: int, col: int) -> float:
        self._materialize()
        pos = self.sparsity.find(row, col)
        return 0.0 if pos < 0 else float(self.values[pos].item())

    def zero(self) -> None:
        """Lazy Mat::zero (data.hpp:201): the next INC treats the values as zeros."""
        self._zero = self._stale = True


def make_mat(sparsity: Sparsity, name: str = "mat") -> Mat:
    return Mat(sparsity, name)


# --------------------------------------------------------------------------- par_loop


@dataclass
class Arg:
    """parloop.hpp:17-28."""
    dat: Optional[Dat] = None
    mat: Optional[Mat] = None
    glob: Optional[Global] = None
    access: int = READ
    maps: list = field(default_factory=list)


def arg(obj, access: int, map1: Map | None = None, map2: Map | None = None) -> Arg:
    """arg(dat, access, map=None) | arg(mat, access, row_map, col_map) | arg(global, access)."""
    if isinstance(obj, Dat):
        return Arg(dat=obj, access=access, maps=[map1] if map1 is not None else [])
    if isinstance(obj, Mat):
        return Arg(mat=obj, access=access, maps=[map1, map2])
    if isinstance(obj, Global):
        return Arg(glob=obj, access=access)
    raise TypeError("arg() expects a Dat, Mat or Global")


@dataclass
class Kernel:
    """ir::Kernel (kernel.hpp:504-511) as a registry key plus its baked literals."""
    name: str
    params: tuple = ()

    def signature(self):
        buf = (C.c_int32 * 64)()
        n = capi.lib().loam_gpu_kernel_signature(self.name.encode(), buf, 64)
        if n < 0:
            raise LoamError(-n, capi.lib().loam_gpu_last_error().decode())
        out, w = [], 0
        for _ in range(n):
            rank = buf[w]
            out.append(list(buf[w + 1:w + 1 + rank]))
            w += 1 + rank
        return out


def kernel(name: str, *params: float) -> Kernel:
    return Kernel(name, tuple(float(p) for p in params))


@dataclass
class Parloop:
    """parloop.hpp:55-59."""
    kernel: Kernel
    iterset: Set
    args: list


def _build(loop: Parloop):
    keep = []
    descs = (capi.ArgDesc * max(len(loop.args), 1))()
    for k, a in enumerate(loop.args):
        d = descs[k]
        d.access = a.access
        if a.dat is not None:
            d.kind, d.data, d.dim = capi.ARG_DAT, a.dat.data.data_ptr(), a.dat.dim
            d.set_size, d.set_id, d.obj_id = a.dat.set.size, a.dat.set.id, a.dat.id
            if a.access == INC and a.dat._zero:
                d.flags = capi.ARG_ZERO  # the device zero-fills only if its path needs it
            else:
                a.dat._materialize()
            _require(len(a.maps) <= 1, "InvalidArgument", "Dat argument with several maps")
            if a.maps:
                md = a.maps[0].desc()
                keep.append(md)
                d.map = C.pointer(md)
        elif a.mat is not None:
            d.kind, d.data, d.obj_id = capi.ARG_MAT, a.mat.values.data_ptr(), a.mat.id
            if a.mat._zero:
                d.flags = capi.ARG_ZERO
            else:
                a.mat._materialize()
            _require(len(a.maps) == 2 and all(m is not None for m in a.maps), "InvalidArgument",
                     "Mat argument requires row and column maps")
            r, c, s = a.maps[0].desc(), a.maps[1].desc(), a.mat.sparsity.desc()
            keep += [r, c, s]
            d.map, d.col_map, d.sparsity = C.pointer(r), C.pointer(c), C.pointer(s)
        elif a.glob is not None:
            d.kind, d.data, d.dim, d.obj_id = capi.ARG_GLOBAL, a.glob.data.data_ptr(), a.glob.dim, a.glob.id
        else:
            _fail("InvalidArgument", "argument must target exactly one object")
    params = (C.c_double * max(len(loop.kernel.params), 1))(*loop.kernel.params)
    kd = capi.KernelDesc(loop.kernel.name.encode(), params, len(loop.kernel.params))
    keep += [params, kd]
    return kd, descs, keep


class HostLoop:
    """A par_loop over HOST memory through loam_gpu_execute_host -- the
    reference's calling convention (execute reads and writes host buffers,
    parloop.hpp:191).  Every object's data is mirrored into (pinned) host
    arrays; Maps and the Sparsity keep their ids, so the library uploads them
    once and keeps them resident (they are immutable in the reference); Dats
    are copied on every call.  ``outputs`` holds the host arrays the loop
    writes; ``h2d_bytes`` / ``d2h_bytes`` count the per-call Dat transfers.
    """

    def __init__(self, loop: Parloop, pin: bool = True, mirrors: Optional[dict] = None):
        self.loop = loop
        self._keep, self.outputs = [], []
        self.h2d_bytes = self.d2h_bytes = 0
        kd, dev_descs, keep = _build(loop)
        self._keep += [kd, keep]
        self.kd = kd
        self.descs = (capi.ArgDesc * max(len(loop.args), 1))()

        # one host mirror per object: an id must name one host buffer.  Loops
        # that run in one call (run_host_blocks) share `mirrors`, so an object
        # they all read (the coordinates) is one host array, uploaded once.
        mirrors = {} if mirrors is None else mirrors

        def host(t) -> torch.Tensor:
            key = (id(t), t.data_ptr() if isinstance(t, torch.Tensor) else t.ctypes.data)
            if key in mirrors:
                return mirrors[key]
            mirrors[key] = h = host_copy(t)
            return h

        def host_copy(t) -> torch.Tensor:
            if isinstance(t, np.ndarray):
                h = torch.from_numpy(np.ascontiguousarray(t))
            else:
                h = t.detach().cpu().contiguous()
            h = h.pin_memory() if pin else h
            self._keep.append(h)
            return h

        maps = {}

        def host_map(m: Map) -> capi.MapDesc:
            if m.id in maps:
                return maps[m.id]
            md = capi.MapDesc()
            C.memmove(C.byref(md), C.byref(m.desc()), C.sizeof(md))
            md.values = host(m.values).data_ptr()
            if m.node_map is not None:
                md.node_values = host(m.node_map.values).data_ptr()
            self._keep.append(md)
            maps[m.id] = md
            return md

        for k, a in enumerate(loop.args):
            d = capi.ArgDesc()
            C.memmove(C.byref(d), C.byref(dev_descs[k]), C.sizeof(d))
            if a.dat is not None:
                h = host(a.dat.data)
                d.data = h.data_ptr()
                if a.maps:
                    d.map = C.pointer(host_map(a.maps[0]))
                if a.access != READ:
                    self.outputs.append(h)
                    self.d2h_bytes += h.numel() * 8
                if a.access != WRITE and not (d.flags & capi.ARG_ZERO):
                    self.h2d_bytes += h.numel() * 8
            elif a.mat is not None:
                h = host(a.mat.values[: max(a.mat.sparsity.nnz, 1)])
                d.data = h.data_ptr()
                sp = capi.SparsityDesc()
                C.memmove(C.byref(sp), C.byref(a.mat.sparsity.desc()), C.sizeof(sp))
                sp.row_ptr = host(a.mat.sparsity.row_ptr).data_ptr()
                sp.col_idx = host(a.mat.sparsity.col_idx).data_ptr()
                self._keep.append(sp)
                d.sparsity = C.pointer(sp)
                d.map, d.col_map = C.pointer(host_map(a.maps[0])), C.pointer(host_map(a.maps[1]))
                self.outputs.append(h)
                self.d2h_bytes += a.mat.sparsity.nnz * 8
                if not (d.flags & capi.ARG_ZERO):
                    self.h2d_bytes += a.mat.sparsity.nnz * 8
            else:
                h = host(a.glob.data)
                d.data = h.data_ptr()
                self.h2d_bytes += h.numel() * 8
                if a.access != READ:
                    self.outputs.append(h)
                    self.d2h_bytes += h.numel() * 8
            self.descs[k] = d

    def run(self, stream: Optional[int] = None) -> None:
        capi.check(capi.lib().loam_gpu_execute_host(C.byref(self.kd), self.loop.iterset.size,
                                                    self.loop.iterset.id, self.descs, len(self.loop.args),
                                                    _stream() if stream is None else stream))

    def step_buffers(self):
        """A second argument array for loam_gpu_execute_host_batch: the same
        maps and sparsity host mirrors, its own pinned Dat / Mat / Global
        buffers (copies of this loop's).  Returns (descs, outputs)."""
        n = len(self.loop.args)
        descs = (capi.ArgDesc * max(n, 1))()
        outs = []
        for k in range(n):
            d = capi.ArgDesc()
            C.memmove(C.byref(d), C.byref(self.descs[k]), C.sizeof(d))
            nbytes = self._arg_bytes(k)
            h = torch.empty(max(nbytes // 8, 1), dtype=torch.float64).pin_memory()
            C.memmove(h.data_ptr(), d.data, nbytes)
            self._keep.append(h)
            d.data = h.data_ptr()
            if self.loop.args[k].access != READ:
                outs.append(h)
            descs[k] = d
        self._keep.append(descs)
        return descs, outs

    def _arg_bytes(self, k: int) -> int:
        a = self.loop.args[k]
        if a.dat is not None:
            return a.dat.set.size * a.dat.dim * 8
        if a.mat is not None:
            return a.mat.sparsity.nnz * 8
        return a.glob.data.numel() * 8

    def run_batch(self, step_descs, stream: Optional[int] = None) -> None:
        """loam_gpu_execute_host_batch over the argument arrays `step_descs`
        (this loop's own and/or step_buffers() ones), pipelined copies."""
        arr = (C.POINTER(capi.ArgDesc) * len(step_descs))(
            *[C.cast(d, C.POINTER(capi.ArgDesc)) for d in step_descs])
        capi.check(capi.lib().loam_gpu_execute_host_batch(
            C.byref(self.kd), self.loop.iterset.size, self.loop.iterset.id, arr, len(self.loop.args),
            len(step_descs), _stream() if stream is None else stream))


def run_host_blocks(host_loops, stream: Optional[int] = None) -> None:
    """fem::assemble_blocks (fem/assemble.hpp:439-448) under the host-memory
    calling convention: the HostLoops' par_loops in one
    loam_gpu_execute_blocks_host call (build them with a shared `mirrors`)."""
    hl = list(host_loops)
    arr = (capi.LoopDesc * max(len(hl), 1))()
    for i, h in enumerate(hl):
        arr[i].kernel = C.pointer(h.kd)
        arr[i].iterset_size = h.loop.iterset.size
        arr[i].iterset_id = h.loop.iterset.id
        arr[i].args = C.cast(h.descs, C.POINTER(capi.ArgDesc))
        arr[i].nargs = len(h.loop.args)
    capi.check(capi.lib().loam_gpu_execute_blocks_host(arr, len(hl), _stream() if stream is None else stream))


def validate(loop: Parloop) -> None:
    """parloop.hpp:89-146: descriptor checks only, no state change."""
    kd, descs, keep = _build(loop)
    capi.check(capi.lib().loam_gpu_validate(C.byref(kd), loop.iterset.size, loop.iterset.id, descs,
                                            len(loop.args)))


def execute(loop: Parloop, threads: int = 1) -> None:
    """parloop.hpp:191: `threads` is accepted for drop-in compatibility (the device decides)."""
    _require(threads >= 1, "InvalidArgument", "thread count must be positive")
    kd, descs, keep = _build(loop)
    capi.check(capi.lib().loam_gpu_execute(C.byref(kd), loop.iterset.size, loop.iterset.id, descs,
                                           len(loop.args), _stream()))
    for a in loop.args:  # written objects: version bump (data.hpp:49-52), no longer known zero
        if a.access != READ:
            if a.dat is not None:
                a.dat.version += 1
                a.dat._zero = a.dat._stale = False
            if a.mat is not None:
                a.mat._zero = a.mat._stale = False


def execute_blocks(loops) -> None:
    """The par_loops of fem::assemble_blocks (fem/assemble.hpp:439-448) in one
    call: every loop validated first, then run in order -- the Taylor-Hood
    Stokes triple as one fused launch (loam_gpu_execute_blocks)."""
    loops = list(loops)
    built = [_build(lp) for lp in loops]
    arr = (capi.LoopDesc * max(len(loops), 1))()
    for i, (lp, (kd, descs, keep)) in enumerate(zip(loops, built)):
        arr[i].kernel = C.pointer(kd)
        arr[i].iterset_size = lp.iterset.size
        arr[i].iterset_id = lp.iterset.id
        arr[i].args = C.cast(descs, C.POINTER(capi.ArgDesc))
        arr[i].nargs = len(lp.args)
    capi.check(capi.lib().loam_gpu_execute_blocks(arr, len(loops), _stream()))
    for lp in loops:
        for a in lp.args:
            if a.access != READ:
                if a.dat is not None:
                    a.dat.version += 1
                    a.dat._zero = a.dat._stale = False
                if a.mat is not None:
                    a.mat._zero = a.mat._stale = False


# --------------------------------------------------------------------------
# Consumers of the assembled matrix: data.hpp:236-250,
# solver.hpp:13-207, on the device through the C ABI.

def mat_spmv(mat: Mat, x) -> torch.Tensor:
    """y = A x (data.hpp:236-250), bitwise equal to the reference's CSR fold."""
    mat._materialize()
    xt = torch.as_tensor(np.asarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x,
                         dtype=torch.float64).to("cuda").contiguous()
    y = torch.empty(max(mat.nrows, 1), dtype=torch.float64, device="cuda")
    capi.check(capi.lib().loam_gpu_spmv(mat.sparsity.desc(), mat.values.data_ptr(), xt.data_ptr(), xt.numel(),
                                        y.data_ptr(), _stream()))
    return y[: mat.nrows]


class BlockMat:
    """solver.hpp:21-28: 2x2 table of blocks; None is a zero block."""

    def __init__(self, blocks=None, row_sizes=(0, 0), col_sizes=(0, 0)):
        self.blocks = [[None, None], [None, None]] if blocks is None else [list(r) for r in blocks]
        self.row_sizes, self.col_sizes = list(row_sizes), list(col_sizes)

    @property
    def nrows(self):
        return sum(self.row_sizes)

    @property
    def ncols(self):
        return sum(self.col_sizes)

    def desc(self):
        d = capi.BlockMatDesc()
        keep = []
        for i in range(2):
            d.row_sizes[i], d.col_sizes[i] = self.row_sizes[i], self.col_sizes[i]
            for j in range(2):
                m = self.blocks[i][j]
                if m is not None:
                    m._materialize()
                    sd = m.sparsity.desc()
                    keep.append(sd)
                    d.sparsity[i][j] = C.pointer(sd)
                    d.values[i][j] = m.values.data_ptr()
        return d, keep


def _vec(x, n=None) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
    return t.to(device="cuda", dtype=torch.float64).contiguous()


def block_spmv(op: BlockMat, x) -> torch.Tensor:
    """solver.hpp:33-58, bitwise equal to the reference's nested fold."""
    xt = _vec(x)
    y = torch.empty(max(op.nrows, 1), dtype=torch.float64, device="cuda")
    d, keep = op.desc()
    capi.check(capi.lib().loam_gpu_block_spmv(C.byref(d), xt.data_ptr(), xt.numel(), y.data_ptr(), _stream()))
    return y[: op.nrows]


class SolveReport:
    """solver.hpp:13-18."""
    REASONS = ("rtol", "atol", "maxit")

    def __init__(self, r: capi.SolveReportDesc):
        self.iterations = int(r.iterations)
        self.final_residual_norm = float(r.final_residual_norm)
        self.converged = bool(r.converged)
        self.reason = self.REASONS[int(r.reason)]


class Preconditioner:
    NONE, JACOBI = 0, 1


def cg_solve(op, b, x0=None, rtol: float = 1e-8, atol: float = 1e-14, maxit: int = 1000,
             precond: int = Preconditioner.NONE):
    """solver.hpp:170-207 (Mat or BlockMat): returns (x, SolveReport)."""
    bt = _vec(b)
    n = bt.numel()
    if x0 is not None and len(x0) != 0:
        _require(len(x0) == n, "DimensionMismatch", "x0 length != rhs length")  # solver.hpp:90
    x = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda") if x0 is None or len(x0) == 0 else _vec(x0).clone()
    rep = capi.SolveReportDesc()
    if isinstance(op, BlockMat):
        d, keep = op.desc()
        capi.check(capi.lib().loam_gpu_cg_solve_block(C.byref(d), bt.data_ptr(), n, x.data_ptr(), rtol, atol,
                                                      maxit, precond, C.byref(rep), _stream()))
    else:
        op._materialize()
        capi.check(capi.lib().loam_gpu_cg_solve(op.sparsity.desc(), op.values.data_ptr(), bt.data_ptr(), n,
                                                x.data_ptr(), rtol, atol, maxit, precond, C.byref(rep), _stream()))
    return x[:n], SolveReport(rep)


# --------------------------------------------------------------------------
# Around the assembly loop: pointwise expressions
# (fem/assemble.hpp:150-319), Dirichlet conditions (fem/bc.hpp,
# fem/assemble.hpp:54-81) and norms, on the device through the C ABI.

class Pw:
    """fem/assemble.hpp:150-205 PwNode tree: constants, Dat fields, + - * / and negation."""

    def __init__(self, kind: str, value: float = 0.0, field: "Dat | None" = None, a=None, b=None):
        self.kind, self.value, self.field, self.a, self.b = kind, float(value), field, a, b

    def __add__(self, o): return Pw("add", a=self, b=_as_pw(o))
    def __radd__(self, o): return Pw("add", a=_as_pw(o), b=self)
    def __sub__(self, o): return Pw("sub", a=self, b=_as_pw(o))
    def __rsub__(self, o): return Pw("sub", a=_as_pw(o), b=self)
    def __mul__(self, o): return Pw("mul", a=self, b=_as_pw(o))
    def __rmul__(self, o): return Pw("mul", a=_as_pw(o), b=self)
    def __truediv__(self, o): return Pw("div", a=self, b=_as_pw(o))
    def __rtruediv__(self, o): return Pw("div", a=_as_pw(o), b=self)
    def __neg__(self): return Pw("neg", a=self)

    def fields(self, out: list) -> list:
        """collect_fields (assemble.hpp:209-220): first-appearance order, unique."""
        if self.kind == "field":
            if not any(f is self.field for f in out):
                out.append(self.field)
        for c in (self.a, self.b):
            if c is not None:
                c.fields(out)
        return out

    def program(self, slot) -> list:
        """Postfix program (left subtree, right subtree, operator)."""
        if self.kind == "const":
            return [(capi.PW_CONST, 0, self.value)]
        if self.kind == "field":
            return [(capi.PW_FIELD, slot(self.field), 0.0)]
        if self.kind == "neg":
            return self.a.program(slot) + [(capi.PW_NEG, 0, 0.0)]
        op = {"add": capi.PW_ADD, "sub": capi.PW_SUB, "mul": capi.PW_MUL, "div": capi.PW_DIV}[self.kind]
        return self.a.program(slot) + self.b.program(slot) + [(op, 0, 0.0)]


def _as_pw(x) -> Pw:
    return x if isinstance(x, Pw) else pw(x)


def pw(x) -> Pw:
    """fem::pw(Real) / fem::pw(DatPtr)."""
    if isinstance(x, Dat):
        return Pw("field", field=x)
    return Pw("const", value=float(x))


class PwOp:
    ASSIGN, ADD, SUB = capi.PW_ASSIGN, capi.PW_ADD_TO, capi.PW_SUB_FROM


def pointwise(out: Dat, op: int, expr) -> None:
    """fem::pointwise (assemble.hpp:252-314): out (=|+=|-=) expr at every node
    and component; every field lives on out's set with out's dim
    (SpaceMismatch otherwise).  Bitwise equal to the reference."""
    expr = _as_pw(expr)
    fields = expr.fields([])
    for f in fields:
        _require(f.set is out.set, "SpaceMismatch", "pointwise fields must share the output's set")
        _require(f.dim == out.dim, "SpaceMismatch", "pointwise fields must share the output's component count")
    inputs = [f for f in fields if f is not out]
    prog = expr.program(lambda f: -1 if f is out else next(i for i, g in enumerate(inputs) if g is f))
    arr = (capi.PwInstr * len(prog))(*[capi.PwInstr(o, fi, v) for o, fi, v in prog])
    for f in fields:
        f._materialize()
    out._materialize()
    ptrs = (C.c_void_p * max(len(inputs), 1))(*[f.data.data_ptr() for f in inputs])
    capi.check(capi.lib().loam_gpu_pointwise(out.data.data_ptr(), out.set.size * out.dim, op, arr, len(prog),
                                             ptrs, len(inputs), _stream()))
    out.version += 1
    out._zero = out._stale = False


class DirichletBC:
    """fem/bc.hpp:11-27: strong condition on `nodes` (sorted) of a scalar node
    set, value = `constant` or a Dat `function` on that set."""

    def __init__(self, node_set: Set, nodes, constant: float = 0.0, function: "Dat | None" = None):
        if function is not None:
            _require(function.set is node_set, "SpaceMismatch", "bc value must live on the constrained space")
        self.node_set, self.constant, self.function = node_set, float(constant), function
        self.nodes = np.unique(np.asarray(nodes, dtype=np.int32))
        self._dev = torch.as_tensor(self.nodes).cuda()

    def value_at(self, node: int) -> float:
        return float(self.function.view()[node]) if self.function is not None else self.constant

    def _values(self):
        if self.function is None:
            return None
        self.function._materialize()
        return self.function.data.data_ptr()

    def apply(self, dat: Dat) -> None:
        """bc.apply(b) (bc.hpp:21-26)."""
        _require(dat.set is self.node_set, "SpaceMismatch", "bc applied to a vector on a different node set")
        dat._materialize()
        capi.check(capi.lib().loam_gpu_bc_apply(dat.data.data_ptr(), dat.set.size, self._dev.data_ptr(),
                                                len(self.nodes), self._values(), self.constant, _stream()))
        dat.version += 1
        dat._zero = dat._stale = False


def apply_dirichlet(A: Mat, b: "Dat | None", bc: DirichletBC) -> None:
    """fem/assemble.hpp:54-66 (b None: apply_dirichlet_rows, :69-79)."""
    _require(b is None or A.nrows == bc.node_set.size, "ShapeMismatch", "matrix is not square on the bc space")
    A._materialize()
    if b is not None:
        b._materialize()
    capi.check(capi.lib().loam_gpu_apply_dirichlet(A.sparsity.desc(), A.values.data_ptr(),
                                                   b.data.data_ptr() if b is not None else None,
                                                   bc._dev.data_ptr(), len(bc.nodes), bc._values(), bc.constant,
                                                   _stream()))
    A._zero = A._stale = False
    if b is not None:
        b.version += 1
        b._zero = b._stale = False


def apply_dirichlet_rows(A: Mat, bc: DirichletBC) -> None:
    apply_dirichlet(A, None, bc)


def reduce(x, kind: int) -> float:
    """Deterministic device reduction (SUM / MIN / MAX / MAX_ABS) of a Dat or tensor."""
    if isinstance(x, Dat):
        x._materialize()
        t, n = x.data, x.set.size * x.dim
    else:
        t = _vec(x)
        n = t.numel()
    r = C.c_double()
    capi.check(capi.lib().loam_gpu_reduce(t.data_ptr(), n, kind, C.byref(r), _stream()))
    return r.value


def inf_norm(x) -> float:
    return reduce(x, capi.REDUCE_MAX_ABS)


# --------------------------------------------------------------------------
# Mesh-side builders on the device.

def p2_cell_node_map(cell_vertex: Map, gdim: int):
    """fem/space.hpp:48-72 on the device: (node Set, cell->node Map) of the P2
    space over a simplex mesh's cell->vertex map."""
    nc, nv = cell_vertex.source.size, cell_vertex.target.size
    nn = 6 if gdim == 2 else 10
    cn = torch.empty(max(nc * nn, 1), dtype=torch.int32, device="cuda")
    out = C.c_int32()
    capi.check(capi.lib().loam_gpu_p2_cell_node_map_dev(nc, nv, gdim, cell_vertex.dev.data_ptr(), cn.data_ptr(),
                                                        C.byref(out), _stream()))
    nodes = Set(out.value, "p2_nodes")
    return nodes, Map(cell_vertex.source, nodes, nn, cn[: nc * nn].cpu().numpy(), "cell_node")


def exterior_facets(cell_vertex: Map, gdim: int):
    """mesh.hpp:48-89 derive_exterior_facets (no markers) on the device:
    (facet_vertices [n x gdim], facet_cell [n x 2]) as numpy arrays."""
    nc, nv = cell_vertex.source.size, cell_vertex.target.size
    fv, fc, n = C.c_void_p(), C.c_void_p(), C.c_int32()
    capi.check(capi.lib().loam_gpu_exterior_facets(nc, nv, gdim, cell_vertex.dev.data_ptr(), C.byref(fv),
                                                   C.byref(fc), C.byref(n), _stream()))
    k = n.value
    a = np.empty(max(k * gdim, 1), np.int32)
    b = np.empty(max(k * 2, 1), np.int32)
    try:
        capi.check(capi.lib().loam_gpu_memcpy(a.ctypes.data, fv, a.nbytes, None))
        capi.check(capi.lib().loam_gpu_memcpy(b.ctypes.data, fc, b.nbytes, None))
    finally:
        capi.lib().loam_gpu_free(fv)
        capi.lib().loam_gpu_free(fc)
    return a[: k * gdim].reshape(k, gdim), b[: k * 2].reshape(k, 2)


def vertex_adjacency(cell_vertex: Map, gdim: int):
    """mesh.hpp:350-362 on the device: (row_ptr int64, col_idx int32) device
    tensors, per vertex the sorted other vertices that share a cell."""
    nc, nv = cell_vertex.source.size, cell_vertex.target.size
    rp, ci, nnz = C.c_void_p(), C.c_void_p(), C.c_int64()
    capi.check(capi.lib().loam_gpu_vertex_adjacency(nc, nv, gdim, cell_vertex.dev.data_ptr(), C.byref(rp),
                                                    C.byref(ci), C.byref(nnz), _stream()))
    try:
        trp = torch.empty(nv + 1, dtype=torch.int64, device="cuda")
        tci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
        capi.check(capi.lib().loam_gpu_memcpy(trp.data_ptr(), rp, 8 * (nv + 1), _stream()))
        capi.check(capi.lib().loam_gpu_memcpy(tci.data_ptr(), ci, 4 * nnz.value, _stream()))
        capi.check(capi.lib().loam_gpu_stream_sync(_stream()))
    finally:
        capi.lib().loam_gpu_free(rp)
        capi.lib().loam_gpu_free(ci)
    return trp, tci[: nnz.value]


def rcm_order(n: int, row_ptr, col_idx) -> torch.Tensor:
    """topology.hpp:131-178 rcm_order on the device over CSR adjacency lists
    (numpy or device tensors); returns perm (int32 device tensor),
    perm[new] = old.  Raises LoamError(IndexOutOfRange / AsymmetricAdjacency)
    like the reference."""
    rp = torch.as_tensor(np.asarray(row_ptr, np.int64) if isinstance(row_ptr, (list, np.ndarray)) else row_ptr)
    ci = torch.as_tensor(np.asarray(col_idx, np.int32) if isinstance(col_idx, (list, np.ndarray)) else col_idx)
    rp = rp.to(device="cuda", dtype=torch.int64).contiguous()
    ci = ci.to(device="cuda", dtype=torch.int32).contiguous()
    # the reference rejects a list count != n (InvalidArgument); here the
    # offsets must also fit the column array (the device checks monotonicity)
    if rp.numel() != n + 1 or (n > 0 and int(rp[-1].item()) > ci.numel()):
        raise capi.LoamError(1 + capi.ERROR_KINDS.index("InvalidArgument"), "adjacency list count != n")
    if ci.numel() == 0:
        ci = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    capi.check(capi.lib().loam_gpu_rcm_order(n, rp.data_ptr(), ci.data_ptr(), out.data_ptr(), _stream()))
    return out[:n]


def reorder(cell_vertex: Map, coordinates: Dat):
    """mesh.hpp:364-396 reorder on the device: RCM over the vertex adjacency,
    then coordinates and the cell->vertex map renumbered consistently.
    Returns (new cell_vertex Map, new coordinates Dat, perm) with
    perm[new] = old (numpy).  Exterior facets keep their (cell, local facet)
    order under the renumbering (cells are not permuted), as the reference
    requires; re-derive them with exterior_facets(new_map, gdim)."""
    gdim = coordinates.dim
    nv, nc = cell_vertex.target.size, cell_vertex.source.size
    _require(cell_vertex.arity == gdim + 1, "ArityMismatch", "cell_vertex arity must be gdim + 1")
    _require(coordinates.set.size == nv, "DimensionMismatch",
             "coordinates must live on the map's target set")
    rp, ci = vertex_adjacency(cell_vertex, gdim)
    perm = rcm_order(nv, rp, ci)
    coordinates._materialize()
    verts = Set(nv, cell_vertex.target.name)
    X = Dat(verts, gdim, coordinates.name)
    cv_out = torch.empty(max(nc * (gdim + 1), 1), dtype=torch.int32, device="cuda")
    capi.check(capi.lib().loam_gpu_renumber_vertices(nv, gdim, coordinates.data.data_ptr(), nc,
                                                     cell_vertex.dev.data_ptr(), perm.data_ptr(),
                                                     X.data.data_ptr(), cv_out.data_ptr(), _stream()))
    X.version += 1
    X._zero = X._stale = False
    cvals = cv_out[: nc * (gdim + 1)].cpu().numpy()
    m = Map(cell_vertex.source, verts, gdim + 1, cvals, cell_vertex.name)
    return m, X, perm.cpu().numpy()
