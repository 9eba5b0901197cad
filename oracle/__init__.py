"""Oracle package -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the
timed CPU baseline.  The product (paper_1501_01809_b200/) never imports it.

  orc()  -> liborc.so            : C restatement of the reference algorithm
  ref()  -> _ref/libloam_ref.so  : the unmodified reference headers compiled
                                   by oracle/Makefile (extern "C" shim)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libloam_ref.so")

# orc_form numbering (loam_oracle.h)
MASS, STIFFNESS, HELMHOLTZ, MASS_ACTION, STIFFNESS_ACTION, HELMHOLTZ_ACTION = range(6)
ELASTICITY, STOKES_A, STOKES_B, STOKES_BT = 6, 7, 8, 9

_orc = _ref = None
IP, DP = C.POINTER(C.c_int32), C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)


def ip(a):
    return a.ctypes.data_as(IP)


def dp(a):
    return None if a is None else a.ctypes.data_as(DP)


def orc():
    global _orc
    if _orc is None:
        L = C.CDLL(ORC_PATH)
        L.orc_color_iteration.argtypes = [C.c_int, C.c_int, C.POINTER(IP), IP, IP, IP]
        L.orc_build_sparsity.restype = C.c_int64
        L.orc_build_sparsity.argtypes = [C.c_int, IP, C.c_int, C.c_int, IP, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.POINTER(I64P), C.POINTER(IP)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_p2_cell_node_map.argtypes = [C.c_int, C.c_int, C.c_int, IP, IP]
        L.orc_element.argtypes = [C.c_int, C.c_int, C.c_int, DP, DP, DP, DP]
        L.orc_element_shape.argtypes = [C.c_int, C.c_int, C.c_int, IP, IP]
        L.orc_assemble_vector.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, IP, C.c_int, IP, DP,
                                          IP, C.c_int, DP, C.c_int, DP]
        L.orc_assemble_matrix.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, IP, C.c_int, IP,
                                          C.c_int, IP, DP, C.c_int, I64P, IP, DP]
        VPP = C.POINTER(C.c_void_p)
        L.orc_block_spmv.argtypes = [IP, IP, VPP, VPP, VPP, DP, DP]
        L.orc_cg.argtypes = [IP, IP, VPP, VPP, VPP, C.c_int, DP, DP, C.c_double, C.c_double, C.c_int, C.c_int,
                             IP, DP, IP]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_unit_square_mesh.argtypes = [C.c_int, DP, IP]
        L.ref_unit_cube_mesh.argtypes = [C.c_int, DP, IP]
        L.ref_color_iteration.argtypes = [C.c_int, C.c_int, C.POINTER(IP), IP, IP, IP]
        L.ref_build_sparsity.restype = C.c_int64
        L.ref_build_sparsity.argtypes = [C.c_int, IP, C.c_int, C.c_int, IP, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.POINTER(I64P), C.POINTER(IP)]
        L.ref_p2_tri_map.argtypes = [C.c_int, C.c_int, IP, DP, IP]
        L.ref_local_kernel.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, DP, DP, DP]
        L.ref_assemble_vector.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, IP, DP,
                                          DP, C.c_int, DP, IP]
        L.ref_assemble_matrix.restype = C.c_int64
        L.ref_assemble_matrix.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, IP, DP,
                                          C.c_int, IP, C.POINTER(I64P), C.POINTER(IP), C.POINTER(DP)]
        L.ref_engine_matrix.restype = C.c_int64
        L.ref_engine_matrix.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, IP, C.c_int, C.c_int, IP,
                                        C.c_int, C.c_int, IP, C.c_int, DP, C.c_int, C.POINTER(I64P),
                                        C.POINTER(IP), C.POINTER(DP)]
        L.ref_engine_vector.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, IP, C.c_int, C.c_int, IP,
                                        C.c_int, DP, DP, C.c_int, DP]
        L.ref_time_execute.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, C.c_int, IP, DP, DP,
                                       C.c_int, C.c_int, C.c_int, C.c_int, DP]
        VPP = C.POINTER(C.c_void_p)
        L.ref_spmv.argtypes = [C.c_int, C.c_int, I64P, IP, DP, DP, C.c_int64, DP]
        L.ref_block_spmv.argtypes = [IP, IP, VPP, VPP, VPP, DP, C.c_int64, DP]
        L.ref_cg_solve.argtypes = [C.c_int, IP, IP, VPP, VPP, VPP, DP, C.c_int64, DP, C.c_int64, C.c_double,
                                   C.c_double, C.c_int, C.c_int, IP, DP]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    pass


def _check(code, lib=None):
    if code != 0:
        msg = lib.ref_last_error().decode() if lib is not None else ""
        raise OracleError(f"oracle error {code}: {msg}")


def _params(params):
    p = np.zeros(4)
    p[: len(params)] = params
    return p


# ---------------------------------------------------------------- C restatement wrappers
def color_iteration(n, maps, arities, targets, lib="orc"):
    maps = [np.ascontiguousarray(m, dtype=np.int32) for m in maps]
    arr = (IP * max(len(maps), 1))(*[ip(m) for m in maps])
    ar = np.asarray(arities, dtype=np.int32)
    tg = np.asarray(targets, dtype=np.int32)
    colors = np.empty(max(n, 1), dtype=np.int32)
    if lib == "orc":
        nc = orc().orc_color_iteration(n, len(maps), arr, ip(ar), ip(tg), ip(colors))
    else:
        nc = ref().ref_color_iteration(n, len(maps), arr, ip(ar), ip(tg), ip(colors))
    if nc < 0:
        raise OracleError(f"colouring failed ({-nc})")
    return colors[:n], nc


def build_sparsity(nsrc, row_map, ar_r, nrt, col_map, ar_c, nct, row_dim=1, col_dim=1, lib="orc"):
    rm = np.ascontiguousarray(row_map, dtype=np.int32)
    cm = np.ascontiguousarray(col_map, dtype=np.int32)
    rp, ci = I64P(), IP()
    L = orc() if lib == "orc" else ref()
    fn = L.orc_build_sparsity if lib == "orc" else L.ref_build_sparsity
    nnz = fn(nsrc, ip(rm), ar_r, nrt, ip(cm), ar_c, nct, row_dim, col_dim, C.byref(rp), C.byref(ci))
    if nnz < 0:
        raise OracleError(f"build_sparsity failed ({-nnz})")
    nrows = nrt * row_dim
    row_ptr = np.ctypeslib.as_array(rp, shape=(nrows + 1,)).copy()
    col_idx = np.ctypeslib.as_array(ci, shape=(max(nnz, 1),))[:nnz].copy()
    free = L.orc_free if lib == "orc" else L.ref_free
    free(C.cast(rp, C.c_void_p))
    free(C.cast(ci, C.c_void_p))
    return row_ptr, col_idx


def p2_cell_node_map(cv, nv, gdim):
    cv = np.ascontiguousarray(cv, dtype=np.int32)
    nc = cv.size // (gdim + 1)
    cn = np.empty(nc * (6 if gdim == 2 else 10), dtype=np.int32)
    nn = orc().orc_p2_cell_node_map(nc, nv, gdim, ip(cv), ip(cn))
    return cn, nn


def element(form, degree, gdim, X, C_=None, params=()):
    r, c = C.c_int32(), C.c_int32()
    _check(orc().orc_element_shape(form, degree, gdim, C.byref(r), C.byref(c)))
    out = np.zeros(r.value * c.value)
    X = np.ascontiguousarray(X, dtype=np.float64)
    Cc = None if C_ is None else np.ascontiguousarray(C_, dtype=np.float64)
    _check(orc().orc_element(form, degree, gdim, dp(_params(params)), dp(X), dp(Cc), dp(out)))
    return out.reshape(r.value, c.value)


def assemble_vector(form, degree, gdim, ncells, test_map, ar_t, coord_map, coords, coeff_map, ar_c,
                    coeff, nout, params=()):
    out = np.zeros(nout)
    tm = np.ascontiguousarray(test_map, dtype=np.int32)
    xm = np.ascontiguousarray(coord_map, dtype=np.int32)
    cm = np.ascontiguousarray(coeff_map, dtype=np.int32)
    _check(orc().orc_assemble_vector(form, degree, gdim, dp(_params(params)), ncells, ip(tm), ar_t,
                                     ip(xm), dp(np.ascontiguousarray(coords)), ip(cm), ar_c,
                                     dp(np.ascontiguousarray(coeff)), nout, dp(out)))
    return out


def assemble_matrix(form, degree, gdim, ncells, row_map, ar_r, col_map, ar_c, coord_map, coords,
                    row_ptr, col_idx, params=()):
    nrows = row_ptr.size - 1
    vals = np.zeros(max(int(row_ptr[-1]), 1))
    rm = np.ascontiguousarray(row_map, dtype=np.int32)
    cm = np.ascontiguousarray(col_map, dtype=np.int32)
    xm = np.ascontiguousarray(coord_map, dtype=np.int32)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    code = orc().orc_assemble_matrix(form, degree, gdim, dp(_params(params)), ncells, ip(rm), ar_r, ip(cm),
                                     ar_c, ip(xm), dp(np.ascontiguousarray(coords)), nrows,
                                     rp.ctypes.data_as(I64P), ip(ci), dp(vals))
    _check(code)
    return vals[: int(row_ptr[-1])]


# ---------------------------------------------------------------- reference (compiled) wrappers
def ref_unit_mesh(gdim, n):
    if gdim == 2:
        coords, cv = np.empty((n + 1) ** 2 * 2), np.empty(2 * n * n * 3, dtype=np.int32)
        _check(ref().ref_unit_square_mesh(n, dp(coords), ip(cv)), ref())
    else:
        coords, cv = np.empty((n + 1) ** 3 * 3), np.empty(6 * n ** 3 * 4, dtype=np.int32)
        _check(ref().ref_unit_cube_mesh(n, dp(coords), ip(cv)), ref())
    return coords, cv


def ref_p2_tri_map(cv, coords):
    cv = np.ascontiguousarray(cv, dtype=np.int32)
    nc, nv = cv.size // 3, coords.size // 2
    cn = np.empty(nc * 6, dtype=np.int32)
    nn = ref().ref_p2_tri_map(nc, nv, ip(cv), dp(np.ascontiguousarray(coords)), ip(cn))
    if nn < 0:
        raise OracleError(ref().ref_last_error().decode())
    return cn, nn


def ref_local_kernel(kind, degree, gdim, X, C_=None, kappa=0.0):
    nb = (gdim + 1) if degree == 1 else (6 if gdim == 2 else 10)
    bil = kind in (MASS, STIFFNESS, HELMHOLTZ)
    out = np.zeros(nb * nb if bil else nb)
    Cc = np.zeros(nb) if C_ is None else np.ascontiguousarray(C_, dtype=np.float64)
    _check(ref().ref_local_kernel(kind, degree, gdim, kappa, dp(np.ascontiguousarray(X, dtype=np.float64)),
                                  dp(Cc), dp(out)), ref())
    return out.reshape(nb, nb) if bil else out


def ref_assemble_vector(kind, degree, gdim, cv, coords, coeff, kappa=1.0, threads=1):
    cv = np.ascontiguousarray(cv, dtype=np.int32)
    nc, nv = cv.size // (gdim + 1), coords.size // gdim
    out = np.zeros(max(coeff.size, nv))
    nout = C.c_int32()
    _check(ref().ref_assemble_vector(kind, degree, gdim, kappa, nc, nv, ip(cv), dp(np.ascontiguousarray(coords)),
                                     dp(np.ascontiguousarray(coeff)), threads, dp(out), C.byref(nout)), ref())
    return out[: nout.value]


def ref_assemble_matrix(kind, degree, gdim, cv, coords, kappa=1.0, threads=1):
    cv = np.ascontiguousarray(cv, dtype=np.int32)
    nc, nv = cv.size // (gdim + 1), coords.size // gdim
    nrows = C.c_int32()
    rp, ci, vals = I64P(), IP(), DP()
    nnz = ref().ref_assemble_matrix(kind, degree, gdim, kappa, nc, nv, ip(cv), dp(np.ascontiguousarray(coords)),
                                    threads, C.byref(nrows), C.byref(rp), C.byref(ci), C.byref(vals))
    if nnz < 0:
        raise OracleError(ref().ref_last_error().decode())
    out = (np.ctypeslib.as_array(rp, shape=(nrows.value + 1,)).copy(),
           np.ctypeslib.as_array(ci, shape=(max(nnz, 1),))[:nnz].copy(),
           np.ctypeslib.as_array(vals, shape=(max(nnz, 1),))[:nnz].copy())
    for p in (rp, ci, vals):
        ref().ref_free(C.cast(p, C.c_void_p))
    return out


def ref_engine_matrix(form, degree, gdim, ncells, row_map, ar_r, nrt, col_map, ar_c, nct, coord_map,
                      coords, params=(), threads=1):
    rm = np.ascontiguousarray(row_map, dtype=np.int32)
    cm = rm if col_map is row_map else np.ascontiguousarray(col_map, dtype=np.int32)
    xm = np.ascontiguousarray(coord_map, dtype=np.int32)
    nv = coords.size // gdim
    rp, ci, vals = I64P(), IP(), DP()
    nnz = ref().ref_engine_matrix(form, degree, gdim, dp(_params(params)), ncells, ip(rm), ar_r, nrt, ip(cm),
                                  ar_c, nct, ip(xm), nv, dp(np.ascontiguousarray(coords)), threads,
                                  C.byref(rp), C.byref(ci), C.byref(vals))
    if nnz < 0:
        raise OracleError(ref().ref_last_error().decode())
    nrows = nrt
    out = (np.ctypeslib.as_array(rp, shape=(nrows + 1,)).copy(),
           np.ctypeslib.as_array(ci, shape=(max(nnz, 1),))[:nnz].copy(),
           np.ctypeslib.as_array(vals, shape=(max(nnz, 1),))[:nnz].copy())
    for p in (rp, ci, vals):
        ref().ref_free(C.cast(p, C.c_void_p))
    return out


def ref_engine_vector(form, degree, gdim, ncells, test_map, ar_t, nt, coord_map, coords, coeff,
                      params=(), threads=1):
    tm = np.ascontiguousarray(test_map, dtype=np.int32)
    xm = np.ascontiguousarray(coord_map, dtype=np.int32)
    out = np.zeros(nt)
    _check(ref().ref_engine_vector(form, degree, gdim, dp(_params(params)), ncells, ip(tm), ar_t, nt, ip(xm),
                                   coords.size // gdim, dp(np.ascontiguousarray(coords)),
                                   dp(np.ascontiguousarray(coeff)), threads, dp(out)), ref())
    return out


def ref_time_execute(form, degree, gdim, cv, coords, coeff=None, params=(), as_shipped=True, threads=1,
                     warmup=1, steps=3):
    cv = np.ascontiguousarray(cv, dtype=np.int32)
    nc, nv = cv.size // (gdim + 1), coords.size // gdim
    times = np.zeros(steps)
    _check(ref().ref_time_execute(form, degree, gdim, dp(_params(params)), nc, nv, ip(cv),
                                  dp(np.ascontiguousarray(coords)),
                                  None if coeff is None else dp(np.ascontiguousarray(coeff)),
                                  int(as_shipped), threads, warmup, steps, dp(times)), ref())
    return times


# ------------------------------------------- consumers of the assembled matrix
# A CSR operand is (nrows, ncols, row_ptr int64, col_idx int32, values f64); a
# nested operator is a 2x2 list of CSR operands or None (zero block) with
# row_sizes / col_sizes (solver.hpp:21-28).
KINDS = ["IndexOutOfRange", "ArityMismatch", "SourceMismatch", "AsymmetricAdjacency", "IllegalAccess",
         "MapSourceMismatch", "ShapeMismatch", "UnboundIdentifier", "NonDividingFactor", "OutsideSparsity",
         "EmptyPartials", "DimensionMismatch", "InvalidSubdivision", "ParseError", "NonManifold", "CellMismatch",
         "UnsupportedForm", "MissingDiagonal", "SpaceMismatch", "IndefiniteBreakdown", "InstabilityDetected",
         "InvalidArgument"]


class KindError(OracleError):
    def __init__(self, code, msg=""):
        self.kind = KINDS[code - 1] if 1 <= code <= len(KINDS) else str(code)
        super().__init__(f"{self.kind}: {msg}")


def _blocks(blocks, row_sizes, col_sizes):
    keep = []
    rp, ci, v = (C.c_void_p * 4)(), (C.c_void_p * 4)(), (C.c_void_p * 4)()
    for i in range(2):
        for j in range(2):
            b = blocks[i][j]
            if b is None:
                continue
            _, _, r, c, vals = b
            r, c, vals = (np.ascontiguousarray(r, np.int64), np.ascontiguousarray(c, np.int32),
                          np.ascontiguousarray(vals, np.float64))
            keep += [r, c, vals]
            rp[2 * i + j], ci[2 * i + j], v[2 * i + j] = r.ctypes.data, c.ctypes.data, vals.ctypes.data
    rs = np.array(row_sizes, np.int32)
    cs = np.array(col_sizes, np.int32)
    keep += [rs, cs]
    return rs, cs, rp, ci, v, keep


def _plain(csr):
    return [[csr, None], [None, None]], (csr[0], 0), (csr[1], 0)


def block_spmv(blocks, row_sizes, col_sizes, x):
    """orc_block_spmv (data.hpp:236-250, solver.hpp:33-58)."""
    rs, cs, rp, ci, v, keep = _blocks(blocks, row_sizes, col_sizes)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(int(rs.sum()))
    orc().orc_block_spmv(ip(rs), ip(cs), rp, ci, v, dp(x), dp(y))
    return y


def spmv(csr, x):
    return block_spmv(*_plain(csr), x)


def cg(op, b, x0=None, rtol=1e-8, atol=1e-14, maxit=1000, jacobi=False, nested=None):
    """orc_cg (solver.hpp:80-207).  op: CSR operand or (blocks, row_sizes, col_sizes)."""
    if nested is None:
        nested = isinstance(op, tuple) and len(op) == 3
    blocks, rsz, csz = op if nested else _plain(op)
    rs, cs, rp, ci, v, keep = _blocks(blocks, rsz, csz)
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros(len(b)) if x0 is None else np.array(x0, np.float64)
    rep = np.zeros(3, np.int32)
    rn = np.zeros(1)
    fail = np.zeros(1, np.int32)
    L = orc()
    rc = L.orc_cg(ip(rs), ip(cs), rp, ci, v, int(nested), dp(b), dp(x), C.c_double(rtol), C.c_double(atol),
                  int(maxit), int(jacobi), ip(rep), dp(rn), ip(fail))
    if rc:
        raise KindError(rc, f"fail={int(fail[0])}")
    return x, {"iterations": int(rep[0]), "converged": bool(rep[1]), "reason": ("rtol", "atol", "maxit")[rep[2]],
               "final_residual_norm": float(rn[0])}


def ref_block_spmv(blocks, row_sizes, col_sizes, x):
    """The compiled reference's block_spmv (solver.hpp:33-58)."""
    rs, cs, rp, ci, v, keep = _blocks(blocks, row_sizes, col_sizes)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(max(int(rs.sum()), 1))
    L = ref()
    rc = L.ref_block_spmv(ip(rs), ip(cs), rp, ci, v, dp(x), C.c_int64(len(x)), dp(y))
    if rc:
        raise KindError(rc, L.ref_last_error().decode())
    return y[: int(rs.sum())]


def ref_spmv(csr, x):
    """The compiled reference's mat_spmv (data.hpp:236-250)."""
    n, m, r, c, vals = csr
    r, c, vals = np.ascontiguousarray(r, np.int64), np.ascontiguousarray(c, np.int32), np.ascontiguousarray(vals)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(max(n, 1))
    L = ref()
    rc = L.ref_spmv(int(n), int(m), r.ctypes.data_as(I64P), ip(c), dp(vals), dp(x), C.c_int64(len(x)), dp(y))
    if rc:
        raise KindError(rc, L.ref_last_error().decode())
    return y[:n]


def ref_cg(op, b, x0=None, rtol=1e-8, atol=1e-14, maxit=1000, jacobi=False, nested=None):
    """The compiled reference's cg_solve (solver.hpp:170-207)."""
    if nested is None:
        nested = isinstance(op, tuple) and len(op) == 3
    blocks, rsz, csz = op if nested else _plain(op)
    rs, cs, rp, ci, v, keep = _blocks(blocks, rsz, csz)
    b = np.ascontiguousarray(b, np.float64)
    x = np.zeros(len(b)) if x0 is None else np.array(x0, np.float64)
    oi = np.zeros(3, np.int32)
    od = np.zeros(1)
    L = ref()
    rc = L.ref_cg_solve(int(nested), ip(rs), ip(cs), rp, ci, v, dp(b), C.c_int64(len(b)), dp(x),
                        C.c_int64(len(x)), C.c_double(rtol), C.c_double(atol), int(maxit), int(jacobi), ip(oi), dp(od))
    if rc:
        raise KindError(rc, L.ref_last_error().decode())
    return x, {"iterations": int(oi[0]), "converged": bool(oi[1]), "reason": ("rtol", "atol", "maxit")[oi[2]],
               "final_residual_norm": float(od[0])}


# ------------------------------------------- around the assembly loop (8f-2, 8f-3)
# A pointwise program is a list of (op, field, value) postfix instructions
# (include/loam_gpu.h loam_pw_opcode; field -1 = the output).

def _program(prog):
    ops = np.array([p[0] for p in prog], np.int32)
    fidx = np.array([p[1] for p in prog], np.int32)
    vals = np.array([p[2] for p in prog], np.float64)
    return ops, fidx, vals


def _ptrs(arrays):
    arrs = [np.ascontiguousarray(a, np.float64) for a in arrays]
    return arrs, (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])


def pointwise(prog, assign, out, fields, lib="orc"):
    """orc_pointwise / the compiled reference's fem::pointwise (assemble.hpp:252-314).
    Returns the new out (a copy); `out` may be 2-D [size, dim] for the reference."""
    out = np.array(out, np.float64)
    ops, fidx, vals = _program(prog)
    arrs, ptrs = _ptrs(fields)
    if lib == "orc":
        rc = orc().orc_pointwise(dp(out.reshape(-1)), C.c_int64(out.size), C.c_int(assign), ip(ops), ip(fidx),
                                 dp(vals), C.c_int(len(prog)), ptrs)
        _check(rc)
    else:
        size, dim = (out.shape[0], out.shape[1]) if out.ndim == 2 else (out.size, 1)
        L = ref()
        rc = L.ref_pointwise(C.c_int(size), C.c_int(dim), C.c_int(assign), ip(ops), ip(fidx), dp(vals),
                             C.c_int(len(prog)), C.c_int(len(arrs)), ptrs, dp(out.reshape(-1)))
        if rc:
            raise KindError(rc, L.ref_last_error().decode())
    return out


def apply_dirichlet(csr, rhs, nodes, node_values=None, constant=0.0, lib="orc"):
    """orc_apply_dirichlet / the compiled reference's fem::apply_dirichlet(_rows)
    (assemble.hpp:54-79).  csr = (nrows, ncols, row_ptr, col_idx, values).
    Returns (values, rhs) copies (rhs None: rows only); raises KindError."""
    n, m, r, c, v = csr
    r, c = np.ascontiguousarray(r, np.int64), np.ascontiguousarray(c, np.int32)
    v = np.array(v, np.float64)
    b = None if rhs is None else np.array(rhs, np.float64)
    nodes = np.ascontiguousarray(nodes, np.int32)
    nv = None if node_values is None else np.ascontiguousarray(node_values, np.float64)
    vp = lambda a: None if a is None else C.c_void_p(a.ctypes.data)  # noqa: E731
    if lib == "orc":
        fail = np.zeros(1, np.int32)
        rc = orc().orc_apply_dirichlet(C.c_int(n), vp(r), vp(c), vp(v), vp(b), vp(nodes), C.c_int(len(nodes)),
                                       vp(nv), C.c_double(constant), vp(fail))
        if rc:
            raise KindError(rc, f"row {int(fail[0])}")
    else:
        L = ref()
        rc = L.ref_apply_dirichlet(C.c_int(n), vp(r), vp(c), vp(v), vp(b), vp(nodes), C.c_int(len(nodes)), vp(nv),
                                   C.c_double(constant))
        if rc:
            raise KindError(rc, L.ref_last_error().decode())
    return v, b


def ref_run_wave(n, dt, T, cap=64):
    """The compiled reference's bench::run_wave (bench.hpp:222-300): samples
    every 100 steps as rows (t, |p|_inf, |phi|_inf, energy)."""
    L = ref()
    if not hasattr(L, "ref_run_wave"):
        raise OracleError("reference built without bench.hpp (json.hpp missing)")
    out = np.zeros((cap, 4))
    ns = np.zeros(1, np.int32)
    rc = L.ref_run_wave(C.c_int(n), C.c_double(dt), C.c_double(T), C.c_int(cap), dp(out.reshape(-1)), ip(ns))
    if rc:
        raise KindError(rc, L.ref_last_error().decode())
    return out[: int(ns[0])]


def ref_exterior_facets(gdim, cv, nv):
    """The compiled reference's derive_exterior_facets (mesh.hpp:48-89):
    (facet_vertices [n x gdim], facet_cell [n x 2])."""
    L = ref()
    cv = np.ascontiguousarray(cv, np.int32)
    fv, fc = C.c_void_p(), C.c_void_p()
    n = L.ref_exterior_facets(C.c_int(gdim), C.c_int(cv.size // (gdim + 1)), C.c_int(nv), ip(cv),
                              C.byref(fv), C.byref(fc))
    if n < 0:
        raise KindError(-n, L.ref_last_error().decode())
    a = np.ctypeslib.as_array(C.cast(fv, C.POINTER(C.c_int32)), shape=(max(n, 1) * gdim,))[: n * gdim].copy()
    b = np.ctypeslib.as_array(C.cast(fc, C.POINTER(C.c_int32)), shape=(max(n, 1) * 2,))[: n * 2].copy()
    L.ref_free(fv)
    L.ref_free(fc)
    return a.reshape(n, gdim), b.reshape(n, 2)


# ------------------------------------------- vertex renumbering (8f-4: RCM)
def _csr_of_lists(adj):
    rp = np.zeros(len(adj) + 1, np.int64)
    rp[1:] = np.cumsum([len(a) for a in adj])
    ci = np.array([v for a in adj for v in a], np.int32) if rp[-1] else np.zeros(0, np.int32)
    return rp, ci


def rcm_order(adj, lib="orc"):
    """rcm_order (topology.hpp:131-178).  adj: list of neighbour lists or a CSR
    (row_ptr, col_idx).  lib="orc": the C restatement; "ref": the compiled
    reference.  Raises KindError(1 + ErrorKind) like the reference."""
    rp, ci = adj if isinstance(adj, tuple) else _csr_of_lists(adj)
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int32)
    n = rp.size - 1
    out = np.zeros(max(n, 1), np.int32)
    if lib == "orc":
        L = orc()
        fail = np.zeros(1, np.int64)
        rc = L.orc_rcm_order(C.c_int(n), rp.ctypes.data_as(I64P), ip(ci), ip(out), fail.ctypes.data_as(I64P))
        if rc:
            raise KindError(rc, f"entry {int(fail[0])}")
    else:
        L = ref()
        rc = L.ref_rcm_order(C.c_int(n), rp.ctypes.data_as(I64P), ip(ci), ip(out))
        if rc:
            raise KindError(-rc, L.ref_last_error().decode())
    return out[:n]


def vertex_adjacency(cv, nv, gdim):
    """mesh.hpp:350-362: sorted other vertices sharing a cell, as CSR."""
    cv = np.asarray(cv, np.int32).reshape(-1, gdim + 1)
    nb = [set() for _ in range(nv)]
    for row in cv:
        for a in row:
            nb[a].update(int(b) for b in row if b != a)
    return _csr_of_lists([sorted(s) for s in nb])


def ref_reorder(gdim, cv, coords):
    """The compiled reference's reorder (mesh.hpp:364-396): (perm, coords, cv)."""
    L = ref()
    cv = np.ascontiguousarray(cv, np.int32)
    coords = np.ascontiguousarray(coords, np.float64)
    nv = coords.size // gdim
    perm = np.zeros(max(nv, 1), np.int32)
    xo = np.zeros(max(coords.size, 1))
    co = np.zeros(max(cv.size, 1), np.int32)
    rc = L.ref_reorder(C.c_int(gdim), C.c_int(cv.size // (gdim + 1)), C.c_int(nv), ip(cv), dp(coords),
                       ip(perm), dp(xo), ip(co))
    if rc:
        raise KindError(-rc, L.ref_last_error().decode())
    return perm[:nv], xo[: coords.size], co[: cv.size]


# ------------------------------------------- seeded synthetic inputs (bench --impl reference)
# BASELINE.json configs[0..4]; the same constants as paper_1501_01809_b200/configs.py
# (tests/test_oracle_cpu.py checks both generators produce identical bits), kept
# here so the reference arm never loads the product library.
FULL = {1: 512, 2: 1024, 3: 64, 4: 96, 5: 768}
JITTER = {1: (0.2, 0), 2: (0.2, 2), 3: (0.15, 4), 4: (0.1, 6), 5: (0.2, 7)}
PERM_SEED = {1: 1, 2: 3, 3: 5, 4: None, 5: 8}


class Inputs:
    def __init__(self, gdim, n, coords, cv):
        self.gdim, self.n, self.coords, self.cv, self.extra = gdim, n, coords, cv, {}

    @property
    def nv(self):
        return self.coords.size // self.gdim

    @property
    def ncells(self):
        return self.cv.size // (self.gdim + 1)


def _gen_protos():
    L = orc()
    if not getattr(L, "_gen", False):
        L.orc_unit_square_mesh.argtypes = [C.c_int, DP, IP]
        L.orc_unit_cube_mesh.argtypes = [C.c_int, DP, IP]
        L.orc_jitter.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, DP]
        L.orc_permute_cells.argtypes = [C.c_int, C.c_int, C.c_uint64, IP]
        L.orc_uniform.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_double, DP]
        L._gen = True
    return L


def mesh(gdim, n, amp=0.0, jitter_seed=None, perm_seed=None):
    L = _gen_protos()
    if gdim == 2:
        coords, cv = np.empty((n + 1) ** 2 * 2), np.empty(2 * n * n * 3, dtype=np.int32)
        _check(L.orc_unit_square_mesh(n, dp(coords), ip(cv)))
    else:
        coords, cv = np.empty((n + 1) ** 3 * 3), np.empty(6 * n ** 3 * 4, dtype=np.int32)
        _check(L.orc_unit_cube_mesh(n, dp(coords), ip(cv)))
    if jitter_seed is not None and amp:
        _check(L.orc_jitter(gdim, n, amp, jitter_seed, dp(coords)))
    if perm_seed is not None:
        _check(L.orc_permute_cells(cv.size // (gdim + 1), gdim + 1, perm_seed, ip(cv)))
    return Inputs(gdim, n, coords, cv)


def uniform(count, seed, lo, hi):
    out = np.empty(count)
    _check(_gen_protos().orc_uniform(count, seed, lo, hi, dp(out)))
    return out


def inputs(cfg, n=None):
    """BASELINE config `cfg` (1..5) at size n (default full), generated by the restatement."""
    n = FULL[cfg] if n is None else n
    gdim = 3 if cfg in (3, 4) else 2
    amp, js = JITTER[cfg]
    m = mesh(gdim, n, amp, js, PERM_SEED[cfg])
    if cfg == 1:
        m.extra["u"] = uniform(m.nv, 1000, 0.0, 1.0)
    if cfg in (3, 5):
        m.extra["p2"], m.extra["nn"] = p2_cell_node_map(m.cv, m.nv, gdim)
    if cfg == 3:
        m.extra["u"] = uniform(m.extra["nn"], 1002, -1.0, 1.0)
    return m


def dof_map(nodes, arity, dim):
    v = np.asarray(nodes, np.int64).reshape(-1, arity)
    return (v[:, :, None] * dim + np.arange(dim)).reshape(-1).astype(np.int32)


def ref_time_engine(form, degree, gdim, ncells, row_map, ar_r, nrt, col_map, ar_c, nct, coord_map, coords,
                    coeff=None, params=(), threads=1, warmup=1, steps=3):
    """The compiled reference ENGINE (build_sparsity + execute + addto) with the
    restated host kernel (kernel.hpp:523-529) on arbitrary maps: per-step
    seconds of zero + execute, and the build_sparsity seconds (matrices)."""
    L = ref()
    L.ref_time_engine.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, IP, C.c_int, C.c_int, IP, C.c_int,
                                  C.c_int, IP, C.c_int, DP, DP, C.c_int, C.c_int, C.c_int, DP, DP]
    rm = np.ascontiguousarray(row_map, dtype=np.int32)
    cm = rm if col_map is None else np.ascontiguousarray(col_map, dtype=np.int32)
    xm = np.ascontiguousarray(coord_map, dtype=np.int32)
    times = np.zeros(steps)
    sp = np.zeros(1)
    _check(L.ref_time_engine(form, degree, gdim, dp(_params(params)), ncells, ip(rm), ar_r, nrt,
                             None if col_map is None else ip(cm), ar_c, nct, ip(xm), coords.size // gdim,
                             dp(np.ascontiguousarray(coords)),
                             None if coeff is None else dp(np.ascontiguousarray(coeff)),
                             threads, warmup, steps, dp(times), dp(sp)), L)
    return times, float(sp[0])
