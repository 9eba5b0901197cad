#!/usr/bin/env python
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/Makefile
built oracle/_ref/libloam_ref.so).  The fixtures let the CPU tests pin the C
restatement (oracle/liborc.so) and the input generator against the reference
on machines where the reference is absent (the GPU box).

Inputs come from the product's seeded generator (paper_1501_01809_b200.configs,
host code only); every fixture stores its inputs next to the reference outputs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1501_01809_b200 import configs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main():
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"
    os.makedirs(OUT, exist_ok=True)
    # reference meshes (mesh.hpp:96-214)
    sq_c, sq_cv = O.ref_unit_mesh(2, 6)
    cu_c, cu_cv = O.ref_unit_mesh(3, 3)
    np.savez_compressed(os.path.join(OUT, "ref_meshes.npz"), sq_coords=sq_c, sq_cv=sq_cv, cube_coords=cu_c, cube_cv=cu_cv)

    # C1-shaped residual (stiffness_action + mass_action, two reference loops)
    m = configs.config_inputs(1, 8)
    b = O.ref_assemble_vector(O.HELMHOLTZ_ACTION, 1, 2, m.cv, m.coords, m.extra["u"], kappa=configs.KAPPA)
    colors, nc = O.color_iteration(m.ncells, [m.cv], [3], [m.nv], lib="ref")
    np.savez_compressed(os.path.join(OUT, "c1_n8.npz"), cv=m.cv, coords=m.coords, u=m.extra["u"], residual=b,
                        colors=colors, ncolors=nc)

    # C2-shaped stiffness CSR (assemble_matrix with the reference's AST kernel)
    m = configs.config_inputs(2, 8)
    rp, ci, vals = O.ref_assemble_matrix(O.STIFFNESS, 1, 2, m.cv, m.coords)
    np.savez_compressed(os.path.join(OUT, "c2_n8.npz"), cv=m.cv, coords=m.coords, row_ptr=rp, col_idx=ci, values=vals)

    # P2 triangle space numbering and Helmholtz matrix (configs 5 velocity space)
    m = configs.config_inputs(5, 4)
    cn, nn = O.ref_p2_tri_map(m.cv, m.coords)
    rp, ci, vals = O.ref_assemble_matrix(O.HELMHOLTZ, 2, 2, m.cv, m.coords, kappa=1.5)
    np.savez_compressed(os.path.join(OUT, "p2tri_n4.npz"), cv=m.cv, coords=m.coords, cn=cn, nn=nn, row_ptr=rp,
                        col_idx=ci, values=vals)

    # P1 tet mass matrix (the reference's only 3D catalogue element) and colouring
    m = configs.config_inputs(4, 3)
    rp, ci, vals = O.ref_assemble_matrix(O.MASS, 1, 3, m.cv, m.coords)
    colors, nc = O.color_iteration(m.ncells, [m.cv], [4], [m.nv], lib="ref")
    np.savez_compressed(os.path.join(OUT, "p1tet_n3.npz"), cv=m.cv, coords=m.coords, row_ptr=rp, col_idx=ci,
                        values=vals, colors=colors, ncolors=nc)

    # dof-expanded sparsity (build_sparsity with row/col dims, data.hpp:149-179)
    rng = np.random.default_rng(7)
    rv = rng.integers(0, 9, 3 * 20).astype(np.int32)
    cvv = rng.integers(0, 7, 2 * 20).astype(np.int32)
    rp, ci = O.build_sparsity(20, rv, 3, 9, cvv, 2, 7, 2, 3, lib="ref")
    np.savez_compressed(os.path.join(OUT, "sparsity_dims.npz"), rv=rv, cv=cvv, row_ptr=rp, col_idx=ci)

    # reference local kernels on one random simplex per element (pipeline of
    # compile_local_kernel -> hoist -> fold -> interpret)
    X2 = np.array([0.1, -0.2, 1.3, 0.05, 0.2, 0.9])
    X3 = np.array([0.0, 0.1, -0.1, 1.1, 0.0, 0.2, 0.1, 0.9, 0.0, 0.05, 0.1, 1.2])
    C3, C6 = np.array([0.3, -0.7, 1.1]), np.array([0.3, -0.7, 1.1, 0.5, -0.2, 0.8])
    ker = {}
    for kind in (O.MASS, O.STIFFNESS, O.HELMHOLTZ, O.MASS_ACTION, O.STIFFNESS_ACTION):
        ker[f"tri_p1_{kind}"] = O.ref_local_kernel(kind, 1, 2, X2, C3, kappa=2.5)
        ker[f"tri_p2_{kind}"] = O.ref_local_kernel(kind, 2, 2, X2, C6, kappa=2.5)
        ker[f"tet_p1_{kind}"] = O.ref_local_kernel(kind, 1, 3, X3, np.append(C3, 0.4), kappa=2.5)
    np.savez_compressed(os.path.join(OUT, "local_kernels.npz"), X2=X2, X3=X3, C3=C3, C6=C6, **ker)
    rcm_fixture()
    print("golden fixtures written to", OUT)


def random_graph(n, m, seed):
    """Seeded symmetric adjacency lists (no self loops), unsorted rows."""
    rng = np.random.default_rng(seed)
    adj = [[] for _ in range(n)]
    for _ in range(m):
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a != b and b not in adj[a]:
            adj[a].append(b)
            adj[b].append(a)
    return adj


def rcm_fixture():
    """rcm_order (topology.hpp:131-178) and reorder (mesh.hpp:364-396) of the
    reference on cell-permuted meshes and seeded random graphs."""
    out = {}
    for tag, gdim, n in (("sq", 2, 6), ("cube", 3, 3)):
        m = configs.mesh(gdim, n, 0.1, 7, 8)
        perm, xo, co = O.ref_reorder(gdim, m.cv, m.coords)
        out.update({f"{tag}_cv": m.cv, f"{tag}_coords": m.coords, f"{tag}_perm": perm, f"{tag}_coords_out": xo,
                    f"{tag}_cv_out": co})
    for k, (n, m_, seed) in enumerate(((40, 50, 1), (200, 300, 2), (64, 20, 3))):
        rp, ci = O._csr_of_lists(random_graph(n, m_, seed))
        out.update({f"g{k}_row_ptr": rp, f"g{k}_col_idx": ci, f"g{k}_order": O.rcm_order((rp, ci), lib="ref")})
    np.savez_compressed(os.path.join(OUT, "rcm.npz"), **out)


if __name__ == "__main__":
    main()
