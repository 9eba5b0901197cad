// mesh.cuh -- host interface of mesh.cu (device P2 numbering, exterior facets).
#pragma once
#include "common.cuh"

namespace loam_gpu {

// fem/space.hpp:48-72 on the device; cn: [ncells x (gd == 2 ? 6 : 10)]; returns the node count.
int p2_cell_node_map_dev(const int32_t* cv, int ncells, int nverts, int gd, int32_t* cn, cudaStream_t s);
// mesh.hpp:48-89 derive_exterior_facets (no markers) on the device; allocates
// *fverts [n x gd] and *fcell [n x 2] (cudaMalloc); returns n.
int exterior_facets_dev(const int32_t* cv, int ncells, int nverts, int gd, int32_t** fverts, int32_t** fcell,
                        cudaStream_t s);

} // namespace loam_gpu

namespace loam_gpu {

// topology.hpp:127-178 rcm_order on the device, bit-exact: adjacency lists
// as CSR (rp [n+1], ci), out[new] = old.  IndexOutOfRange /
// AsymmetricAdjacency at the first offending entry in CSR order (order.cu).
void rcm_order_dev(int n, const int64_t* rp, const int32_t* ci, int32_t* out, cudaStream_t s);
// mesh.hpp:350-362 vertex_adjacency: the cell-vertex sparsity without the
// diagonal (sorted rows); allocates *rp [nverts+1], *ci; returns the entry count.
int64_t vertex_adjacency_dev(const int32_t* cv, int ncells, int nverts, int gd, int64_t** rp, int32_t** ci,
                             cudaStream_t s);
// mesh.hpp:369-386: coords_out[new] = coords[perm[new]], cv_out = new_of[cv].
void renumber_vertices_dev(int nverts, int gd, const double* coords, int ncells, const int32_t* cv,
                           const int32_t* perm, double* coords_out, int32_t* cv_out, cudaStream_t s);

} // namespace loam_gpu
