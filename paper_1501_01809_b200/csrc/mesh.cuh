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
