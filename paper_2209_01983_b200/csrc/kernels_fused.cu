// kernels_fused.cu -- fused z-marching kernels (not yet implemented).
#include <cuda_runtime.h>

#include "sale_mesh.cuh"

namespace sale {

bool fused_available() { return false; }

int launch_lagrange_fused(const Slab&, const Phys&, int, Stream) { return 0; }
int launch_remap_fused(const Slab&, const Phys&, int, Stream) { return 0; }

}  // namespace sale
