// fp32 FLAT kernels with unroll factor U = 1 (see coll_flat.cuh).
#include "coll_flat.cuh"

namespace fc {
FC_FLAT_TABLE(1)
}  // namespace fc
