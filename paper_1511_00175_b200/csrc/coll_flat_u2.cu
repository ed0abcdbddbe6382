// fp32 FLAT kernels with unroll factor U = 2 (see coll_flat.cuh).
#include "coll_flat.cuh"

namespace fc {
FC_FLAT_TABLE(2)
}  // namespace fc
