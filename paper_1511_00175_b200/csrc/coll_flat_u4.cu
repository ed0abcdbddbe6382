// fp32 FLAT kernels with unroll factor U = 4 (see coll_flat.cuh).
#include "coll_flat.cuh"

namespace fc {
FC_FLAT_TABLE(4)
}  // namespace fc
