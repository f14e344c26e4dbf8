// sparse_inst.cu -- explicit instantiations of the sparse restricted-enumeration kernel (sparse.cuh),
// compiled with -DPERM_PART=p (p = 0..5) for N = 8p+1 .. 8p+8 (n <= 48: one lane holds the row sums).
#include "sparse.cuh"

#ifndef PERM_PART
#error "PERM_PART must be defined"
#endif

namespace perm {
#define PERM_INST(N)                                                \
    template cudaError_t sparse_launch_t<N>(const SparseLaunch&);   \
    template cudaError_t sparse_occupancy_t<N>(int*);
#define PERM_P(b) PERM_INST(b + 1) PERM_INST(b + 2) PERM_INST(b + 3) PERM_INST(b + 4) \
                  PERM_INST(b + 5) PERM_INST(b + 6) PERM_INST(b + 7) PERM_INST(b + 8)
PERM_P(PERM_PART * 8)
}  // namespace perm
