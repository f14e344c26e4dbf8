// walk_inst.cu -- explicit instantiations of the single-matrix walk for a range of orders N.
// Compiled several times with -DPERM_PART=p (p = 0..7) so the 64 instantiations build in parallel;
// part p instantiates N = 8p+1 .. 8p+8.
#include "walk.cuh"

#ifndef PERM_PART
#error "PERM_PART must be defined"
#endif

namespace perm {
#define PERM_INST(N)                                                                             \
    template cudaError_t walk_launch<N>(const WalkLaunch&);                                      \
    template cudaError_t walk_occupancy<N>(int*, int*);                                          \
    template cudaError_t walk_occupancy_c<N>(int*);                                              \
    template cudaError_t walk_seed_launch<N>(const double2*, const uint64_t*, int, double2*, cudaStream_t); \
    template cudaError_t walk_small_launch<N>(const double2*, int, uint64_t, ddc*, ddc*, double2*, cudaStream_t);
#define PERM_P(b) PERM_INST(b + 1) PERM_INST(b + 2) PERM_INST(b + 3) PERM_INST(b + 4) \
                  PERM_INST(b + 5) PERM_INST(b + 6) PERM_INST(b + 7) PERM_INST(b + 8)
PERM_P(PERM_PART * 8)
}  // namespace perm
