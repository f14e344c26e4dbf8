// walk_dispatch.cu -- runtime n -> compile-time N dispatch for the single-matrix walk.
#include "internal.h"

namespace perm {

#define PERM_R8(M, b) M(b + 1) M(b + 2) M(b + 3) M(b + 4) M(b + 5) M(b + 6) M(b + 7) M(b + 8)
#define PERM_R64(M) PERM_R8(M, 0) PERM_R8(M, 8) PERM_R8(M, 16) PERM_R8(M, 24) \
                    PERM_R8(M, 32) PERM_R8(M, 40) PERM_R8(M, 48) PERM_R8(M, 56)

cudaError_t walk_launch_n(int n, const WalkLaunch& L) {
#define PERM_CASE(N) case N: return walk_launch<N>(L);
    switch (n) { PERM_R64(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

cudaError_t walk_occupancy_n(int n, int* blocks_per_sm, int* walkers_per_block) {
#define PERM_CASE(N) case N: return walk_occupancy<N>(blocks_per_sm, walkers_per_block);
    switch (n) { PERM_R64(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

cudaError_t walk_occupancy_c_n(int n, int* blocks_per_sm) {
#define PERM_CASE(N) case N: return walk_occupancy_c<N>(blocks_per_sm);
    switch (n) { PERM_R64(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

cudaError_t walk_seed_launch_n(int n, const double2* A_dev, const uint64_t* ranks_dev, int count, double2* w_out,
                               cudaStream_t s) {
#define PERM_CASE(N) case N: return walk_seed_launch<N>(A_dev, ranks_dev, count, w_out, s);
    switch (n) { PERM_R64(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

cudaError_t walk_small_launch_n(int n, const double2* A_dev, int e, uint64_t chunks, ddc* raw, ddc* out_dd,
                                double2* out_c, cudaStream_t s) {
#define PERM_CASE(N) case N: return walk_small_launch<N>(A_dev, e, chunks, raw, out_dd, out_c, s);
    switch (n) { PERM_R8(PERM_CASE, 0) PERM_R8(PERM_CASE, 8) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

#define PERM_R48(M) PERM_R8(M, 0) PERM_R8(M, 8) PERM_R8(M, 16) PERM_R8(M, 24) PERM_R8(M, 32) PERM_R8(M, 40)

cudaError_t sparse_launch(const SparseLaunch& L) {
#define PERM_CASE(N) case N: return sparse_launch_t<N>(L);
    switch (L.n) { PERM_R48(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

cudaError_t sparse_occupancy(int n, int* blocks_per_sm) {
#define PERM_CASE(N) case N: return sparse_occupancy_t<N>(blocks_per_sm);
    switch (n) { PERM_R48(PERM_CASE) default: return cudaErrorInvalidValue; }
#undef PERM_CASE
}

}  // namespace perm
