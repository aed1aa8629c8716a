// fused.cu -- fused z-marching kernels (K1 leapfrog, K2 pair) -- placeholder until written.
#include "internal.h"

namespace pe {
bool fused_supported(const Grid &) { return false; }
int k_leapfrog_fused(const KernelArgs &, void *[2], int64_t, const SrcDev *, int, const void *) {
    return fail(PARAEXP_ENOTSUP, "fused kernels not built");
}
int k_poly_substep_fused(const KernelArgs &, const Plan &, void *[4]) {
    return fail(PARAEXP_ENOTSUP, "fused kernels not built");
}
}  // namespace pe
