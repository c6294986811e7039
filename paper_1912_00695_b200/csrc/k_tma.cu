// TMA-staged 2.5D factorised stencil (placeholder plan: not yet enabled).
#include <cuda_runtime.h>

#include "kernels.h"

namespace swb {

TmaPlan tma_plan(int H, const Geo& g, int num_sms) {
    (void)g;
    (void)num_sms;
    TmaPlan p{};
    p.ok = 0;
    p.H = H;
    return p;
}

cudaError_t tma_make_maps(const TmaPlan&, const Geo&, int, void*) { return cudaErrorNotSupported; }

cudaError_t launch_tma(const TmaPlan&, const void*, const Geo&, const Coef&, const Ctl&,
                       const Peer&, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace swb
