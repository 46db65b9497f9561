// Step a4: tensor-core Gaussian path (placeholder until the tcgen05 kernel lands).
#include "internal.cuh"

namespace kde {

int launch_tc(kde_ctx* c, float* out, cudaStream_t s) {
    (void)c;
    (void)out;
    (void)s;
    set_error("kde_eval: tensor-core path not built yet");
    return KDE_EUNSUPPORTED;
}

}  // namespace kde
