// train.cu -- forward+backward training step and Adam (in progress).
#include "engine.hpp"

namespace detnet {

int train_batch_gradient(detnet_model *, long, const float *, const float *, const int8_t *,
                         const detnet_loss_spec *, int, double *, detnet_eval *) {
    return fail(DETNET_ERR_UNSUPPORTED, "batch_gradient: not built yet");
}

int train_adam_step(detnet_ctx *, int, int, int, int, int, double *, const double *,
                    const double *, double *, double *, int64_t *, const detnet_adam_config *) {
    return fail(DETNET_ERR_UNSUPPORTED, "adam_step: not built yet");
}

} // namespace detnet
