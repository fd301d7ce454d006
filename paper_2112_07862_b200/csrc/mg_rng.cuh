// numpy Generator(PCG64).standard_normal stream on the device (mg_rng.cu).
#pragma once
#include "mg_common.cuh"

namespace mg {
// the state / inc of np.random.default_rng(seed).bit_generator.state['state']
void normal_stream(mg_ctx *ctx, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                   uint64_t inc_lo, int64_t count, double *out);
}  // namespace mg
