// prefill_kernel.cu -- N2: tensor-core (tcgen05) path for long prefill segments.
// Placeholder until the tcgen05 kernel lands: prefill_supported() returns false, so the
// planner routes every token through the SIMT kernel (N1), which is exact for any length.
#include <cuda_runtime.h>

#include "plan.h"

namespace lora {

bool prefill_supported(int, int, int) { return false; }

int launch_prefill(const Plan&, const PrefillLaunch&, cudaStream_t, int*) { return (int)cudaErrorNotSupported; }

}  // namespace lora
