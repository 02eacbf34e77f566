// render_tc.cu -- tcgen05/TMEM renderer engine (placeholder until the
// tensor-core kernel lands; the dispatcher falls back to SIMT).
#include "common.cuh"
#include "kernels.h"

namespace dmv3d {

bool tc_supported(int, int, int) { return false; }

cudaError_t launch_render_tc(const RenderParams &, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace dmv3d
