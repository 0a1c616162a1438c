// F(4x4,3x3) instantiations of the fused Winograd-GEMM (wino_fused.cuh);
// one translation unit per tile size so the build compiles them in parallel.
#include "wino_fused.cuh"

namespace wino {
cudaError_t launch_fused_f4(int prec, const FusedArgs& f, cudaStream_t s) {
  return launch_fused_m<4>(prec, f, s);
}
}  // namespace wino
