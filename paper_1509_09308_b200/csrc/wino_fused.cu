// Host entry of the fused Winograd-GEMM (kernels in wino_fused.cuh,
// instantiated per tile size in wino_fused_f2.cu / wino_fused_f4.cu).
#include "wino_internal.h"

namespace wino {

cudaError_t launch_fused_f2(int prec, const FusedArgs& f, cudaStream_t s);
cudaError_t launch_fused_f4(int prec, const FusedArgs& f, cudaStream_t s);

// channels per pipeline stage (one operand swizzle row): 3xTF32 32 B, else 64 B
int fused_num_kblocks(int prec, int C) {
  const int bkc = (prec == kFP32) ? 8 : (prec == kTF32 ? 16 : 32);
  return (C + bkc - 1) / bkc;
}
int fused_tiles_per_unit(int m) { return m == 4 ? 64 : 128; }

cudaError_t launch_fused(int m, int prec, const FusedArgs& f, cudaStream_t s) {
  if (f.P <= 0 || f.K <= 0) return cudaSuccess;
  if (prec == kFP64) return cudaErrorInvalidValue;
  return m == 2 ? launch_fused_f2(prec, f, s) : launch_fused_f4(prec, f, s);
}

}  // namespace wino
