// Probe: TMA tiled loads -- rank 3 vs 4, negative vs non-negative start coords.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_1509_09308_b200/csrc/sm100_ptx.cuh"

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap tm, float* out, int bytes, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { wino::ptx::mbar_init(&bar, 1); wino::ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    wino::ptx::mbar_arrive_expect_tx(&bar, bytes);
    if (RANK == 4) wino::ptx::tma_load_4d(sm, &tm, &bar, x0, y0, 0, 0);
    else wino::ptx::tma_load_3d(sm, &tm, &bar, x0, y0, 0);
  }
  wino::ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int W = 64, H = 16, C = 8;
  std::vector<float> h(W * H * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  for (int rank : {3, 4}) for (int neg : {0, 1}) for (int sw : {0, 1}) {
    float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1 << 20);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[4] = {W, H, C, 1};
    cuuint64_t str[3] = {W * 4ull, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
    cuuint32_t box[4] = {32, 4, 8, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int bytes = 32 * 4 * 8 * 4;
    cudaError_t e;
    if (rank == 4) { cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
      probe<4><<<1, 128, bytes>>>(tm, o, bytes, neg ? -1 : 1, neg ? -1 : 1); }
    else { cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
      probe<3><<<1, 128, bytes>>>(tm, o, bytes, neg ? -1 : 1, neg ? -1 : 1); }
    e = cudaDeviceSynchronize();
    printf("rank %d neg %d swizzle128 %d: encode=%d run=%s\n", rank, neg, sw, (int)r, cudaGetErrorString(e));
    cudaDeviceReset();
  }
}
