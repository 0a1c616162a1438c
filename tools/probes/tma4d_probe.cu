// Probe: which 4D TMA box geometries (fp32, no swizzle) load correctly.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_1509_09308_b200/csrc/sm100_ptx.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap tm, float* out, int bytes, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { wino::ptx::mbar_init(&bar, 1); wino::ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    wino::ptx::mbar_arrive_expect_tx(&bar, bytes);
    wino::ptx::tma_load_4d(sm, &tm, &bar, x0, y0, 0, 0);
  }
  wino::ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int W = 64, H = 16, C = 40, N = 1;
  std::vector<float> h(W * H * C * N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int boxes[][3] = {{32, 4, 8}, {36, 5, 8}, {36, 5, 32}, {64, 7, 8}, {68, 7, 8}, {68, 7, 32}, {40, 5, 8}};
  for (auto& b : boxes) {
    alignas(64) CUtensorMap tm;
    cuuint64_t dims[4] = {W, H, C, N};
    cuuint64_t str[3] = {W * 4ull, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
    cuuint32_t box[4] = {(cuuint32_t)b[0], (cuuint32_t)b[1], (cuuint32_t)b[2], 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int bytes = b[0] * b[1] * b[2] * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    probe<<<1, 128, bytes>>>(tm, o, bytes, -1, -1);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(bytes / 4);
    int bad = -1;
    if (e == cudaSuccess) {
      cudaMemcpy(got.data(), o, bytes, cudaMemcpyDeviceToHost);
      for (int c = 0; c < b[2] && bad < 0; ++c)
        for (int y = 0; y < b[1] && bad < 0; ++y)
          for (int x = 0; x < b[0]; ++x) {
            int gx = x - 1, gy = y - 1;
            float want = (gx >= 0 && gx < W && gy >= 0 && gy < H && c < C) ? h[(c * H + gy) * W + gx] : 0.f;
            if (got[(c * b[1] + y) * b[0] + x] != want) { bad = (c * b[1] + y) * b[0] + x; break; }
          }
    }
    printf("box %3d x %d x %2d  encode=%d  run=%s  check=%s\n", b[0], b[1], b[2], (int)r,
           cudaGetErrorString(e), e == cudaSuccess ? (bad < 0 ? "OK" : "MISMATCH") : "-");
    if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1 << 20);
      cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice); }
  }
}
