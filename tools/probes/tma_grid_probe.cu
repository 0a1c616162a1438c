// Probe: TMA tiled load validity vs rank, start coordinates and box shape.
// usage: tma_grid_probe RANK X0 Y0 BOXW BOXH BOXC [PDL]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1509_09308_b200/csrc/sm100_ptx.cuh"

template <int RANK, bool PDL>
__global__ void probe(const __grid_constant__ CUtensorMap tm, float* out, int bytes, int x0, int y0) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  if (PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) { wino::ptx::mbar_init(&bar, 1); wino::ptx::fence_mbar_init(); }
  __syncthreads();
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    wino::ptx::prefetch_tmap(&tm);
    wino::ptx::mbar_arrive_expect_tx(&bar, bytes);
    if (RANK == 4) wino::ptx::tma_load_4d(base, &tm, &bar, x0, y0, 0, 0);
    else wino::ptx::tma_load_3d(base, &tm, &bar, x0, y0, 0);
  }
  wino::ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(base)[i];
}

int main(int argc, char** argv) {
  int rank = atoi(argv[1]), x0 = atoi(argv[2]), y0 = atoi(argv[3]);
  int bw = atoi(argv[4]), bh = atoi(argv[5]), bc = atoi(argv[6]);
  bool pdl = argc > 7;
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int W = 96, H = 16, C = 40;
  std::vector<float> h(W * H * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1 << 22);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  alignas(64) CUtensorMap tm;
  cuuint64_t dims[4] = {W, H, C, 1};
  cuuint64_t str[3] = {W * 4ull, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
  cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bc, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = bw * bh * bc * 4;
  size_t smem = bytes + 1024;
  cudaError_t e;
#define RUN(R, P) { cudaFuncSetAttribute(probe<R, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    probe<R, P><<<1, 128, smem>>>(tm, o, bytes, x0, y0); }
  if (rank == 4) { if (pdl) RUN(4, true) else RUN(4, false) } else { if (pdl) RUN(3, true) else RUN(3, false) }
  e = cudaDeviceSynchronize();
  int bad = 0;
  if (e == cudaSuccess) {
    std::vector<float> got(bytes / 4);
    cudaMemcpy(got.data(), o, bytes, cudaMemcpyDeviceToHost);
    for (int c = 0; c < bc; ++c) for (int y = 0; y < bh; ++y) for (int x = 0; x < bw; ++x) {
      int gx = x0 + x, gy = y0 + y;
      float want = (gx >= 0 && gx < W && gy >= 0 && gy < H && c < C) ? h[(c * H + gy) * W + gx] : 0.f;
      bad += got[(c * bh + y) * bw + x] != want;
    }
  }
  printf("rank %d x0 %d y0 %d box %dx%dx%d pdl %d: encode=%d run=%s bad=%d\n", rank, x0, y0, bw, bh, bc,
         (int)pdl, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
