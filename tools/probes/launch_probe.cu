// Latency probe: what does one dependent kernel boundary cost inside a CUDA
// graph (with and without programmatic dependent launch), versus one grid-wide
// barrier inside a persistent kernel?  Decides whether an N=1 layer should be
// one kernel with phases or a chain of kernels.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void gd_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void gd_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void step_kernel(float* buf, int n) {
  gd_launch();
  gd_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[i] * 1.0001f + 1.0f;
}

// one grid barrier: monotonically increasing counter, generation = target
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr));
    } while (v < target);
  }
  __syncthreads();
}

__global__ void phases_kernel(float* buf, int n, unsigned int* ctr, int phases) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (int p = 0; p < phases; ++p) {
    if (i < n) buf[i] = buf[i] * 1.0001f + 1.0f;
    grid_barrier(ctr, (p + 1) * gridDim.x);
  }
}

static float time_graph(cudaGraphExec_t ge, cudaStream_t s, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int L = 48, grid = 148, threads = 256, n = grid * threads;
  float* buf;
  unsigned int* ctr;
  cudaMalloc(&buf, n * sizeof(float));
  cudaMalloc(&ctr, sizeof(unsigned int));
  cudaMemset(buf, 0, n * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int smem_kb : {0, 200}) {
    cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int l = 0; l < L; ++l) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem_kb * 1024;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, step_kernel, buf, n);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t ge;
      cudaGraphInstantiate(&ge, g, 0);
      float ms = time_graph(ge, s, 50);
      printf("chain of %d kernels, smem %3d KB, pdl %d: %.2f us per kernel\n", L, smem_kb, pdl,
             ms * 1e3 / L);
    }
  }
  // persistent kernel with L grid barriers
  for (int smem_kb : {0, 200}) {
    cudaFuncSetAttribute(phases_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s);
      cudaEventRecord(a, s);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem_kb * 1024;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, phases_kernel, buf, n, ctr, L);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("one kernel, %d grid barriers, smem %3d KB: %.2f us per phase (%s)\n", L, smem_kb,
           best * 1e3 / L, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
