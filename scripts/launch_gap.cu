// Kernel-to-kernel gap inside a CUDA graph on this device, with and without
// programmatic dependent launch (experiment, not part of the library):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/launch_gap scripts/launch_gap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_work(float *p, int n, int iters, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = p[i];
    for (int k = 0; k < iters; k++) v = v * 1.0000001f + 1e-7f;
    p[i] = v;
  }
}

int main() {
  const int nk = 40;
  float *p;
  cudaMalloc(&p, 1 << 26);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int blocks : {1, 148, 1184, 4096}) {
    for (int pdl = 0; pdl < 2; pdl++) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < nk; k++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_work, p, blocks * 256, 100, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; w++) cudaGraphLaunch(ge, s);
      cudaEventRecord(a, s);
      for (int r = 0; r < 20; r++) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("blocks %5d pdl %d: %.2f us per kernel\n", blocks, pdl, 1e3 * ms / (20 * nk));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
