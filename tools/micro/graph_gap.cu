// Launch gap between dependent kernels inside a CUDA graph on this GPU:
// N dependent launches of a kernel that does (almost) nothing, captured
// into one graph, with ordinary or programmatic edges; prints us/kernel.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a graph_gap.cu -o graph_gap
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void k_noop(int* p, int grid_work) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (grid_work && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
static void to_programmatic(cudaGraph_t g) {
  size_t ne = 0;
  cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne);
  std::vector<cudaGraphNode_t> f(ne), t(ne);
  std::vector<cudaGraphEdgeData> ed(ne);
  cudaGraphGetEdges_v2(g, f.data(), t.data(), ed.data(), &ne);
  for (size_t k = 0; k < ne; ++k) {
    cudaGraphEdgeData pe = {};
    pe.type = cudaGraphDependencyTypeProgrammatic;
    pe.from_port = cudaGraphKernelNodePortLaunchCompletion;
    cudaGraphRemoveDependencies_v2(g, &f[k], &t[k], &ed[k], 1);
    cudaGraphAddDependencies_v2(g, &f[k], &t[k], &pe, 1);
  }
}
int main() {
  int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int N = 2000;
  int grids[] = {1, 148, 1184};
  for (int gi = 0; gi < 3; ++gi)
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g; cudaGraphExec_t ex;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < N; ++i) k_noop<<<grids[gi], 256, 0, s>>>(d, 1);
      cudaStreamEndCapture(s, &g);
      if (pdl) to_programmatic(g);
      if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, s);
      cudaEventRecord(a, s);
      for (int r = 0; r < 5; ++r) cudaGraphLaunch(ex, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %5d blocks  pdl %d : %.3f us per dependent kernel\n", grids[gi], pdl, ms * 1000.0 / (5.0 * N));
      cudaGraphExecDestroy(ex); cudaGraphDestroy(g);
    }
  // plain stream launches (no graph)
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < N; ++i) k_noop<<<1184, 256, 0, s>>>(d, 1);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("stream launches, 1184 blocks: %.3f us per kernel\n", ms * 1000.0 / N);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
