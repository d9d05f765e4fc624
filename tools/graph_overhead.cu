// graph_overhead.cu -- what a step-graph boundary costs on this GPU.
//
// Times CUDA-graph replays of chains of tiny kernels (one block of 256 threads
// or a 1184-block grid, each kernel waiting on its predecessor with
// griddepcontrol.wait) launched plain or with programmatic dependent launch,
// optionally with an IF conditional node (condition false) after every
// kernel.  Per-boundary cost = (replay time) / (kernels in the chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/graph_overhead tools/graph_overhead.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__global__ void k_tiny(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}

struct BigParam {
  int* p;
  char pad[1384];  // the engine's Ctx is ~1.4 KB
};
__global__ void k_tiny_big(BigParam b) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(b.p, 1);
}

__global__ void k_set(cudaGraphConditionalHandle h, int v) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (v) cudaGraphSetConditional(h, 1u);
}

static bool g_big = false;
static cudaError_t launch(cudaStream_t s, bool pdl, int grid, int* p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (g_big) {
    BigParam b{};
    b.p = p;
    return cudaLaunchKernelEx(&cfg, k_tiny_big, b);
  }
  return cudaLaunchKernelEx(&cfg, k_tiny, p);
}

// chain of n kernels; cond: an IF node (false) after each kernel
static int run(int n, bool pdl, bool cond, int grid, float* us_per) {
  cudaStream_t s, body;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&body, cudaStreamNonBlocking));
  int* p;
  CK(cudaMalloc(&p, 4));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < n; i++) {
    CK(launch(s, pdl, grid, p));
    if (cond) {
      cudaStreamCaptureStatus st;
      unsigned long long id;
      cudaGraph_t cg;
      const cudaGraphNode_t* deps;
      size_t nd;
      CK(cudaStreamGetCaptureInfo(s, &st, &id, &cg, &deps, &nd));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
      k_set<<<1, 32, 0, s>>>(h, 0);
      CK(cudaStreamGetCaptureInfo(s, &st, &id, &cg, &deps, &nd));
      cudaGraphNodeParams prm = {};
      prm.type = cudaGraphNodeTypeConditional;
      prm.conditional.handle = h;
      prm.conditional.type = cudaGraphCondTypeIf;
      prm.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, cg, deps, nd, &prm));
      CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
      CK(cudaStreamBeginCaptureToGraph(body, prm.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      k_tiny<<<1, 32, 0, body>>>(p);
      cudaGraph_t bg;
      CK(cudaStreamEndCapture(body, &bg));
    }
  }
  CK(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 20; i++) CK(cudaGraphLaunch(ge, s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int reps = 200;
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < reps; i++) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  *us_per = ms * 1000.f / reps / n;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(p);
  return 0;
}

int main() {
  std::printf("{\"per_boundary_us\": {");
  bool first = true;
  for (int grid : {1, 1184})
    for (int pdl = 0; pdl < 2; pdl++)
      for (int cond = 0; cond < 2; cond++) {
        float us;
        if (run(32, pdl, cond, grid, &us)) return 1;
        std::printf("%s\"grid%d_%s%s\": %.2f", first ? "" : ", ", grid, pdl ? "pdl" : "plain",
                    cond ? "_if" : "", us);
        first = false;
      }
  g_big = true;
  for (int grid : {1, 1184}) {
    float us;
    if (run(32, true, false, grid, &us)) return 1;
    std::printf(", \"grid%d_pdl_1400B_params\": %.2f", grid, us);
  }
  std::printf("}}\n");
  return 0;
}
