// Micro-check of the device-resident control design (a12): nested WHILE / IF
// conditional graph nodes built during stream capture (cudaStreamBeginCaptureToGraph on one
// stream per nesting depth), with a thread-block-cluster kernel, a memset and plain kernels
// inside the bodies, conditions set on the device by cudaGraphSetConditional.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/graph_cond scripts/micro/graph_cond.cu
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      printf("FAIL %s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));         \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

__global__ void k_inc(long long* c, int i) { atomicAdd((unsigned long long*)&c[i], 1ull); }
__global__ void __cluster_dims__(4, 1, 1) k_cluster(long long* c) {
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)&c[5], 1ull);
}
// counter i counts up to n, then clears the handle (and resets for the next entry)
__global__ void k_cond(long long* c, int i, long long n, cudaGraphConditionalHandle h) {
  c[i] += 1;
  const bool more = c[i] < n;
  if (!more) c[i] = 0;
  cudaGraphSetConditional(h, more ? 1u : 0u);
}
__global__ void k_set(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }

static cudaStream_t S[4];
static int depth = 0;

static int add_cond(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, cudaGraph_t* body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps;
  size_t nd;
  CK(cudaStreamGetCaptureInfo(S[depth], &st, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
  *body = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(S[depth], &node, 1, cudaStreamSetCaptureDependencies));
  return 0;
}

int main() {
  for (int i = 0; i < 4; ++i) CK(cudaStreamCreateWithFlags(&S[i], cudaStreamNonBlocking));
  long long* c;
  CK(cudaMalloc(&c, 16 * sizeof(long long)));
  CK(cudaMemset(c, 0, 16 * sizeof(long long)));
  double* buf;
  CK(cudaMalloc(&buf, 1 << 20));
  cudaGraph_t top;
  CK(cudaGraphCreate(&top, 0));
  cudaGraphConditionalHandle ho, hi, hif;
  CK(cudaGraphConditionalHandleCreate(&ho, top, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hi, top, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hif, top, 0, 0));
  CK(cudaStreamBeginCaptureToGraph(S[0], top, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_inc<<<1, 1, 0, S[0]>>>(c, 0);
  k_set<<<1, 1, 0, S[0]>>>(ho, 1);
  cudaGraph_t bo;
  if (add_cond(ho, cudaGraphCondTypeWhile, &bo)) return 1;
  {
    depth = 1;
    CK(cudaStreamBeginCaptureToGraph(S[1], bo, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_inc<<<1, 1, 0, S[1]>>>(c, 1);
    CK(cudaMemsetAsync(buf, 0, 1 << 20, S[1]));
    k_set<<<1, 1, 0, S[1]>>>(hi, 1);
    cudaGraph_t bi;
    if (add_cond(hi, cudaGraphCondTypeWhile, &bi)) return 1;
    {
      depth = 2;
      CK(cudaStreamBeginCaptureToGraph(S[2], bi, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      k_inc<<<1, 1, 0, S[2]>>>(c, 2);
      k_cluster<<<8, 32, 0, S[2]>>>(c);
      k_cond<<<1, 1, 0, S[2]>>>(c, 8, 3, hi);     // 3 inner iterations per entry
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(S[2], &tmp));
      depth = 1;
    }
    k_cond<<<1, 1, 0, S[1]>>>(c, 9, 5, hif);       // IF: runs on the first 4 outer passes
    // trick: k_cond resets the counter when it clears; use a separate counter for the loop
    cudaGraph_t bif;
    if (add_cond(hif, cudaGraphCondTypeIf, &bif)) return 1;
    {
      depth = 2;
      CK(cudaStreamBeginCaptureToGraph(S[2], bif, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      k_inc<<<1, 1, 0, S[2]>>>(c, 3);
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(S[2], &tmp));
      depth = 1;
    }
    k_cond<<<1, 1, 0, S[1]>>>(c, 10, 5, ho);      // 5 outer iterations
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(S[1], &tmp));
    depth = 0;
  }
  k_inc<<<1, 1, 0, S[0]>>>(c, 4);
  cudaGraph_t out;
  CK(cudaStreamEndCapture(S[0], &out));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, out, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(a, S[0]));
    CK(cudaGraphLaunch(ex, S[0]));
    CK(cudaEventRecord(b, S[0]));
    CK(cudaStreamSynchronize(S[0]));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    long long h[16];
    CK(cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost));
    printf("rep %d: top %lld outer %lld inner %lld if %lld tail %lld cluster-CTAs %lld  (%.3f ms)\n", rep, h[0], h[1],
           h[2], h[3], h[4], h[5], ms);
    const long long R = rep + 1;
    const bool ok = h[0] == R && h[1] == 5 * R && h[2] == 15 * R && h[3] == 4 * R && h[4] == R && h[5] == 8 * 15 * R;
    printf(ok ? "OK\n" : "MISMATCH\n");
    if (!ok) return 2;
  }
  return 0;
}
