// Feasibility probe (not product code): do runtime-API kernels and CUDA-graph
// launches issued into a green-context stream stay on that context's SMs?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/green_probe tools/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    CUresult r_ = (x);                                                                    \
    if (r_ != CUDA_SUCCESS) {                                                             \
      const char* s_;                                                                     \
      cuGetErrorString(r_, &s_);                                                          \
      printf("FAIL %s -> %d %s\n", #x, (int)r_, s_);                                      \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)
#define CR(x)                                                                             \
  do {                                                                                    \
    cudaError_t r_ = (x);                                                                 \
    if (r_ != cudaSuccess) {                                                              \
      printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_));                              \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

__global__ void smid_kernel(int* out, long long spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

static std::set<int> sms(const std::vector<int>& v) { return std::set<int>(v.begin(), v.end()); }

int main() {
  CR(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u (min partition %u, alignment %u)\n", all.sm.smCount, 0u, 0u);
  CUdevResource grp[8], rest;
  unsigned n = 1;
  CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rest, 0, 16));
  printf("split: %u group(s) of %u SMs, remaining %u SMs\n", n, grp[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dsmall, dbig;
  CK(cuDevResourceGenerateDesc(&dsmall, &grp[0], 1));
  CK(cuDevResourceGenerateDesc(&dbig, &rest, 1));
  CUgreenCtx gsmall, gbig;
  CK(cuGreenCtxCreate(&gsmall, dsmall, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gbig, dbig, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream ssmall, sbig;
  CK(cuGreenCtxStreamCreate(&ssmall, gsmall, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sbig, gbig, CU_STREAM_NON_BLOCKING, 0));
  const int NB = 296;
  int* d;
  CR(cudaMalloc(&d, NB * 4));
  std::vector<int> h(NB);

  // 1. runtime <<<>>> launch into the green stream
  smid_kernel<<<NB, 32, 0, (cudaStream_t)ssmall>>>(d, 20000);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)ssmall);
  printf("runtime launch into small green stream: %s\n", cudaGetErrorString(e));
  if (e == cudaSuccess) {
    CR(cudaMemcpy(h.data(), d, NB * 4, cudaMemcpyDeviceToHost));
    printf("  distinct SMs used: %zu (want <= %u)\n", sms(h).size(), grp[0].sm.smCount);
  }
  smid_kernel<<<NB, 32, 0, (cudaStream_t)sbig>>>(d, 20000);
  e = cudaStreamSynchronize((cudaStream_t)sbig);
  CR(cudaMemcpy(h.data(), d, NB * 4, cudaMemcpyDeviceToHost));
  std::set<int> big = sms(h);
  printf("runtime launch into big green stream: %s, distinct SMs %zu\n", cudaGetErrorString(e), big.size());

  // 2. graph captured on an ordinary stream, launched into the green stream
  cudaStream_t cap;
  CR(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CR(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  smid_kernel<<<NB, 32, 0, cap>>>(d, 20000);
  CR(cudaStreamEndCapture(cap, &g));
  CR(cudaGraphInstantiate(&ge, g, 0));
  CR(cudaMemset(d, 0xff, NB * 4));
  e = cudaGraphLaunch(ge, (cudaStream_t)ssmall);
  printf("graph launch into small green stream: %s\n", cudaGetErrorString(e));
  CR(cudaStreamSynchronize((cudaStream_t)ssmall));
  CR(cudaMemcpy(h.data(), d, NB * 4, cudaMemcpyDeviceToHost));
  std::set<int> gs = sms(h);
  printf("  distinct SMs used: %zu (want <= %u); overlap with big partition: %d\n", gs.size(), grp[0].sm.smCount,
         (int)std::count_if(gs.begin(), gs.end(), [&](int x) { return big.count(x) > 0; }));

  // 3. graph captured ON the green stream
  CR(cudaStreamBeginCapture((cudaStream_t)ssmall, cudaStreamCaptureModeThreadLocal));
  smid_kernel<<<NB, 32, 0, (cudaStream_t)ssmall>>>(d, 20000);
  e = cudaStreamEndCapture((cudaStream_t)ssmall, &g);
  printf("capture on green stream: %s\n", cudaGetErrorString(e));
  if (e == cudaSuccess) {
    CR(cudaGraphInstantiate(&ge, g, 0));
    CR(cudaMemset(d, 0xff, NB * 4));
    CR(cudaGraphLaunch(ge, cap));  // launched into an ordinary stream
    CR(cudaStreamSynchronize(cap));
    CR(cudaMemcpy(h.data(), d, NB * 4, cudaMemcpyDeviceToHost));
    printf("  green-captured graph launched on ordinary stream: distinct SMs %zu\n", sms(h).size());
  }
  // 4. events between green and ordinary streams
  cudaEvent_t ev;
  CR(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CR(cudaEventRecord(ev, (cudaStream_t)ssmall));
  e = cudaStreamWaitEvent(cap, ev, 0);
  printf("cross-context event wait: %s\n", cudaGetErrorString(e));
  printf("done\n");
  return 0;
}
