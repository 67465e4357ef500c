// SM partition for the pipelined schedule (SSM drafting beside LLM verify on
// one GPU): two green contexts that split the device's SMs, one stream each.
//
// Why: the verify GEMMs run two register-full CTAs per SM (146 regs x 448
// threads = the whole register file), so a drafter kernel launched on an
// ordinary concurrent stream only gets an SM when a GEMM CTA retires, and then
// holds it against the next GEMM CTA — each of the ~90 dependent drafter
// kernels of a step waits for a wave tail (drafting 5.6 ms per round alone,
// ~32 ms beside the verifier; the verifier +2-3 ms).  With disjoint SM sets the
// drafter kernels never wait for verify CTAs and never displace them.  The
// paper runs its SSMs on their own GPUs / streams; this is the
// one-GPU form of that placement.
//
// Driver entry points are resolved at run time (no -lcuda); kernels launched
// through the runtime API into these streams run on the stream's context's
// SMs, device memory is the primary context's (tools/green_probe.cu checks
// both).
#include <cuda.h>

#include "common.cuh"

namespace {
template <typename F>
F drv(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(f);
}
}  // namespace

extern "C" int ms_sm_partition(int device, int draft_sms, int draft_priority, int verify_priority,
                               void** draft_stream, void** verify_stream, int* got_draft, int* got_verify) {
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
  using GCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
  using GStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
  using DevGet = CUresult (*)(CUdevice*, int);
  if (draft_sms <= 0 || !draft_stream || !verify_stream) return MS_ERR_VALUE;
  auto dev_get = drv<DevGet>("cuDeviceGet");
  auto get_res = drv<GetRes>("cuDeviceGetDevResource");
  auto split = drv<Split>("cuDevSmResourceSplitByCount");
  auto gen = drv<GenDesc>("cuDevResourceGenerateDesc");
  auto gcreate = drv<GCreate>("cuGreenCtxCreate");
  auto gstream = drv<GStream>("cuGreenCtxStreamCreate");
  if (!dev_get || !get_res || !split || !gen || !gcreate || !gstream) return MS_ERR_UNSUPPORTED;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return MS_ERR_CUDA;
  CUdevice dev;
  CUdevResource all, grp, rest;
  if (dev_get(&dev, device) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return MS_ERR_UNSUPPORTED;
  if ((unsigned)draft_sms >= all.sm.smCount) return MS_ERR_VALUE;
  unsigned n = 1;
  if (split(&grp, &n, &all, &rest, 0, (unsigned)draft_sms) != CUDA_SUCCESS || n != 1) return MS_ERR_UNSUPPORTED;
  CUdevResourceDesc dd, dv;
  CUgreenCtx gd, gv;
  if (gen(&dd, &grp, 1) != CUDA_SUCCESS || gen(&dv, &rest, 1) != CUDA_SUCCESS) return MS_ERR_UNSUPPORTED;
  if (gcreate(&gd, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      gcreate(&gv, dv, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return MS_ERR_UNSUPPORTED;
  CUstream sd, sv;
  if (gstream(&sd, gd, CU_STREAM_NON_BLOCKING, draft_priority) != CUDA_SUCCESS ||
      gstream(&sv, gv, CU_STREAM_NON_BLOCKING, verify_priority) != CUDA_SUCCESS)
    return MS_ERR_UNSUPPORTED;
  *draft_stream = sd;
  *verify_stream = sv;
  if (got_draft) *got_draft = (int)grp.sm.smCount;
  if (got_verify) *got_verify = (int)rest.sm.smCount;
  return MS_OK;
}
