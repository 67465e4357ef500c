// Library-level C-ABI: version, error strings, launch accounting.
#include <atomic>
#include <cstdlib>

#include "common.cuh"

namespace ms {
static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
static std::atomic<int> g_pdl{-1};  // -1: not yet read from MS_PDL
bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("MS_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return v == 1;
}
int set_pdl(int on) {
  const int old = pdl_enabled() ? 1 : 0;
  g_pdl.store(on ? 1 : 0, std::memory_order_relaxed);
  return old;
}
}  // namespace ms

namespace ms {
int preload_accept();
int preload_accept_stochastic();
int preload_vote();
int preload_spec();
int preload_model();
int preload_attention();
int preload_gemv();
int preload_gemm();
int preload_wide();
int preload_tp();
int preload_fp32();
int preload_attention_tc();
int set_coresident(int on);
}  // namespace ms

extern "C" int ms_version(void) { return 200; }

extern "C" int ms_preload(void) {
  const int bad = ms::preload_accept() + ms::preload_accept_stochastic() + ms::preload_vote() +
                  ms::preload_spec() + ms::preload_model() + ms::preload_attention() + ms::preload_gemv() +
                  ms::preload_gemm() + ms::preload_wide() + ms::preload_tp() + ms::preload_fp32() +
                  ms::preload_attention_tc();
  return bad ? MS_ERR_CUDA : MS_OK;
}

extern "C" const char* ms_strerror(int status) {
  switch (status) {
    case MS_OK: return "ok";
    case MS_ERR_VALUE: return "invalid argument";
    case MS_ERR_LENGTH: return "length mismatch";
    case MS_ERR_DIST_MISMATCH: return "distribution shape mismatch";
    case MS_ERR_UNSUPPORTED: return "shape outside the kernel's supported range";
    case MS_ERR_CUDA: return cudaGetErrorString(cudaPeekAtLastError());
    default: return "unknown status";
  }
}

// Programmatic dependent launch for the launches that follow (a captured CUDA
// graph keeps the setting it was captured with); returns the previous value.
extern "C" int ms_set_pdl(int on) { return ms::set_pdl(on); }

// Co-resident launch shapes for the launches that follow: drafter decode
// kernels sized to fit beside the verifier's GEMM CTAs (include/minions.h).
extern "C" int ms_set_coresident(int on) { return ms::set_coresident(on); }

extern "C" int64_t ms_launch_count(void) { return ms::g_launches.load(); }
extern "C" void ms_reset_launch_count(void) { ms::g_launches.store(0); }
