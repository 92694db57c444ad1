// C-ABI plumbing: thread-local errors, version, GEMM dispatch.
#include <cuda_runtime.h>

#include <string>

#include "../../include/adaptra.h"
#include "kernels/kernels.h"
#include "util.h"

namespace adaptra {
static thread_local std::string g_last_error;
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
const char* last_error() { return g_last_error.c_str(); }
int gemm_tc(const adaptra_gemm_desc_t& g, cudaStream_t st);
int gemm_simt(const adaptra_gemm_desc_t& g, cudaStream_t st);
}  // namespace adaptra

extern "C" const char* adaptra_last_error(void) { return adaptra::last_error(); }

extern "C" const char* adaptra_version(void) { return "adaptra-b200 0.1 (sm_100a)"; }

extern "C" int adaptra_gemm(const adaptra_gemm_desc_t* g, void* stream) {
  if (!g || g->M < 0 || g->N < 0 || g->K < 1 || g->Z < 1 || g->zdiv < 1)
    return adaptra::set_error(ADAPTRA_EINVAL, "adaptra_gemm: bad shape");
  if (!g->A || !g->B || !g->C) return adaptra::set_error(ADAPTRA_EINVAL, "adaptra_gemm: null operand");
  if (g->M == 0 || g->N == 0) return ADAPTRA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == ADAPTRA_BF16) return adaptra::gemm_tc(*g, st);
  if (g->dtype == ADAPTRA_F32) {
    if (g->epi == ADAPTRA_EPI_STORE_ROWDOT) return adaptra::set_error(ADAPTRA_EINVAL, "STORE_ROWDOT is bf16-only");
    return adaptra::gemm_simt(*g, st);
  }
  return adaptra::set_error(ADAPTRA_EINVAL, "adaptra_gemm: bad dtype");
}

extern "C" int adaptra_p2p_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (!dst || !src || bytes < 0) return adaptra::set_error(ADAPTRA_EINVAL, "adaptra_p2p_copy: bad args");
  if (bytes == 0) return ADAPTRA_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  for (const void* p : {(const void*)dst, src}) {  // a peer GPU's buffer: enable peer access once
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice && a.device != cur) {
      cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return adaptra::set_error(ADAPTRA_ECUDA, "adaptra_p2p_copy: no peer access");
    }
    cudaGetLastError();
  }
  return adaptra::copy_async(dst, src, (long)bytes, (cudaStream_t)stream);
}
