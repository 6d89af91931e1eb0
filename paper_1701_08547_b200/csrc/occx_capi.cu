// occx_capi.cu -- library / context entry points of the C ABI (include/occx.h).
#include <cstdlib>
#include "occx_common.cuh"

extern "C" int occx_abi_version(void) { return OCCX_ABI_VERSION; }

extern "C" const char* occx_status_string(int status) {
  switch (status) {
    case OCCX_OK: return "ok";
    case OCCX_ERR_VALUE: return "invalid argument (ValueError)";
    case OCCX_ERR_ILLEGAL_LAUNCH: return "illegal launch (IllegalLaunchError)";
    case OCCX_ERR_UNSUPPORTED_ARCH: return "no throughput column (UnsupportedArchitectureError)";
    case OCCX_ERR_NO_CANDIDATES: return "no thread candidates (NoCandidatesError)";
    case OCCX_ERR_ARCH_SPEC: return "architecture invariant violated (ArchSpecError)";
    case OCCX_ERR_CUDA: return "CUDA runtime error";
    case OCCX_ERR_NCCL: return "NCCL error";
    case OCCX_ERR_CAPACITY: return "input exceeds a device table limit";
    case OCCX_ERR_KEY: return "missing throughput-table entry (KeyError)";
    case OCCX_ERR_INDEX: return "empty thread-candidate list (IndexError)";
    case OCCX_ERR_PARSE: return "unparseable input line (ParseError)";
    case OCCX_ERR_EMPTY: return "input has no instructions (EmptyInputError)";
    case OCCX_ERR_ATTRIBUTE: return "reference parser AttributeError (sass.py:278-279 quirk)";
    default: return "unknown status";
  }
}

extern "C" int occx_stream_sync(void* stream) {
  OCCX_CUDA_TRY(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  return OCCX_OK;
}

extern "C" int occx_ctx_create(int device, occx_ctx** out) {
  return occx_ctx_create_ex(device, 0u, out);
}

extern "C" int occx_ctx_create_ex(int device, uint32_t options, occx_ctx** out) {
  if (!out) return OCCX_ERR_VALUE;
  *out = nullptr;
  if (options & ~(uint32_t)(OCCX_CTX_K2_FEED_LDG | OCCX_CTX_K2_ONE_SLICE |
                            OCCX_CTX_K2_NO_STEAL))
    return OCCX_ERR_VALUE;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return OCCX_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return OCCX_ERR_CUDA;
  occx_ctx* c = static_cast<occx_ctx*>(std::malloc(sizeof(occx_ctx)));
  if (!c) return OCCX_ERR_VALUE;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  c->cc_major = prop.major;
  c->cc_minor = prop.minor;
  c->options = options;
  *out = c;
  return OCCX_OK;
}

extern "C" int occx_ctx_destroy(occx_ctx* ctx) {
  std::free(ctx);
  return OCCX_OK;
}

extern "C" int occx_ctx_sm_count(const occx_ctx* ctx) { return ctx ? ctx->sm_count : 0; }

extern "C" uint32_t occx_ctx_options(const occx_ctx* ctx) { return ctx ? ctx->options : 0u; }
