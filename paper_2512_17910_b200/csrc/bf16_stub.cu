// Temporary: tensor-core GEMM and attention land in gemm_sm100.cu / attn_sm100.cu.
#include "common.cuh"
#include "kernels.h"
namespace alora {
int attn_bf16(const __nv_bfloat16*, int64_t, int, int, const int32_t*, const int32_t*, const int32_t*, int, int, int,
              const __nv_bfloat16*, int, int, int, int, int, int, __nv_bfloat16*, int64_t, void*, int64_t,
              cudaStream_t) { return ALORA_EUNSUPPORTED; }
int64_t attn_bf16_workspace(int, int, int, int, int, int, int) { return 0; }
}
