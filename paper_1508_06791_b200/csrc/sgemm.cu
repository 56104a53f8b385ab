// sgemm.cu -- JACC_OP_SGEMM_F32 dispatch (reading R13).
#include "kernels.h"

namespace jacc_k {

cudaError_t sgemm_ffma(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p, cudaStream_t st,
                       int *launches);
size_t sgemm_3xtf32_ws_bytes(const jacc_sgemm_params_t *p);
cudaError_t sgemm_3xtf32(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p, void *ws,
                         cudaStream_t st, int *launches);

size_t sgemm_ws_bytes(const jacc_sgemm_params_t *p) {
    return p->mode == JACC_SGEMM_3XTF32 ? sgemm_3xtf32_ws_bytes(p) : 0;
}

cudaError_t sgemm_f32(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p, void *ws,
                      cudaStream_t st, int *launches) {
    if (p->mode == JACC_SGEMM_FFMA) return sgemm_ffma(A, B, C, p, st, launches);
    return sgemm_3xtf32(A, B, C, p, ws, st, launches);
}

}  // namespace jacc_k
