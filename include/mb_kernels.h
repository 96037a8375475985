/* C-ABI of the B200 (sm_100a) data-plane kernels: libmb_sm100.so
 *
 * The reference (moebalance, /root/reference/pkg) has NO data plane: it models the MoE
 * layer analytically.  Each entry point below replaces one modelled quantity with the
 * real device computation; the reference interface it stands in for is cited per call.
 *
 * Conventions: all pointers are device pointers unless stated; every call is
 * asynchronous on the given cudaStream_t (passed as void*), never allocates, and
 * returns 0 on success or a nonzero status (1 invalid argument, 2 CUDA error,
 * 3 unsupported, 4 timeout); mb_last_error() returns the thread-local message.
 */
#ifndef MB_KERNELS_H
#define MB_KERNELS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* mb_last_error(void);
int mb_version(void);

/* ---------------------------------------------------------------- K1 histogram
 * counts[b][e] = #{(t,i) : idx[b][t][i] == e}, for nb independent (micro-batch, layer)
 * batches of T tokens x k choices.  One launch for every batch (routing is replayed, so all
 * of it is known up front).  Also emits per-chunk counts used by the stable permutation.
 * Replaces: RoutingTrace.matrices row (routing.py:151-168; routing.bin layout routing.py:3-13),
 * i.e. np.bincount over the top-k indices.                                                  */
int mb_expert_histogram(const int32_t* idx, int64_t nb, int64_t tokens, int32_t topk, int32_t num_experts,
                        uint32_t* counts, uint32_t* chunk_counts, int32_t chunk_tokens, void* stream);

/* ---------------------------------------------------------------- K4 grouped GEMM
 * tcgen05/TMEM/TMA persistent grouped GEMM (bf16 in, fp32 accumulate).
 * Replaces: costmodel.comp_time (costmodel.py:161-163), the modelled 6*h*h' FLOP/token expert
 * FFN ("three GEMMs").  groups: device array of
 * struct {int32 rows, a0, slot, flags, seg_begin, seg_count, pad, pad}; segs (W mode only, may be
 * NULL): device array of struct {int32 a0, rows} K-segments, so one wgrad launch can contract
 * over every micro-batch of the step.                                                         */
enum {
  MB_GEMM_FWD_STORE = 0,     /* C[rows_g,N] = A[rows_g,K] . B_slot[N,K]^T           (Y = Act W2^T) */
  MB_GEMM_FWD_SWIGLU = 1,    /* as above, epilogue C=H, C2=silu(gate)*up             (H = X W1^T)   */
  MB_GEMM_DGRAD_STORE = 2,   /* C[rows_g,N] = A[rows_g,K] . B_slot[K,N]              (dX = dH W1)   */
  MB_GEMM_DGRAD_DSWIGLU = 3, /* as above, epilogue SwiGLU backward with aux=H -> C=dH (dAct = dY W2) */
  MB_GEMM_WGRAD = 4          /* C_slot[M,N] (+)= A[K_g,M]^T . B[K_g,N]               (dW)           */
};
int mb_grouped_gemm(int mode, const void* A, int64_t a_rows, int64_t a_cols, const void* B0, int64_t b0_rows,
                    const void* B1, int64_t b1_rows, int64_t b_cols, const void* groups, const void* segs,
                    int num_groups, int M,
                    int N, int K, void* C, int64_t ldc, int64_t c_slot_stride, void* C2, int64_t ldc2,
                    const void* aux, int64_t ld_aux, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MB_KERNELS_H */
