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

/* Bits a kernel ORs into a caller-provided int32 error flag (host-visible pinned memory in the
 * data plane, read without a device sync; the host raises on any nonzero value). */
#define MB_ERR_ROUTING_MISMATCH 1  /* routing has more tokens for an expert than the plan's counts */
#define MB_ERR_COUNTS_MISMATCH 2   /* K1 histogram differs from the counts the plan was built for */

/* ---------------------------------------------------------------- K1 histogram
 * counts[b][e] = #{(t,i) : idx[b][t][i] == e}, for nb independent (micro-batch, layer)
 * batches of T tokens x k choices.  One launch for every batch (routing is replayed, so all
 * of it is known up front).  Also emits per-chunk counts used by the stable permutation.
 * Replaces: RoutingTrace.matrices row (routing.py:151-168; routing.bin layout routing.py:3-13),
 * i.e. np.bincount over the top-k indices.                                                  */
int mb_expert_histogram(const int32_t* idx, int64_t nb, int64_t tokens, int32_t topk, int32_t num_experts,
                        uint32_t* counts, uint32_t* chunk_counts, int32_t chunk_tokens, void* stream);

/* Process default of the SMs the persistent grouped GEMM may occupy (0 = all; env MB_GEMM_SMS
 * overrides); a call's own gemm_sms > 0 wins.  The SMs left free run the dispatch / combine
 * kernels of the comm stream while the GEMM runs (the reference models comm and compute as
 * separate resources, costmodel.py:205-213). */
int mb_set_gemm_sms(int sms);

/* ---------------------------------------------------------------- K4 grouped GEMM
 * tcgen05/TMEM/TMA persistent grouped GEMM (bf16 in, fp32 accumulate).
 * Replaces: costmodel.comp_time (costmodel.py:161-163), the modelled 6*h*h' FLOP/token expert
 * FFN ("three GEMMs").  groups: device array of
 * struct {int32 rows, a0, slot, flags, seg_begin, seg_count, rows_real, kblocks}; segs (W mode
 * only, may be NULL): device array of struct {int32 a0, rows} K-segments (rows a multiple of 16,
 * kblocks = sum of ceil(rows / 64)), so one wgrad launch can contract over every micro-batch. */
enum {
  MB_GEMM_FWD_STORE = 0,     /* C[rows_g,N] = A[rows_g,K] . B_slot[N,K]^T           (Y = Act W2^T) */
  MB_GEMM_FWD_SWIGLU = 1,    /* as above, epilogue C=H, C2=silu(gate)*up             (H = X W1^T)   *
                              * row_scale != NULL (pair family): C2 = row_scale[row]*silu(gate)*up,
                              * 0 on pad rows -- the data plane's pre-gated activation, so the down
                              * GEMM yields gate*Y and dW2 = dY^T C2 needs no rewrite            */
  MB_GEMM_DGRAD_STORE = 2,   /* C[rows_g,N] = A[rows_g,K] . B_slot[K,N]              (dX = dH W1)   */
  MB_GEMM_DGRAD_DSWIGLU = 3, /* as above, epilogue SwiGLU backward with aux=H -> C=dH (dAct = dY W2) */
  MB_GEMM_WGRAD = 4,         /* C_slot[M,N] (+)= A[K_g,M]^T . B[K_g,N]               (dW)           */
  MB_GEMM_DGRAD_DSWIGLU_GATED = 5 /* A = raw dout rows; epilogue applies row_scale (gate): C = dH,
                                     C2 (optional, NULL = not written) = gate*act,
                                     row_partial[row][N/64] = partial <dout.W2, act>
                                     whose sum is dgate = <dout, Y> (replaces the combine backward) */
};
/* mode | 0x100 forces the 1-CTA kernel (default: CTA-pair 256x256 tiles when the shape allows);
 * mode | 0x200 runs the single-CTA member of the pair family (cta_group::1, 128 x 256 tiles, every
 * F-mode epilogue incl. the gated dSwiGLU) -- the 128-row tail blocks of odd groups.
 * gemm_sms > 0: SMs this launch's persistent grid covers (each data plane passes its own split;
 * <= 0 = the process default of mb_set_gemm_sms). */
int mb_grouped_gemm(int mode, const void* A, int64_t a_rows, int64_t a_cols, const void* B0, int64_t b0_rows,
                    const void* B1, int64_t b1_rows, int64_t b_cols, const void* groups, const void* segs,
                    int num_groups, int M,
                    int N, int K, void* C, int64_t ldc, int64_t c_slot_stride, void* C2, int64_t ldc2,
                    const void* aux, int64_t ld_aux, const float* row_scale, float* row_partial, int32_t gemm_sms,
                    void* stream);

/* Both weight gradients of the expert FFN in ONE persistent launch (one dynamically scheduled tile
 * list): groups without flag 4 compute C0_slot[M0][N0] (+)= A0[K_g, M0]^T . B0[K_g, N0] (dW2 =
 * dY^T Act), groups with flag 4 compute C1_slot[M1][N1] (+)= A1^T . B1 (dW1 = dH^T X); A*, B* are
 * [k_rows, .] bf16 row-major, C* fp32 [slots][M][N]; groups / segs as MB_GEMM_WGRAD (flag 1 =
 * accumulate).  Replaces: the wgrad third of costmodel.comp_time (12 h h' of the 18 per row). */
int mb_grouped_wgrad2(const void* A0, const void* B0, int32_t M0, int32_t N0, void* C0, const void* A1,
                      const void* B1, int32_t M1, int32_t N1, void* C1, int64_t k_rows, const void* groups,
                      const void* segs, int num_groups, int32_t gemm_sms, void* stream);

/* ---------------------------------------------------------------- K2 permutation
 * chunk_base[b][c][e] = exclusive prefix over chunks of chunk_counts (from mb_expert_histogram). */
int mb_chunk_scan(const uint32_t* chunk_counts, uint32_t* chunk_base, int64_t nb, int32_t chunks, int32_t E,
                  void* stream);
/* Canonical permutation of one source GPU: perm[t][i] = {dst_gpu, dst_row} with the stable rank
 * of (t,i) among the source's entries of expert e split over its copies by the integer counts in
 * route_tab[E][maxc][4] {cum_end, dst_gpu, dst_row_base, 0} (round_split, replicate.py:501-525;
 * copy order ReplicaPlacement.copies, replicate.py:55-56).  gate values are stored at
 * dst_gate[dst_gpu][dst_row] (peer pointers) when both are non-NULL.  A choice whose rank is past
 * the last copy's cum_end (routing != the planned counts) gets perm = {-1,-1} and ORs
 * MB_ERR_ROUTING_MISMATCH into *error_flag (may be NULL): nothing is ever written past a slot.
 * Replaces: the dispatch leg of costmodel.flow_matrix (costmodel.py:91-108), which only counts. */
int mb_permute_rank(const int32_t* idx, int64_t T, int32_t k, const float* gate, int32_t E, const uint32_t* chunk_base,
                    int32_t chunk_tokens, const int32_t* route_tab, const int32_t* ncopies, int32_t maxc,
                    float* const* dst_gate, int32_t* perm, int32_t* error_flag, void* stream);

/* The same over nb consecutive micro-batches in one launch: idx / gate / perm advance by T*k
 * entries, chunk_base by chunks*E, route_tab by E*maxc*4, ncopies by E, and dst_gate holds
 * `world` receive-gate pointers per micro-batch. */
int mb_permute_rank_nb(const int32_t* idx, int64_t T, int32_t k, const float* gate, int32_t E,
                       const uint32_t* chunk_base, int32_t chunk_tokens, const int32_t* route_tab,
                       const int32_t* ncopies, int32_t maxc, float* const* dst_gate, int32_t world, int32_t* perm,
                       int32_t nb, int32_t* error_flag, void* stream);

/* On-device per-micro-batch tables (one block): round_split of every replicated expert's tokens
 * over its copies (replicate.py:501-525; fractions from the host token-split LP, per replicated
 * expert [G][1+R_e] f64 concatenated in rep_experts order, counts out in the same layout), then the
 * receive layout of every GPU (slot_tab, slot_w, nslots, total_rows), the route table every
 * source places its rows with (route_tab, ncopies, as mb_permute_rank consumes them) and the
 * executed flow [G][G] (costmodel.flow_matrix with integer splits, costmodel.py:91-108).
 * x: [G][E] routing counts (the gathered K1 histograms); home: ReorderPlan.assignment; replicas
 * as CSR (rep_ptr[n_rep+1] into rep_gpus, ReplicaPlacement.copies order, replicate.py:55-56).
 * Bit-identical to mbp_round_split + mbp_dispatch_plan (include/mb_planner.h).  *error != 0 on
 * inconsistent input (bit 1 split sums, 2 copies > maxc, 4 slots > max_slots, 8 rows >= 2^31). */
int mb_dispatch_tables(int32_t G, int32_t E, const int32_t* x, const int32_t* home, int32_t n_rep,
                       const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus, const double* frac,
                       int32_t pad, int32_t maxc, int32_t max_slots, int64_t* counts, int32_t* route_tab,
                       int32_t* ncopies, int32_t* slot_tab, int32_t* slot_w, int32_t* nslots, int64_t* total_rows,
                       int64_t* flow, int32_t* error, void* stream);

/* error_flag |= code when counts[i] != expected[i] for any i < n (the K1 histogram against the
 * counts the step plan was built from, RoutingTrace.matrices row, routing.py:151-168). */
int mb_check_counts(const uint32_t* counts, const int32_t* expected, int64_t n, int32_t* error_flag, int32_t code,
                    void* stream);

/* ---------------------------------------------------------------- K3 dispatch all-to-all
 * Row scatter: row t of x ([T,h] bf16) is stored at dst_rows[perm.gpu] + perm.row*h for every
 * choice i (device array of per-GPU base pointers, peers mapped over NVLink; 128-bit stores).
 * Replaces: the dispatch link loads of costmodel._accumulate_direction (costmodel.py:64-88, 148). */
int mb_scatter_rows(const void* x, int64_t T, int32_t k, int32_t h, const int32_t* perm, void* const* dst_rows,
                    int32_t comm_blocks, void* stream);

/* Row-mover engine for mb_scatter_rows / mb_combine_rows: blocks > 0 selects the TMA bulk-copy
 * kernels (cp.async.bulk rows through shared memory; one block per SM, ~190 KB of rows in flight,
 * never co-resident with a GEMM CTA) on that many blocks; 0 = the register-copy kernels.  This
 * sets the process default; a call's own comm_blocks >= 0 wins (each data plane passes its own
 * engine), -1 = use the default. */
int mb_set_comm_blocks(int32_t blocks);

/* ---------------------------------------------------------------- K6 combine
 * out[t] = sum_i w[t,i] * src_rows[perm.gpu][perm.row] in fp32 (w = gate, or 1 when gate == NULL),
 * rows read from peers; optionally scalar_out[t,i] = sum of the npart per-row partials at
 * src_scalar[perm.gpu][perm.row*npart ...] (the dgate gather).
 * Replaces: the mirrored combine leg of compute_loads (costmodel.py:149-150). */
int mb_combine_rows(const void* const* src_rows, const int32_t* perm, const float* gate, int64_t T, int32_t k,
                    int32_t h, void* out, const float* const* src_scalar, float* scalar_out, int32_t npart,
                    int32_t comm_blocks, void* stream);
/* Expert-side combine backward (unfused reference variant of the gated dSwiGLU epilogue):
 * dY = gate*dout in place, dgate = <dout, Y>, pad rows zeroed. */
int mb_combine_bwd_expert(void* dout_rows, const void* y_rows, const float* gate_rows, float* dgate_rows,
                          const int32_t* slot_tab, int32_t nslots, int64_t total_rows, int32_t h, void* stream);
/* Zero the padding rows of every receive slot (slot_tab [nslots][4] {row_begin, rows_real, rows_pad, expert}). */
int mb_zero_pad_rows(void* rows, const int32_t* slot_tab, int32_t nslots, int32_t h, void* stream);
/* Batched: micro-batch b uses rows + b*rows_stride rows and slot_tab + b*max_slots entries
 * (entries past a micro-batch's slot count are all-zero). */
int mb_zero_pad_rows_nb(void* rows, int64_t rows_stride, const int32_t* slot_tab, int32_t max_slots, int32_t nb,
                        int32_t h, void* stream);

/* ---------------------------------------------------------------- K5 replicas
 * dst[i] += sum_s srcs[s][i] (fp32, sources in list order): replica-gradient reduce into the owner,
 * sources read from peers (replica_memory replicate.py:528-534). */
int mb_accumulate_f32(float* dst, const float* const* srcs, int32_t nsrc, int64_t n, void* stream);
/* Batched form, one launch per micro-batch: tasks is a device array of
 *   struct { float* dst; const float* src[MB_ACC_MAX_SRC]; int64_t n; int32_t nsrc; int32_t store; }
 * (n a multiple of 4, max_n >= every n); store = 1 writes dst = sum(src) (the first contribution to a
 * gradient of a freshly zeroed step), else dst += sum(src).  Sources are summed in list order. */
#define MB_ACC_MAX_SRC 8
int mb_accumulate_f32_tasks(const void* tasks, int32_t ntasks, int64_t max_n, void* stream);
/* Copy-engine copy (replica weight pull from the owner into the layer-shared replica slots). */
int mb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* ---------------------------------------------------------------- peer memory / barrier
 * CUDA-IPC symmetric buffers for the one-process-per-GPU box; the reference models links only
 * (HardwareProfile.bw_nvlink/bw_rdma, topology.py:29-47). */
int mb_ipc_handle_size(void);
int mb_ipc_malloc(int64_t bytes, void** ptr, void* handle_out);
int mb_ipc_open(const void* handle, void** ptr);
int mb_ipc_close(void* ptr);
int mb_device_free(void* ptr);
/* Zeroed, device-mapped pinned host memory (the data plane's error flag: kernels OR bits into it,
 * the host reads it without a device synchronisation). */
int mb_host_alloc_mapped(int64_t bytes, void** host, void** dev);
int mb_host_free(void* host);
/* Device-side barrier over per-rank flag arrays (flags[p] = rank p's array of world u32); traps
 * after timeout_ns instead of hanging. */
int mb_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t world, uint32_t* epoch, int64_t timeout_ns,
                    int32_t* error_flag, void* stream);

/* ---------------------------------------------------------------- GPU-side planning
 * The annealing chains of reorder.anneal_reorder (reorder.py:299-326) on the device, one warp
 * per chain (lanes split the O(G) element work, lane 0 owns the PCG64 stream), every (layer, seed) chain of a model in one launch: chain c anneals layer
 * c / chains_per_layer with contrib[layer] ([E][G][5][G] f64) and base[layer] ([E], the LPT start);
 * consts[5] and rng[nchains][4] as mbp_anneal_prepare (include/mb_planner.h) writes them.  Writes
 * each chain's best plan best[nchains][E] and its iteration count; pick each layer's plan with
 * mbp_anneal_select.  G <= 32, E <= 1024. */
int mb_anneal_chains(const double* contrib, int32_t E, int32_t G, const int64_t* base, const double* consts,
                     double beta, const uint64_t* rng, int32_t nchains, int32_t chains_per_layer, double cooling,
                     double eps_frac, double term_eps, int64_t* best, int64_t* iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MB_KERNELS_H */
