/* C-ABI of the host planners: libmb_planner.so (C++17, OpenMP)
 *
 * Each entry point is the native body of one function of the reference package's planner
 * API (moebalance 0.1.0, /root/reference/pkg/src/moebalance); the Python mirror in
 * paper_2605_08639_b200/ keeps the reference names, dataclasses and error behaviour and
 * calls these.  Reference interface replaced is cited per call.
 *
 * Conventions: row-major arrays, caller-allocated outputs, no global mutable state
 * (reentrant under a thread pool), status 0 = ok, 1 = invalid argument (-> ValueError),
 * 5 = solver failure (-> LPError), 6 = capacity exceeded; mbp_last_error() gives the
 * thread-local message.  Topology = (num_nodes, gpus_per_node), GPU ids node-major
 * (topology.py:50-115); hardware = (flops_per_gpu, bw_nvlink, bw_rdma, bytes_per_token)
 * (topology.py:29-47); model = (hidden_size, intermediate_size) (routing.py:53-77).
 * Replica placements are passed in CSR form in dict insertion order:
 *   n_rep experts rep_experts[n_rep], rep_ptr[n_rep+1], rep_gpus[rep_ptr[n_rep]]
 * and per-expert [G][1+R_e] fraction / count blocks concatenated in the same order.
 */
#ifndef MB_PLANNER_H
#define MB_PLANNER_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* mbp_last_error(void);

/* Route the simplex warm-start products through the ILP64 CBLAS that numpy links (path to
 * numpy.libs/libscipy_openblas64_*.so, symbol prefix "scipy_"), issuing the same
 * gemm/gemv/dot calls numpy's matmul dispatch makes in lp.DenseSimplex.add_columns /
 * add_row (lp.py:79-80, 100), so LP vertices match the reference bit for bit on one host.
 * path NULL restores the built-in loops.  Call once before planning (not thread-safe). */
int mbp_use_numpy_blas(const char* path, const char* prefix);
int mbp_numpy_blas_active(void);

/* reorder.static_plan (reorder.py:291-296) */
int mbp_static_plan(int32_t E, int32_t G, int64_t* assignment);

/* reorder.lpt_initial (reorder.py:265-288) */
int mbp_lpt_initial(const double* x, int32_t G, int32_t E, int64_t* assignment);

/* reorder.anneal_reorder (reorder.py:329-362): LPT start, one SA chain per seed (OpenMP,
 * `threads` 0 = all cores), best exact T_MoE among [LPT, extra plans, chains in seed order].
 * term_eps <= 0 means AnnealConfig.termination_eps = None.                                  */
int mbp_anneal_reorder(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden, int64_t inter,
                       double flops, double bw_nv, double bw_rd, double bpt, const uint64_t* seeds, int32_t nseeds,
                       double cooling, double eps_frac, double term_eps, double beta, const int64_t* extra,
                       int32_t nextra, int32_t threads, int64_t* assignment, int64_t* iterations);

/* Device annealing (GPU-side planning): the chains of anneal_reorder run on the GPU
 * (mb_anneal_chains, include/mb_kernels.h), one thread per seed.  mbp_anneal_prepare computes what
 * they share exactly as mbp_anneal_reorder does on the host -- the LPT start (base[E]), the
 * contribution tensor contrib[E][G][5][G] (reorder.py:179-194), the time units consts[5] =
 * {comp_unit, nv_tx, nv_rx, rd_tx, rd_rx seconds per row} -- and each seed's numpy PCG64 state
 * rng[nseeds][4] = {state_hi, state_lo, inc_hi, inc_lo} (SeedSequence(seed), reorder.py:303).
 * mbp_anneal_select returns the first minimum of the exact T_MoE over ncand candidate plans
 * (LPT, extras, chains in seed order: reorder.py:352-362). */
int mbp_anneal_prepare(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden, int64_t inter,
                       double flops, double bw_nv, double bw_rd, double bpt, double beta, const uint64_t* seeds,
                       int32_t nseeds, int64_t* base, double* contrib, double* consts, uint64_t* rng);
int mbp_anneal_select(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden, int64_t inter,
                      double flops, double bw_nv, double bw_rd, double bpt, double beta, const int64_t* cands,
                      int32_t ncand, int64_t* assignment);

/* Data-locality sample placement (reorder.py:365-568): greedy_sample_initial (greedy_only != 0)
 * or anneal_sample_placement (greedy start, one swap-SA chain per seed over samples inside each
 * micro-batch's +/-band token window, best exact summed T_MoE).  counts [S][L][E] (float64 of
 * the u32 sample counts), micro_batch[S], source_gpu[S], tokens[S], plans [L][E]; out placement[S]. */
int mbp_sample_placement(int32_t nodes, int32_t gpn, int32_t E, int32_t L, int32_t MB, int32_t S, const double* counts,
                         const int32_t* micro_batch, const int64_t* source_gpu, const double* tokens,
                         const int64_t* plans, int64_t hidden, int64_t inter, double flops, double bw_nv,
                         double bw_rd, double bpt, const uint64_t* seeds, int32_t nseeds, double cooling,
                         double eps_frac, double term_eps, double beta, double band, int32_t greedy_only,
                         int32_t threads, int64_t* placement);

/* costmodel.compute_loads (costmodel.py:127-158) -> loads[5][G] = comp, nvlink_tx, nvlink_rx,
 * rdma_tx, rdma_rx; optional flow[G][G] (costmodel.flow_matrix, costmodel.py:91-108).
 * Splits: nsplit experts split_expert[], copies CSR split_ptr/split_gpus, fractions concatenated. */
int mbp_compute_loads(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* placement,
                      int32_t nsplit, const int32_t* split_expert, const int32_t* split_ptr,
                      const int32_t* split_gpus, const double* split_frac, double* loads, double* flow);

/* replicate.greedy_replicate (replicate.py:365-437).  Capacities: rep_experts[E], rep_ptr[E+1],
 * rep_gpus[E*G], frac[E*G*G].                                                                */
int mbp_greedy_replicate(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home, int64_t hidden,
                         int64_t inter, double flops, double bw_nv, double bw_rd, double bpt, int32_t slots,
                         int32_t* n_rep, int32_t* rep_experts, int32_t* rep_ptr, int32_t* rep_gpus, double* frac,
                         double* objective);

/* replicate.solve_token_split_lp (replicate.py:305-321) for a given placement; writes the
 * fractions of every replicated expert in ascending expert order (the LP insertion order).   */
int mbp_solve_token_split(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home, int64_t hidden,
                          int64_t inter, double flops, double bw_nv, double bw_rd, double bpt, int32_t n_rep,
                          const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus,
                          int32_t* out_experts, double* frac);

/* replicate.round_split (replicate.py:501-525): integer counts per (source, copy). */
int mbp_round_split(const double* x, int32_t G, int32_t E, const int64_t* home, int32_t n_rep,
                    const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus, const double* frac,
                    int64_t* counts);

/* sim._eplb_replication (sim.py:142-194); max_rep < 0 means unlimited. */
int mbp_eplb_replication(const double* loads, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home,
                         int32_t slots, int32_t max_rep, int32_t* n_rep, int32_t* rep_experts, int32_t* rep_ptr,
                         int32_t* rep_gpus);

/* sim._uniform_matrices (sim.py:127-139): rows of E u32 counts -> balanced rows, same sums. */
int mbp_uniform_matrices(const uint32_t* in, int64_t rows, int32_t E, uint32_t* out);

/* Dispatch tables for one (micro-batch, layer): the integer counterpart of flow_matrix with
 * round_split counts (no reference equivalent: the reference only models the flow).
 * counts: [G][1+R_e] blocks in rep order.  Outputs: route_tab[G][E][maxc][4]
 * {cum_end, dst_gpu, dst_row_base, 0}, ncopies[E], slot_tab[G][max_slots][4]
 * {row_begin, rows_real, rows_pad, expert}, slot_w[G][max_slots][2] {weight slot, replica},
 * nslots[G], total_rows[G], flow[G][G] rows src->dst.                                      */
int mbp_dispatch_plan(int32_t G, int32_t E, const int64_t* x, const int64_t* home, int32_t n_rep,
                      const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus,
                      const int64_t* counts, int32_t pad, int32_t maxc, int32_t max_slots, int32_t* route_tab,
                      int32_t* ncopies, int32_t* slot_tab, int32_t* slot_w, int32_t* nslots, int64_t* total_rows,
                      int64_t* flow);

#ifdef __cplusplus
}
#endif
#endif /* MB_PLANNER_H */
