/* pipefreeze host C-ABI (libpf_host.so).
 *
 * The reference exposes a C++ static-library API (namespace pipefreeze,
 * proj/include/pipefreeze/*.hpp) with no C ABI; libpf_host.so exports the same
 * C++ API and, for FFI consumers (Python ctypes here), the flat functions
 * below. Each cites the reference function it replaces.
 *
 * Conventions
 *   kind       0 gpipe, 1 1f1b, 2 interleaved-1f1b, 3 zbv  (ScheduleKind order),
 *              4 zbv-split (ZBV with B = dX and W = dW actions; not in the reference:
 *              3*M*S action nodes, plan ratios and masks keyed by the w nodes)
 *   plan[4]    {t_warmup, t_monitor, t_freeze, t_total}     (PhasePlan)
 *   node id    DAG node numbering of proj/src/dag.cpp:18-23: 0 = src,
 *              1 + [b ? M*S : 0] + (s-1)*M + (m-1), N-1 = dst; per-action
 *              arrays of length 2*M*S are indexed by node id - 1
 *   ratios     per backward action, index (s-1)*M + (m-1)
 *   masks      64-bit words, bit i of word i/64 = unit i frozen
 *              (FreezeMask::test, proj/include/pipefreeze/freezectl.hpp:47)
 *   status     PF_* codes of pf_status.h; pf_last_error() has the message
 */
#ifndef PIPEFREEZE_C_H
#define PIPEFREEZE_C_H

#include <stddef.h>
#include <stdint.h>

#include "pf_status.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* pf_last_error(void);

/* build_schedule (proj/include/pipefreeze/schedule.hpp:41). actions: R blocks of
 * 2*M*C triples (kind 0 f / 1 b / 2 w, microbatch, stage; 3*M*C for zbv-split);
 * lens[r] = actions on rank r. */
int pf_schedule_build(int kind, int R, int C, int M, int* actions, int* lens);
/* stage_to_rank (schedule.hpp:30) */
int pf_stage_to_rank(int kind, int R, int C, int M, int stage, int* rank);
/* The issue program of one rank (addition; the reference has no transport): its actions in
 * schedule order (build_schedule) with the P2P transfers of the cross-rank DAG rule-3 edges
 * (proj/src/dag.cpp:90-93) around each. ops: rows of 5 ints (kind, microbatch, stage,
 * recv_from rank or -1, send_to rank or -1); *n = rows (at most 3*M*C). The device trainer walks
 * exactly this program (trainer.cpp); tests/test_pipeline_p2p_gloo.py replays it over gloo. */
int pf_issue_program(int kind, int R, int C, int M, int rank, int* ops, int* n);

/* build_dag + topological_order + dag_to_json_text (dag.hpp:69, :45, :84).
 * edges: insertion order (from, to) pairs; json may be NULL. */
int pf_dag_build(int kind, int R, int C, int M, int* edges, int edge_cap, int* n_edges, int* topo,
                 char* json, int json_cap);
/* longest_path_start_times (dag.hpp:80): weights/start have N = 2*M*R*C + 2 entries. */
int pf_longest_path(int kind, int R, int C, int M, const double* weights, double* start,
                    double* makespan);
/* critical path through tight edges (not exported by the reference). */
int pf_critical_path(int kind, int R, int C, int M, const double* weights, int* nodes, int* len);

/* phase_of / actual_freeze_ratio (freezectl.hpp:31, :35) */
int pf_phase_of(int t, const int* plan, int* phase);
int pf_actual_freeze_ratio(int t, const int* plan, double expected_ratio, double* out);

/* Rng::next_u64 stream (types.hpp:50-56) */
int pf_rng_u64(uint64_t seed, int n, uint64_t* out);
/* `count` sample_mask calls on ONE Rng(seed) stream (freezectl.hpp:63) */
int pf_sample_masks(uint64_t seed, int n_units, int count, const double* ratios, uint64_t* words);
/* reconcile_mask with Rng(seed) (freezectl.hpp:68, Alg. 2) */
int pf_reconcile_mask(uint64_t seed, int n_units, const uint64_t* base, int target, uint64_t* out);

/* run_freezing_masks (freezectl.hpp:124) over the whole horizon: popcounts in
 * t->s->m order (plan[3]*S*M ints) and per-stage index hit counts (S*n longs). */
int pf_freezing_masks_horizon(int M, int S, const int* plan, const double* ratios, int n_units,
                              uint64_t seed, int* popcounts, long* stage_counts);
/* Jump-ahead into the same stream: the M masks of (step t, stage s), generated in
 * parallel; bit-identical to the sequential run. words: M * ceil(n/64).
 * *exact_parallel = 0 when a rejection event forced an in-order replay. */
int pf_mask_stream_stage_step(int M, int S, const int* plan, const double* ratios, int n_units,
                              uint64_t seed, int t, int s, uint64_t* words, int threads,
                              int* exact_parallel);
/* As pf_mask_stream_stage_step with per-stage unit counts stage_units[S] (stages of one
 * model differ: the first holds the embedding, the last the LM head). */
int pf_mask_stream_stage_step_units(int M, int S, const int* plan, const double* ratios, const int* stage_units,
                                    uint64_t seed, int t, int s, uint64_t* words, int threads, int* exact_parallel);
int pf_mask_stream_offset(int M, int S, const int* plan, const double* ratios, int n_units,
                          uint64_t seed, int t, int s, int m, uint64_t* offset);

/* build_lp + solve_lp + extract_freeze_plan (lp.hpp:52, :65, :83) on per-node
 * bounds (w_min/w_max: 2*M*R*C entries by node id - 1).
 * out5 = {makespan_base, makespan_opt, makespan_floor, lp_makespan, iterations}. */
int pf_plan_solve(int kind, int R, int C, int M, const double* w_min, const double* w_max,
                  double r_max, int lambda_mode, int budget_all, double* ratios,
                  double* durations, double* out5, double* stage_avg);
/* verify_solution (lp.hpp:114) for a plan given as ratios + durations. */
int pf_plan_verify(int kind, int R, int C, int M, const double* w_min, const double* w_max,
                   double r_max, const double* ratios, const double* durations,
                   double makespan_opt, int* ok, double* recomputed);
/* plan_weights (lp.cpp:275-286) */
int pf_plan_weights(int kind, int R, int C, int M, const double* w_min, const double* w_max,
                    const double* ratios, double afr_scale, double* weights);

/* aggregate_monitoring (timing.hpp:83) over n samples: node id - 1, step,
 * duration (ms), frozen flag (FreezeState::Full). Outputs per-node bounds.
 * Node ids >= 2*M*S are w nodes of a zbv-split DAG (3*M*S outputs; b nodes fixed). */
int pf_monitor_aggregate(int M, int S, int n, const int* node, const int* step,
                         const double* sample_ms, const int* frozen, double* w_min,
                         double* w_max);
/* run_monitoring + aggregate_monitoring (freezectl.hpp:119) on a stage-default
 * truth profile (per-stage fwd / bwd_act / bwd_param). */
int pf_simulate_monitoring(int M, int S, const double* fwd, const double* bact,
                           const double* bparam, const int* plan, double sigma, uint64_t seed,
                           double* w_min, double* w_max);

/* run_masked_sgd (sandbox.hpp:111) on a diagonal quadratic: policy 0 none,
 * 1 uniform_bernoulli(param = update probability), 2 uniform_exact_count(param =
 * freeze ratio). Outputs the final theta [d] and ||grad||^2 per step [steps]. */
int pf_masked_sgd_host(int d, const double* diag, const double* theta0, double eta, int M, int steps,
                       double sigma, int policy, double param, uint64_t seed, double* theta_out,
                       double* grad_sq_out);
/* run_masked_sgd with MaskPolicy::plan_driven (sandbox.cpp:97-115, per-coordinate Bernoulli of the
 * AFR of the coordinate's stage block at :158): ratios[(s-1)*M + (m-1)] = the plan's b(m,s) ratio,
 * phases = {T_w, T_m, T_f, T_total}, step < 0 = t_total. */
int pf_masked_sgd_plan_host(int d, const double* diag, const double* theta0, double eta, int M, int steps,
                            double sigma, int S, const double* ratios, const int* phases, int step, uint64_t seed,
                            double* theta_out, double* grad_sq_out);
/* AutoFreeze baseline (freezectl.hpp; freezectl.cpp:116-136): relative layer-norm change score and
 * the nearest-rank percentile prefix selection. */
int pf_autofreeze_score(double norm_prev, double norm_cur, double* out);
int pf_autofreeze_select(const double* scores, int n, int frozen_prefix_len, double percentile, int* out);

/* apf_update (freezectl.hpp:88) in fp64 on the host. */
int pf_apf_update_host(int n, double alpha, double* ema, double* ema_abs, const double* delta,
                       double* scores);

#ifdef __cplusplus
}
#endif

#endif
