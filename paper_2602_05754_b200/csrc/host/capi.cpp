// extern "C" surface of libpf_host.so (include/pipefreeze_c.h). Exceptions of
// the C++ layer map onto the reference's error taxonomy (pf_status.h).
#include <cstring>
#include <string>

#include "dag.hpp"
#include "freezectl.hpp"
#include "lp.hpp"
#include "pipefreeze_c.h"
#include "sandbox.hpp"
#include "schedule.hpp"
#include "timing.hpp"

using namespace pipefreeze;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return PF_OK;
  } catch (const config_error& e) {
    g_err = e.what();
    return PF_ERR_CONFIG;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return PF_ERR_DOMAIN;
  } catch (const numerical_error& e) {
    g_err = e.what();
    return PF_ERR_NUMERICAL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PF_ERR_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PF_ERR_INTERNAL;
  }
}

PipelineConfig make_cfg(int kind, int R, int C, int M) {
  if (kind < 0 || kind > 4) throw config_error("unknown schedule kind code " + std::to_string(kind));
  PipelineConfig c;
  c.schedule_kind = static_cast<ScheduleKind>(kind);
  c.num_ranks = R;
  c.stages_per_rank = C;
  c.num_microbatches = M;
  return c;
}

PhasePlan make_plan(const int* p) {
  if (!p) throw std::invalid_argument("null phase plan");
  return PhasePlan{p[0], p[1], p[2], p[3]};
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null pointer: ") + what);
}

TimingProfile profile_from_nodes(const PipelineDag& dag, const double* w_min, const double* w_max) {
  TimingProfile prof;
  for (int v = 1; v + 1 < dag.node_count(); ++v)
    prof.set_bounds(dag.action_at(v), {w_min[v - 1], w_max[v - 1]});
  return prof;
}

std::vector<double> ratio_vec(const double* r, int n) { return std::vector<double>(r, r + n); }

void copy_words(const FreezeMask& m, uint64_t* out) {
  std::memcpy(out, m.words().data(), m.words().size() * sizeof(uint64_t));
}

}  // namespace

extern "C" {

const char* pf_last_error(void) { return g_err.c_str(); }

int pf_schedule_build(int kind, int R, int C, int M, int* actions, int* lens) {
  return guard([&] {
    need(actions, "actions");
    need(lens, "lens");
    const auto tl = build_schedule(make_cfg(kind, R, C, M));
    int k = 0;
    for (int r = 0; r < R; ++r) {
      lens[r] = static_cast<int>(tl.rank_order[static_cast<std::size_t>(r)].size());
      for (const auto& a : tl.rank_order[static_cast<std::size_t>(r)]) {
        actions[k++] = static_cast<int>(a.kind);  // 0 f, 1 b, 2 w (zbv-split)
        actions[k++] = a.microbatch;
        actions[k++] = a.stage;
      }
    }
  });
}

int pf_stage_to_rank(int kind, int R, int C, int M, int stage, int* rank) {
  return guard([&] {
    need(rank, "rank");
    const auto c = make_cfg(kind, R, C, M);
    validate_config(c);
    *rank = stage_to_rank(c, stage);
  });
}

int pf_issue_program(int kind, int R, int C, int M, int rank, int* ops, int* n) {
  return guard([&] {
    need(ops, "ops");
    need(n, "n");
    const auto prog = issue_program(make_cfg(kind, R, C, M), rank);
    int i = 0;
    for (const auto& op : prog) {
      ops[5 * i] = static_cast<int>(op.action.kind);
      ops[5 * i + 1] = op.action.microbatch;
      ops[5 * i + 2] = op.action.stage;
      ops[5 * i + 3] = op.recv_from;
      ops[5 * i + 4] = op.send_to;
      ++i;
    }
    *n = i;
  });
}

int pf_dag_build(int kind, int R, int C, int M, int* edges, int edge_cap, int* n_edges, int* topo, char* json,
                 int json_cap) {
  return guard([&] {
    const auto dag = build_dag(build_schedule(make_cfg(kind, R, C, M)));
    const auto& e = dag.edges();
    if (n_edges) *n_edges = static_cast<int>(e.size());
    if (edges) {
      if (static_cast<int>(e.size()) > edge_cap) throw std::invalid_argument("edge buffer too small");
      for (std::size_t i = 0; i < e.size(); ++i) {
        edges[2 * i] = e[i].first;
        edges[2 * i + 1] = e[i].second;
      }
    }
    if (topo) {
      const auto order = dag.topological_order();
      std::copy(order->begin(), order->end(), topo);
    }
    if (json && json_cap > 0) {
      const auto s = dag_to_json_text(dag);
      if (static_cast<int>(s.size()) >= json_cap) throw std::invalid_argument("json buffer too small");
      std::memcpy(json, s.c_str(), s.size() + 1);
    }
  });
}

int pf_longest_path(int kind, int R, int C, int M, const double* weights, double* start, double* makespan) {
  return guard([&] {
    need(weights, "weights");
    const auto dag = build_dag(build_schedule(make_cfg(kind, R, C, M)));
    const auto st = longest_path_start_times(dag, std::vector<double>(weights, weights + dag.node_count()));
    if (start) std::copy(st.start.begin(), st.start.end(), start);
    if (makespan) *makespan = st.makespan;
  });
}

int pf_critical_path(int kind, int R, int C, int M, const double* weights, int* nodes, int* len) {
  return guard([&] {
    need(weights, "weights");
    need(nodes, "nodes");
    need(len, "len");
    const auto dag = build_dag(build_schedule(make_cfg(kind, R, C, M)));
    const auto path = critical_path(dag, std::vector<double>(weights, weights + dag.node_count()));
    *len = static_cast<int>(path.size());
    std::copy(path.begin(), path.end(), nodes);
  });
}

int pf_phase_of(int t, const int* plan, int* phase) {
  return guard([&] {
    need(phase, "phase");
    *phase = static_cast<int>(phase_of(t, make_plan(plan)));
  });
}

int pf_actual_freeze_ratio(int t, const int* plan, double r, double* out) {
  return guard([&] {
    need(out, "out");
    *out = actual_freeze_ratio(t, make_plan(plan), r);
  });
}

int pf_rng_u64(uint64_t seed, int n, uint64_t* out) {
  return guard([&] {
    need(out, "out");
    Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
  });
}

int pf_sample_masks(uint64_t seed, int n, int count, const double* ratios, uint64_t* words) {
  return guard([&] {
    need(ratios, "ratios");
    need(words, "words");
    Rng rng(seed);
    const int w = (n + 63) / 64;
    for (int c = 0; c < count; ++c) copy_words(sample_mask(n, ratios[c], rng), words + static_cast<std::size_t>(c) * static_cast<std::size_t>(w));
  });
}

int pf_reconcile_mask(uint64_t seed, int n, const uint64_t* base, int target, uint64_t* out) {
  return guard([&] {
    need(base, "base");
    need(out, "out");
    FreezeMask b(n);
    std::memcpy(b.words().data(), base, b.words().size() * sizeof(uint64_t));
    Rng rng(seed);
    copy_words(reconcile_mask(b, target, rng), out);
  });
}

int pf_freezing_masks_horizon(int M, int S, const int* plan, const double* ratios, int n, uint64_t seed,
                              int* popcounts, long* stage_counts) {
  return guard([&] {
    need(ratios, "ratios");
    std::map<ActionId, double> exp;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) exp[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
    Rng rng(seed);
    const auto h = run_freezing_masks(exp, make_plan(plan), M, S, n, rng);
    if (popcounts) {
      int k = 0;
      for (const auto& r : h.records()) popcounts[k++] = r.popcount;
    }
    if (stage_counts)
      for (int s = 0; s < S; ++s)
        for (int i = 0; i < n; ++i) {
          const auto& sc = h.stage_counts();
          stage_counts[static_cast<std::size_t>(s) * static_cast<std::size_t>(n) + static_cast<std::size_t>(i)] =
              static_cast<std::size_t>(s) < sc.size() && static_cast<std::size_t>(i) < sc[static_cast<std::size_t>(s)].size()
                  ? sc[static_cast<std::size_t>(s)][static_cast<std::size_t>(i)]
                  : 0;
        }
  });
}

int pf_mask_stream_stage_step(int M, int S, const int* plan, const double* ratios, int n, uint64_t seed, int t, int s,
                              uint64_t* words, int threads, int* exact_parallel) {
  return guard([&] {
    need(ratios, "ratios");
    need(words, "words");
    MaskStream ms(ratio_vec(ratios, M * S), make_plan(plan), M, S, n, seed);
    const bool ok = ms.stage_step_masks(t, s, words, threads);
    if (exact_parallel) *exact_parallel = ok ? 1 : 0;
  });
}

int pf_mask_stream_stage_step_units(int M, int S, const int* plan, const double* ratios, const int* stage_units,
                                    uint64_t seed, int t, int s, uint64_t* words, int threads, int* exact_parallel) {
  return guard([&] {
    need(ratios, "ratios");
    need(stage_units, "stage_units");
    need(words, "words");
    MaskStream ms(ratio_vec(ratios, M * S), make_plan(plan), M, std::vector<int>(stage_units, stage_units + S), seed);
    const bool ok = ms.stage_step_masks(t, s, words, threads);
    if (exact_parallel) *exact_parallel = ok ? 1 : 0;
  });
}

int pf_mask_stream_offset(int M, int S, const int* plan, const double* ratios, int n, uint64_t seed, int t, int s,
                          int m, uint64_t* offset) {
  return guard([&] {
    need(ratios, "ratios");
    need(offset, "offset");
    MaskStream ms(ratio_vec(ratios, M * S), make_plan(plan), M, S, n, seed);
    *offset = ms.offset(t, s, m);
  });
}

int pf_plan_solve(int kind, int R, int C, int M, const double* w_min, const double* w_max, double r_max,
                  int lambda_mode, int budget_all, double* ratios, double* durations, double* out5,
                  double* stage_avg) {
  return guard([&] {
    need(w_min, "w_min");
    need(w_max, "w_max");
    const auto cfg = make_cfg(kind, R, C, M);
    const int S = cfg.total_stages();
    const auto dag = build_dag(build_schedule(cfg));
    const auto prof = profile_from_nodes(dag, w_min, w_max);
    LpOptions opt;
    opt.lambda_mode = lambda_mode ? LambdaMode::Explicit : LambdaMode::Lexicographic;
    opt.budget_over_all_stage_nodes = budget_all != 0;
    const auto lp = build_lp(dag, prof, r_max, opt);
    const auto sol = solve_lp(lp, opt);
    const auto plan = extract_freeze_plan(dag, prof, sol, r_max, opt.tol);
    if (ratios)
      for (int s = 1; s <= S; ++s)
        for (int m = 1; m <= M; ++m) ratios[(s - 1) * M + (m - 1)] = plan.ratio_of(freeze_node(cfg, m, s));
    if (durations)
      for (int v = 1; v + 1 < dag.node_count(); ++v) durations[v - 1] = plan.durations.at(dag.action_at(v));
    if (out5) {
      out5[0] = plan.makespan_base;
      out5[1] = plan.makespan_opt;
      out5[2] = plan.makespan_floor;
      out5[3] = sol.makespan;
      out5[4] = static_cast<double>(sol.iterations);
    }
    if (stage_avg)
      for (int s = 1; s <= S; ++s) {
        const auto it = plan.stage_avg_ratio.find(s);
        stage_avg[s - 1] = it == plan.stage_avg_ratio.end() ? 0.0 : it->second;
      }
  });
}

int pf_plan_verify(int kind, int R, int C, int M, const double* w_min, const double* w_max, double r_max,
                   const double* ratios, const double* durations, double makespan_opt, int* ok, double* recomputed) {
  return guard([&] {
    need(ratios, "ratios");
    need(durations, "durations");
    const auto cfg = make_cfg(kind, R, C, M);
    const int S = cfg.total_stages();
    const auto dag = build_dag(build_schedule(cfg));
    const auto prof = profile_from_nodes(dag, w_min, w_max);
    FreezePlan plan;
    plan.r_max = r_max;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) plan.ratios[freeze_node(cfg, m, s)] = ratios[(s - 1) * M + (m - 1)];
    for (int v = 1; v + 1 < dag.node_count(); ++v) plan.durations[dag.action_at(v)] = durations[v - 1];
    plan.makespan_opt = makespan_opt;
    plan.makespan_base = longest_path_start_times(dag, prof.weights_max(dag)).makespan;
    const auto rep = verify_solution(dag, prof, plan, r_max);
    if (ok) *ok = rep.ok() ? 1 : 0;
    if (recomputed) *recomputed = rep.makespan_recomputed;
  });
}

int pf_plan_weights(int kind, int R, int C, int M, const double* w_min, const double* w_max, const double* ratios,
                    double afr_scale, double* weights) {
  return guard([&] {
    need(ratios, "ratios");
    need(weights, "weights");
    const auto cfg = make_cfg(kind, R, C, M);
    const int S = cfg.total_stages();
    const auto dag = build_dag(build_schedule(cfg));
    const auto prof = profile_from_nodes(dag, w_min, w_max);
    FreezePlan plan;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) plan.ratios[freeze_node(cfg, m, s)] = ratios[(s - 1) * M + (m - 1)];
    const auto w = plan_weights(dag, prof, plan, afr_scale);
    std::copy(w.begin(), w.end(), weights);
  });
}

int pf_monitor_aggregate(int M, int S, int n, const int* node, const int* step, const double* ms, const int* frozen,
                         double* w_min, double* w_max) {
  return guard([&] {
    need(node, "node");
    need(ms, "sample_ms");
    bool split = false;  // node ids past the backwards are w nodes (zbv-split dag)
    for (int i = 0; i < n; ++i) split |= node[i] >= 2 * M * S;
    PipelineDag dag(M, S, split);
    MonitorLog log;
    for (int i = 0; i < n; ++i)
      log.record(dag.action_at(node[i] + 1), step ? step[i] : 0, ms[i],
                 frozen && frozen[i] ? FreezeState::Full : FreezeState::None);
    const auto prof = aggregate_monitoring(log);
    for (int v = 1; v + 1 < dag.node_count(); ++v) {
      const auto& b = prof.bounds(dag.action_at(v));
      w_min[v - 1] = b.w_min;
      w_max[v - 1] = b.w_max;
    }
  });
}

int pf_simulate_monitoring(int M, int S, const double* fwd, const double* bact, const double* bparam, const int* plan,
                           double sigma, uint64_t seed, double* w_min, double* w_max) {
  return guard([&] {
    std::vector<StageTiming> st(static_cast<std::size_t>(S));
    for (int s = 0; s < S; ++s) st[static_cast<std::size_t>(s)] = {fwd[s], bact[s], bparam[s]};
    const auto truth = TimingProfile::from_stage_defaults(M, st);
    Rng rng(seed);
    const auto log = run_monitoring(truth, M, S, make_plan(plan), NoiseSpec{sigma}, rng);
    const auto prof = aggregate_monitoring(log);
    PipelineDag dag(M, S);
    for (int v = 1; v + 1 < dag.node_count(); ++v) {
      const auto& b = prof.bounds(dag.action_at(v));
      w_min[v - 1] = b.w_min;
      w_max[v - 1] = b.w_max;
    }
  });
}

int pf_masked_sgd_host(int d, const double* diag, const double* theta0, double eta, int M, int steps, double sigma,
                       int policy, double param, uint64_t seed, double* theta_out, double* grad_sq_out) {
  return guard([&] {
    need(diag, "diag");
    need(theta0, "theta0");
    const auto obj = SyntheticObjective::quadratic(Vec(diag, diag + d), sigma);
    const MaskPolicy pol = policy == 0   ? MaskPolicy::none()
                           : policy == 1 ? MaskPolicy::uniform_bernoulli(param)
                                         : MaskPolicy::uniform_exact_count(param);
    SgdHyper h;
    h.eta = eta;
    h.microbatches = M;
    h.total_steps = steps;
    const auto run = run_masked_sgd(obj, pol, h, Vec(theta0, theta0 + d), seed);
    if (theta_out) std::copy(run.theta_final.begin(), run.theta_final.end(), theta_out);
    if (grad_sq_out) std::copy(run.grad_sq_norms.begin(), run.grad_sq_norms.end(), grad_sq_out);
  });
}

int pf_masked_sgd_plan_host(int d, const double* diag, const double* theta0, double eta, int M, int steps,
                            double sigma, int S, const double* ratios, const int* phases, int step, uint64_t seed,
                            double* theta_out, double* grad_sq_out) {
  return guard([&] {
    need(diag, "diag");
    need(theta0, "theta0");
    need(ratios, "ratios");
    need(phases, "phases");
    const auto obj = SyntheticObjective::quadratic(Vec(diag, diag + d), sigma);
    FreezePlan plan;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) plan.ratios[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
    const PhasePlan ph{phases[0], phases[1], phases[2], phases[3]};
    const auto pol = MaskPolicy::plan_driven(plan, ph, M, S, step < 0 ? std::nullopt : std::optional<int>(step));
    SgdHyper h;
    h.eta = eta;
    h.microbatches = M;
    h.total_steps = steps;
    const auto run = run_masked_sgd(obj, pol, h, Vec(theta0, theta0 + d), seed);
    if (theta_out) std::copy(run.theta_final.begin(), run.theta_final.end(), theta_out);
    if (grad_sq_out) std::copy(run.grad_sq_norms.begin(), run.grad_sq_norms.end(), grad_sq_out);
  });
}

int pf_autofreeze_score(double norm_prev, double norm_cur, double* out) {
  return guard([&] {
    need(out, "out");
    *out = autofreeze_score(norm_prev, norm_cur);
  });
}

int pf_autofreeze_select(const double* scores, int n, int frozen_prefix_len, double percentile, int* out) {
  return guard([&] {
    need(scores, "scores");
    need(out, "out");
    *out = autofreeze_select(std::vector<double>(scores, scores + n), frozen_prefix_len, percentile);
  });
}

int pf_apf_update_host(int n, double alpha, double* ema, double* ema_abs, const double* delta, double* scores) {
  return guard([&] {
    need(ema, "ema");
    need(ema_abs, "ema_abs");
    need(delta, "delta");
    ApfState st{Vector(ema, ema + n), Vector(ema_abs, ema_abs + n), alpha};
    if (!(alpha > 0.0 && alpha < 1.0)) throw config_error("apf alpha must lie in (0, 1)");
    const auto sc = apf_update(st, std::vector<double>(delta, delta + n));
    std::copy(st.ema.begin(), st.ema.end(), ema);
    std::copy(st.ema_abs.begin(), st.ema_abs.end(), ema_abs);
    if (scores) std::copy(sc.begin(), sc.end(), scores);
  });
}

}  // extern "C"
