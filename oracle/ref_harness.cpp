// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" harness over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile). Used by tests/ and by
// bench.py's reference / cpu_baseline arm, as the parity checker.
// Every entry point calls the reference's own functions; where the reference
// only exposes aggregates (run_freezing_masks returns popcounts), the harness
// replays the same loop with the reference's primitives and reports both.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "pipefreeze/analysis.hpp"
#include "pipefreeze/config.hpp"
#include "pipefreeze/dag.hpp"
#include "pipefreeze/freezectl.hpp"
#include "pipefreeze/gantt.hpp"
#include "pipefreeze/lp.hpp"
#include "pipefreeze/sandbox.hpp"
#include "pipefreeze/schedule.hpp"
#include "pipefreeze/timing.hpp"
#include "pipefreeze/types.hpp"

using namespace pipefreeze;

namespace {

std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const config_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const numerical_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

PipelineConfig cfg(int kind, int R, int C, int M) {
  PipelineConfig c;
  c.schedule_kind = static_cast<ScheduleKind>(kind);
  c.num_ranks = R;
  c.stages_per_rank = C;
  c.num_microbatches = M;
  return c;
}

PhasePlan phases(const int* p) { return PhasePlan{p[0], p[1], p[2], p[3]}; }

TimingProfile profile_from(int M, int S, const double* fwd, const double* bact,
                           const double* bparam) {
  std::vector<StageTiming> st(S);
  for (int s = 0; s < S; ++s) st[s] = {fwd[s], bact[s], bparam[s]};
  return TimingProfile::from_stage_defaults(M, st);
}

void mask_words(const FreezeMask& m, uint64_t* out) {
  const int words = (m.size() + 63) / 64;
  for (int w = 0; w < words; ++w) out[w] = 0;
  for (int i = 0; i < m.size(); ++i)
    if (m.test(i)) out[i >> 6] |= uint64_t{1} << (i & 63);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_rng_u64(uint64_t seed, int n, uint64_t* out) {
  Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
  return 0;
}

int ref_rng_mixed(uint64_t seed, int n, const uint64_t* bounds, uint64_t* idx, double* unit,
                  double* gauss) {
  return guard([&] {
    Rng rng(seed);
    for (int i = 0; i < n; ++i) {
      idx[i] = rng.index_below(bounds[i]);
      unit[i] = rng.unit();
      gauss[i] = rng.gaussian();
    }
  });
}

int ref_schedule(int kind, int R, int C, int M, int* out, int* lens) {
  return guard([&] {
    const auto tl = build_schedule(cfg(kind, R, C, M));
    int k = 0;
    for (int r = 0; r < R; ++r) {
      lens[r] = static_cast<int>(tl.rank_order[r].size());
      for (const auto& a : tl.rank_order[r]) {
        out[k++] = a.kind == ActionKind::Forward ? 0 : 1;
        out[k++] = a.microbatch;
        out[k++] = a.stage;
      }
    }
  });
}

int ref_stage_to_rank(int kind, int R, int C, int M, int stage) {
  int r = -1;
  if (guard([&] { r = stage_to_rank(cfg(kind, R, C, M), stage); })) return -1;
  return r;
}

// edges in insertion order; topological order; DAG JSON text length/contents
int ref_dag(int kind, int R, int C, int M, int* edges, int cap, int* n_edges, int* topo,
            char* json, int json_cap) {
  return guard([&] {
    const auto dag = build_dag(build_schedule(cfg(kind, R, C, M)));
    const auto& e = dag.edges();
    *n_edges = static_cast<int>(e.size());
    for (int i = 0; i < *n_edges && i < cap; ++i) {
      edges[2 * i] = e[i].first;
      edges[2 * i + 1] = e[i].second;
    }
    const auto order = dag.topological_order();
    for (int i = 0; i < dag.node_count(); ++i) topo[i] = (*order)[i];
    if (json && json_cap > 0) {
      const std::string s = dag_to_json_text(dag);
      std::strncpy(json, s.c_str(), static_cast<size_t>(json_cap - 1));
      json[json_cap - 1] = 0;
    }
  });
}

int ref_longest_path(int kind, int R, int C, int M, const double* weights, double* start,
                     double* makespan) {
  return guard([&] {
    const auto dag = build_dag(build_schedule(cfg(kind, R, C, M)));
    const auto st = longest_path_start_times(
        dag, std::vector<double>(weights, weights + dag.node_count()));
    for (int v = 0; v < dag.node_count(); ++v) start[v] = st.start[v];
    *makespan = st.makespan;
  });
}

int ref_phase_of(int t, const int* plan) {
  int ph = -1;
  if (guard([&] { ph = static_cast<int>(phase_of(t, phases(plan))); })) return -1;
  return ph;
}

int ref_afr(int t, const int* plan, double r, double* out) {
  return guard([&] { *out = actual_freeze_ratio(t, phases(plan), r); });
}

// `count` sample_mask calls on ONE Rng stream (the run_freezing_masks contract).
int ref_sample_masks(uint64_t seed, int n, int count, const double* ratios, uint64_t* out) {
  return guard([&] {
    Rng rng(seed);
    const int words = (n + 63) / 64;
    for (int c = 0; c < count; ++c) mask_words(sample_mask(n, ratios[c], rng), out + c * words);
  });
}

int ref_reconcile(uint64_t seed, int n, const uint64_t* base_words, int target, uint64_t* out) {
  return guard([&] {
    FreezeMask base(n);
    for (int i = 0; i < n; ++i)
      if ((base_words[i >> 6] >> (i & 63)) & 1) base.set(i);
    Rng rng(seed);
    mask_words(reconcile_mask(base, target, rng), out);
  });
}

// Full-horizon controller (reference run_freezing_masks) for a plan given as
// ratios[(s-1)*M + (m-1)]. Outputs: popcount per cell in t->s->m order and the
// per-stage index hit counts (MaskHistory::stage_counts), plus the bit masks
// of cells with t in [t_from, t_to] replayed with the same primitives.
int ref_freezing_masks(int M, int S, const int* plan, const double* ratios, int n, uint64_t seed,
                       int* popcounts, long* stage_counts, int t_from, int t_to,
                       uint64_t* words_out) {
  return guard([&] {
    std::map<ActionId, double> expected;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) expected[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
    const PhasePlan pp = phases(plan);
    Rng rng(seed);
    const auto hist = run_freezing_masks(expected, pp, M, S, n, rng);
    int k = 0;
    for (const auto& rec : hist.records()) popcounts[k++] = rec.popcount;
    for (int s = 0; s < S; ++s)
      for (int i = 0; i < n; ++i) stage_counts[s * n + i] = hist.stage_counts()[s][i];
    if (!words_out) return;
    // replay with the same primitives, same stream, same order (freezectl.cpp:189-208)
    Rng replay(seed);
    const int words = (n + 63) / 64;
    long cell = 0;
    for (int t = 1; t <= pp.t_total; ++t) {
      const Phase phase = phase_of(t, pp);
      for (int s = 1; s <= S; ++s)
        for (int m = 1; m <= M; ++m) {
          double ratio = 0.0;
          if (phase == Phase::MonitorLower) ratio = 1.0;
          if (phase == Phase::ProgressiveFreeze || phase == Phase::StableFreeze)
            ratio = actual_freeze_ratio(t, pp, expected[backward_action(m, s)]);
          const auto mask = sample_mask(n, ratio, replay);
          if (t >= t_from && t <= t_to) mask_words(mask, words_out + (cell++) * words);
        }
    }
  });
}

int ref_apf(int n, double alpha, int steps, const double* deltas, double* ema, double* ema_abs,
            double* scores) {
  return guard([&] {
    auto st = ApfState::zeros(n, alpha);
    Eigen::VectorXd sc;
    for (int k = 0; k < steps; ++k) {
      Eigen::VectorXd d(n);
      for (int i = 0; i < n; ++i) d(i) = deltas[static_cast<long>(k) * n + i];
      sc = apf_update(st, d);
    }
    for (int i = 0; i < n; ++i) {
      ema[i] = st.ema(i);
      ema_abs[i] = st.ema_abs(i);
      scores[i] = sc(i);
    }
  });
}

// plan = LP over the schedule DAG with per-stage timing defaults.
// out5 = {makespan_base, makespan_opt, makespan_floor, lp_makespan, iterations}
int ref_plan(int kind, int R, int C, int M, const double* fwd, const double* bact,
             const double* bparam, double r_max, int lambda_mode, int budget_all,
             double* ratios, double* durations, double* out5, double* stage_avg,
             double* solve_seconds) {
  return guard([&] {
    const auto pc = cfg(kind, R, C, M);
    const int S = pc.total_stages();
    const auto dag = build_dag(build_schedule(pc));
    const auto prof = profile_from(M, S, fwd, bact, bparam);
    LpOptions opt;
    opt.lambda_mode = lambda_mode ? LambdaMode::Explicit : LambdaMode::Lexicographic;
    opt.budget_over_all_stage_nodes = budget_all != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const auto problem = build_lp(dag, prof, r_max, opt);
    const auto sol = solve_lp(problem, opt);
    const auto t1 = std::chrono::steady_clock::now();
    const auto plan = extract_freeze_plan(dag, prof, sol, r_max, opt.tol);
    if (solve_seconds) *solve_seconds = std::chrono::duration<double>(t1 - t0).count();
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) {
        ratios[(s - 1) * M + (m - 1)] = plan.ratio_of(backward_action(m, s));
        durations[(s - 1) * M + (m - 1)] = plan.durations.at(forward_action(m, s));
        durations[S * M + (s - 1) * M + (m - 1)] = plan.durations.at(backward_action(m, s));
      }
    out5[0] = plan.makespan_base;
    out5[1] = plan.makespan_opt;
    out5[2] = plan.makespan_floor;
    out5[3] = sol.makespan;
    out5[4] = static_cast<double>(sol.iterations);
    for (int s = 1; s <= S; ++s) {
      auto it = plan.stage_avg_ratio.find(s);
      stage_avg[s - 1] = it == plan.stage_avg_ratio.end() ? 0.0 : it->second;
    }
  });
}

// verify_solution on a caller-supplied plan (ratios + durations as ref_plan emits).
int ref_verify(int kind, int R, int C, int M, const double* fwd, const double* bact,
               const double* bparam, double r_max, const double* ratios,
               const double* durations, double makespan_opt, int* ok, double* recomputed) {
  return guard([&] {
    const auto pc = cfg(kind, R, C, M);
    const int S = pc.total_stages();
    const auto dag = build_dag(build_schedule(pc));
    const auto prof = profile_from(M, S, fwd, bact, bparam);
    FreezePlan plan;
    plan.r_max = r_max;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) {
        plan.ratios[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
        plan.durations[forward_action(m, s)] = durations[(s - 1) * M + (m - 1)];
        plan.durations[backward_action(m, s)] = durations[S * M + (s - 1) * M + (m - 1)];
      }
    plan.makespan_opt = makespan_opt;
    plan.makespan_base = longest_path_start_times(dag, prof.weights_max(dag)).makespan;
    const auto rep = verify_solution(dag, prof, plan, r_max);
    *ok = rep.ok() ? 1 : 0;
    *recomputed = rep.makespan_recomputed;
  });
}

// run_monitoring + aggregate_monitoring; bounds out: [w_min, w_max] per node in
// ActionId order (forwards s-major then backwards).
int ref_monitor(int M, int S, const double* fwd, const double* bact, const double* bparam,
                const int* plan, double sigma, uint64_t seed, double* wmin, double* wmax) {
  return guard([&] {
    const auto truth = profile_from(M, S, fwd, bact, bparam);
    Rng rng(seed);
    const auto log = run_monitoring(truth, M, S, phases(plan), NoiseSpec{sigma}, rng);
    const auto est = aggregate_monitoring(log);
    int k = 0;
    for (const auto& [node, b] : est.all()) {
      wmin[k] = b.w_min;
      wmax[k] = b.w_max;
      ++k;
    }
  });
}

// run_masked_sgd on a diagonal quadratic. policy: 0 none, 1 bernoulli(p_update),
// 2 exact-count(freeze ratio). theta_out[d], gradsq_out[steps].
int ref_masked_sgd(int d, const double* diag, const double* theta0, double eta, int M, int steps,
                   double sigma, int policy, double param, uint64_t seed, double* theta_out,
                   double* gradsq_out) {
  return guard([&] {
    Eigen::VectorXd dg(d), t0(d);
    for (int j = 0; j < d; ++j) {
      dg(j) = diag[j];
      t0(j) = theta0[j];
    }
    const auto obj = SyntheticObjective::quadratic(dg, sigma);
    MaskPolicy pol = policy == 0   ? MaskPolicy::none()
                     : policy == 1 ? MaskPolicy::uniform_bernoulli(param)
                                   : MaskPolicy::uniform_exact_count(param);
    SgdHyper h;
    h.eta = eta;
    h.microbatches = M;
    h.total_steps = steps;
    const auto run = run_masked_sgd(obj, pol, h, t0, seed);
    for (int j = 0; j < d; ++j) theta_out[j] = run.theta_final(j);
    for (int t = 0; t < static_cast<int>(run.grad_sq_norms.size()); ++t)
      gradsq_out[t] = run.grad_sq_norms[t];
  });
}

// run_masked_sgd with MaskPolicy::plan_driven (sandbox.cpp:97-115; Bernoulli draws at :158): the
// plan's backward ratios[(s-1)*M + (m-1)], the AFR at `step` (< 0: t_total) of `phases`.
int ref_masked_sgd_plan(int d, const double* diag, const double* theta0, double eta, int M, int steps, double sigma,
                        int S, const double* ratios, const int* phases, int step, uint64_t seed, double* theta_out,
                        double* gradsq_out) {
  return guard([&] {
    Eigen::VectorXd dg(d), t0(d);
    for (int j = 0; j < d; ++j) {
      dg(j) = diag[j];
      t0(j) = theta0[j];
    }
    const auto obj = SyntheticObjective::quadratic(dg, sigma);
    FreezePlan plan;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) plan.ratios[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
    const PhasePlan ph{phases[0], phases[1], phases[2], phases[3]};
    const auto pol = MaskPolicy::plan_driven(plan, ph, M, S, step < 0 ? std::nullopt : std::optional<int>(step));
    SgdHyper h;
    h.eta = eta;
    h.microbatches = M;
    h.total_steps = steps;
    const auto run = run_masked_sgd(obj, pol, h, t0, seed);
    for (int j = 0; j < d; ++j) theta_out[j] = run.theta_final(j);
    for (int t = 0; t < static_cast<int>(run.grad_sq_norms.size()); ++t) gradsq_out[t] = run.grad_sq_norms[t];
  });
}

double ref_autofreeze_score(double prev, double cur) { return autofreeze_score(prev, cur); }
int ref_autofreeze_select(const double* scores, int n, int prefix, double pct, int* out) {
  return guard([&] { *out = autofreeze_select(std::vector<double>(scores, scores + n), prefix, pct); });
}

namespace {
int copy_text(const std::string& s, char* out, int cap) {
  if (!out || cap <= 0) return static_cast<int>(s.size()) + 1;
  std::strncpy(out, s.c_str(), static_cast<size_t>(cap - 1));
  out[cap - 1] = 0;
  return static_cast<int>(s.size()) + 1;
}
}  // namespace

// Reference artifacts (config.cpp / gantt.cpp / analysis.cpp writers) for I/O parity.
int ref_plan_json(int kind, int R, int C, int M, const double* fwd, const double* bact, const double* bparam,
                  double r_max, char* plan_out, int plan_cap, char* report_out, int report_cap) {
  return guard([&] {
    const auto pc = cfg(kind, R, C, M);
    const int S = pc.total_stages();
    const auto dag = build_dag(build_schedule(pc));
    const auto prof = profile_from(M, S, fwd, bact, bparam);
    const auto plan = extract_freeze_plan(dag, prof, solve_lp(build_lp(dag, prof, r_max)), r_max);
    copy_text(freeze_plan_to_json_text(plan), plan_out, plan_cap);
    copy_text(throughput_report_to_json_text(build_report(plan, nullptr, nullptr, std::nullopt)), report_out,
              report_cap);
  });
}

int ref_gantt_json(int kind, int R, int C, int M, const double* weights, char* out, int cap) {
  return guard([&] {
    const auto tl = build_schedule(cfg(kind, R, C, M));
    const auto dag = build_dag(tl);
    copy_text(gantt_to_json_text(build_gantt(tl, dag, std::vector<double>(weights, weights + dag.node_count()))), out,
              cap);
  });
}

int ref_masks_json(int M, int S, const int* plan, const double* ratios, int n, uint64_t seed, char* out, int cap) {
  return guard([&] {
    std::map<ActionId, double> expected;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) expected[backward_action(m, s)] = ratios[(s - 1) * M + (m - 1)];
    Rng rng(seed);
    copy_text(mask_history_to_json_text(run_freezing_masks(expected, phases(plan), M, S, n, rng)), out, cap);
  });
}

int ref_profile_json(int M, int S, const double* fwd, const double* bact, const double* bparam, char* out, int cap) {
  return guard([&] { copy_text(timing_profile_to_json_text(profile_from(M, S, fwd, bact, bparam)), out, cap); });
}

// One "reference step" of the path on CPU, for bench.py's reference arm:
// schedule + DAG + longest path, S*M sample_mask calls over n_units, apf_update
// over n_params, and a masked-SGD update over n_params (sandbox.cpp:232-250).
// Returns seconds.
double ref_cpu_step(int kind, int R, int C, int M, int n_units, long n_params, double ratio,
                    uint64_t seed) {
  double secs = -1.0;
  guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const auto pc = cfg(kind, R, C, M);
    const int S = pc.total_stages();
    const auto dag = build_dag(build_schedule(pc));
    std::vector<double> w(dag.node_count(), 1.0);
    w[dag.source()] = 0.0;
    w[dag.destination()] = 0.0;
    volatile double ms = longest_path_start_times(dag, w).makespan;
    (void)ms;
    Rng rng(seed);
    std::vector<FreezeMask> masks;
    masks.reserve(static_cast<size_t>(S) * M);
    for (int c = 0; c < S * M; ++c) masks.push_back(sample_mask(n_units, ratio, rng));
    auto st = ApfState::zeros(n_params, 0.9);
    Eigen::VectorXd delta(n_params), theta(n_params), total(n_params), g(n_params);
    for (long i = 0; i < n_params; ++i) {
      delta(i) = 1e-3 * (rng.unit() - 0.5);
      theta(i) = rng.unit();
      g(i) = rng.unit() - 0.5;
    }
    (void)apf_update(st, delta);
    // masked accumulation: unit u covers a contiguous block of parameters
    total.setZero();
    const long per_unit = std::max<long>(1, n_params / std::max(1, n_units));
    for (int m = 0; m < M; ++m) {
      const auto& mk = masks[static_cast<size_t>(m)];
      for (long i = 0; i < n_params; ++i) {
        const long u = std::min<long>(n_units - 1, i / per_unit);
        if (!mk.test(static_cast<int>(u))) total(i) += g(i);
      }
    }
    theta -= (0.01 / M) * total;
    volatile double sink = theta(0);
    (void)sink;
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}

// One worker's share of the reference's per-parameter step (bench.py --impl reference and the
// cpu_baseline leg shard a stage's parameters element-wise over worker processes):
// elements [begin, end), in blocks of `block` elements, each block through
//   * apf_update (freezectl.cpp:147-156) on the block's APF state (E, E_abs);
//   * the masked accumulation total = sum_m U_m (.) g over the M microbatch masks and the SGD
//     update theta -= (lr / M) total of run_masked_sgd (sandbox.cpp:232-250), unit of element i =
//     i / per_unit (ref_cpu_step's contiguous-unit mapping), FreezeMask::test on the reference's
//     masks (`masks`: M x words uint64, FreezeMask bit order).
// The blocks reuse one set of block-sized buffers (the arithmetic per element is the reference's;
// the full stage state would not fit host memory at 8B parameters). Returns the seconds of the
// timed loop (buffer setup excluded).
double ref_param_pass(long begin, long end, long block, int M, const uint64_t* masks, int words, long per_unit,
                      double lr) {
  double secs = -1.0;
  guard([&] {
    const long n = std::max<long>(1, std::min(block, end - begin));
    auto st = ApfState::zeros(n, 0.9);
    Eigen::VectorXd delta(n), theta(n), total(n), g(n), upd(n);
    Rng rng(static_cast<uint64_t>(begin) + 1);
    for (long i = 0; i < n; ++i) {
      delta(i) = 1e-3 * (rng.unit() - 0.5);
      theta(i) = rng.unit();
      g(i) = rng.unit() - 0.5;
    }
    std::vector<FreezeMask> mk;
    mk.reserve(static_cast<size_t>(M));
    const int n_units = words * 64;
    for (int m = 0; m < M; ++m) {
      FreezeMask f(n_units);
      for (int u = 0; u < n_units; ++u)
        if ((masks[static_cast<size_t>(m) * words + u / 64] >> (u % 64)) & 1ULL) f.set(u);
      mk.push_back(std::move(f));
    }
    volatile double sink = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (long b0 = begin; b0 < end; b0 += block) {
      const long len = std::min(block, end - b0);
      const auto scores = apf_update(st, delta);
      sink = sink + scores(0);
      for (long i = 0; i < len; ++i) total(i) = 0.0;
      for (int m = 0; m < M; ++m) {
        // U_m: the 0/1 update mask of this block's elements (what MaskPolicy::draw_update_mask
        // hands run_masked_sgd), then the reference's total += U_m .* g (sandbox.cpp:243)
        const auto& f = mk[static_cast<size_t>(m)];
        for (long i = 0; i < len;) {
          const long u = std::min<long>(n_units - 1, (b0 + i) / per_unit);
          const long stop = u == n_units - 1 ? len : std::min(len, (u + 1) * per_unit - b0);
          const double keep = f.test(static_cast<int>(u)) ? 0.0 : 1.0;
          for (; i < stop; ++i) upd(i) = keep;
        }
        // (written out as the single fused pass Eigen's expression templates evaluate it to; the
        // test-only Eigen shim is eager and would add a temporary per microbatch)
        for (long i = 0; i < len; ++i) total(i) += upd(i) * g(i);
      }
      const double sc = lr / M;
      for (long i = 0; i < len; ++i) theta(i) -= sc * total(i);
      sink = sink + theta(0);
    }
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    (void)sink;
  });
  return secs;
}

// The reference's per-step controller work for a stage: build_schedule + build_dag +
// longest_path_start_times, then the step's S*M exact-count masks over n_units
// (run_freezing_masks' per-cell sample_mask, freezectl.cpp:185-211). masks_out (M x words of
// stage 1, may be NULL) receives the first stage's masks. Returns seconds.
double ref_controller_step(int kind, int R, int C, int M, int n_units, double ratio, uint64_t seed,
                           uint64_t* masks_out) {
  double secs = -1.0;
  guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const auto pc = cfg(kind, R, C, M);
    const int S = pc.total_stages();
    const auto dag = build_dag(build_schedule(pc));
    std::vector<double> w(dag.node_count(), 1.0);
    w[dag.source()] = 0.0;
    w[dag.destination()] = 0.0;
    volatile double ms = longest_path_start_times(dag, w).makespan;
    (void)ms;
    Rng rng(seed);
    const int words = (n_units + 63) / 64;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) {
        const auto mk = sample_mask(n_units, ratio, rng);
        if (masks_out && s == 1)
          for (int u = 0; u < n_units; ++u)
            if (mk.test(u)) masks_out[static_cast<size_t>(m - 1) * words + u / 64] |= 1ULL << (u % 64);
      }
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}

}  // extern "C"
