// Freeze controller (proj/src/freezectl.cpp). Phase machine :28-38, AFR ramp
// :40-52, exact-count masks :77-98, reconciliation :100-114, AutoFreeze
// :116-136, APF :138-163, monitoring driver :165-183, horizon driver :185-211.
#include "freezectl.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <numeric>
#include <thread>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace pipefreeze {

void validate_phase_plan(const PhasePlan& p) {
  if (!(0 < p.t_warmup && p.t_warmup < p.t_monitor && p.t_monitor <= p.t_freeze && p.t_freeze <= p.t_total))
    throw config_error("phase plan must satisfy 0 < T_w < T_m <= T_f <= T_total");
}

std::string to_string(Phase phase) {
  switch (phase) {
    case Phase::Warmup: return "warmup";
    case Phase::MonitorUpper: return "monitor-upper";
    case Phase::MonitorLower: return "monitor-lower";
    case Phase::Solve: return "solve";
    case Phase::ProgressiveFreeze: return "progressive-freeze";
    case Phase::StableFreeze: return "stable-freeze";
  }
  return "unknown";
}

Phase phase_of(int t, const PhasePlan& p) {
  if (t < 1 || t > p.t_total)
    throw std::domain_error("step " + std::to_string(t) + " outside [1, " + std::to_string(p.t_total) + "]");
  if (t <= p.t_warmup) return Phase::Warmup;
  if (t == p.t_monitor) return Phase::Solve;
  if (t <= p.t_mid()) return Phase::MonitorUpper;
  if (t < p.t_monitor) return Phase::MonitorLower;
  return t <= p.t_freeze ? Phase::ProgressiveFreeze : Phase::StableFreeze;
}

double actual_freeze_ratio(int t, const PhasePlan& p, double r) {
  if (r < 0.0 || r > 1.0) throw std::domain_error("expected ratio must be in [0, 1]");
  if (p.t_freeze == p.t_monitor) return r;
  const double ramp = static_cast<double>(t - p.t_monitor) / static_cast<double>(p.t_freeze - p.t_monitor);
  return std::min(r, r * ramp);
}

double afr_at(int t, const PhasePlan& p, double r) { return t <= p.t_monitor ? 0.0 : actual_freeze_ratio(t, p, r); }

int FreezeMask::popcount() const {
  int c = 0;
  for (auto w : words_) c += std::popcount(w);
  return c;
}

std::vector<int> FreezeMask::set_indices() const {
  std::vector<int> out;
  for (int i = 0; i < n_; ++i)
    if (test(i)) out.push_back(i);
  return out;
}

std::vector<int> FreezeMask::unset_indices() const {
  std::vector<int> out;
  for (int i = 0; i < n_; ++i)
    if (!test(i)) out.push_back(i);
  return out;
}

namespace {

// Partial Fisher-Yates: positions [0, k) of `pool` receive k distinct draws.
// Returns the number of RNG outputs consumed (k unless rejection occurred).
std::uint64_t partial_shuffle(int* pool, int n, int k, Rng& rng) {
  const std::uint64_t before = rng.state();
  for (int i = 0; i < k; ++i) {
    const int j = i + static_cast<int>(rng.index_below(static_cast<std::uint64_t>(n - i)));
    std::swap(pool[i], pool[j]);
  }
  // state advances by gamma per output; gamma is odd, so divide via its inverse mod 2^64
  constexpr std::uint64_t kGammaInv = [] {
    std::uint64_t x = Rng::kGamma;  // Newton iteration for the 2-adic inverse
    for (int it = 0; it < 6; ++it) x *= 2 - Rng::kGamma * x;
    return x;
  }();
  return (rng.state() - before) * kGammaInv;
}

void fill_words(const int* idx, int k, std::uint64_t* words, int nwords) {
  std::fill(words, words + nwords, 0);
  for (int i = 0; i < k; ++i) words[idx[i] >> 6] |= std::uint64_t{1} << (idx[i] & 63);
}

std::vector<int>& scratch_pool(int n) {
  thread_local std::vector<int> pool;
  pool.resize(static_cast<std::size_t>(n));
  std::iota(pool.begin(), pool.end(), 0);
  return pool;
}

}  // namespace

int mask_count(int n, double ratio) { return static_cast<int>(std::floor(ratio * n)); }

FreezeMask sample_mask(int n, double ratio, Rng& rng) {
  if (ratio < 0.0 || ratio > 1.0) throw std::domain_error("mask ratio must be in [0, 1]");
  if (n < 0) throw std::domain_error("n_params must be nonnegative");
  FreezeMask mask(n);
  const int k = mask_count(n, ratio);
  if (k == 0) return mask;
  auto& pool = scratch_pool(n);
  partial_shuffle(pool.data(), n, k, rng);
  fill_words(pool.data(), k, mask.words().data(), static_cast<int>(mask.words().size()));
  return mask;
}

FreezeMask reconcile_mask(const FreezeMask& base, int target, Rng& rng) {
  if (target < 0 || target > base.size()) throw std::domain_error("target_count must be in [0, n_params]");
  const int have = base.popcount();
  if (have == target) return base;
  FreezeMask out = base;
  const bool grow = have < target;
  std::vector<int> pool = grow ? base.unset_indices() : base.set_indices();
  const int k = grow ? target - have : have - target;
  partial_shuffle(pool.data(), static_cast<int>(pool.size()), k, rng);
  for (int i = 0; i < k; ++i) grow ? out.set(pool[static_cast<std::size_t>(i)]) : out.reset(pool[static_cast<std::size_t>(i)]);
  return out;
}

double autofreeze_score(double prev, double cur) {
  if (prev <= 0.0) throw std::domain_error("previous gradient norm must be positive");
  return std::abs(prev - cur) / prev;
}

int autofreeze_select(const std::vector<double>& scores, int prefix, double percentile) {
  const int L = static_cast<int>(scores.size());
  if (prefix < 0 || prefix > L) throw std::domain_error("frozen prefix out of range");
  if (L == 0 || prefix == L) return prefix;
  std::vector<double> sorted = scores;
  std::sort(sorted.begin(), sorted.end());
  const int rank = std::max(1, static_cast<int>(std::ceil(percentile / 100.0 * L)));
  const double threshold = sorted[static_cast<std::size_t>(std::min(rank, L) - 1)];
  while (prefix < L && scores[static_cast<std::size_t>(prefix)] < threshold) ++prefix;
  return prefix;
}

ApfState ApfState::zeros(std::size_t n, double alpha) {
  if (!(alpha > 0.0 && alpha < 1.0)) throw config_error("apf alpha must lie in (0, 1)");
  return ApfState{Vector(n, 0.0), Vector(n, 0.0), alpha};
}

Vector apf_update(ApfState& st, const std::vector<double>& delta) {
  if (delta.size() != st.ema.size()) throw std::domain_error("apf update dimension mismatch");
  const double a = st.alpha, b = 1.0 - st.alpha;
  std::vector<double> score(delta.size());
  for (std::size_t i = 0; i < delta.size(); ++i) {
    st.ema[i] = a * st.ema[i] + b * delta[i];
    st.ema_abs[i] = a * st.ema_abs[i] + b * std::abs(delta[i]);
    score[i] = st.ema_abs[i] == 0.0 ? 1.0 : std::abs(st.ema[i]) / st.ema_abs[i];
  }
  return score;
}

std::vector<int> apf_eligible(const std::vector<double>& scores, double threshold) {
  std::vector<int> out;
  for (std::size_t i = 0; i < scores.size(); ++i)
    if (scores[i] < threshold) out.push_back(static_cast<int>(i));
  return out;
}

void MaskHistory::add(int step, const ActionId& action, const FreezeMask& mask) {
  records_.push_back(MaskRecord{step, action.stage, action, mask.popcount(), mask.size()});
  const auto si = static_cast<std::size_t>(action.stage - 1);
  if (stage_counts_.size() <= si) {
    stage_counts_.resize(si + 1);
    stage_draws_.resize(si + 1, 0);
  }
  auto& counts = stage_counts_[si];
  if (counts.size() < static_cast<std::size_t>(mask.size())) counts.resize(static_cast<std::size_t>(mask.size()), 0);
  const auto& w = mask.words();
  for (std::size_t wi = 0; wi < w.size(); ++wi)
    for (std::uint64_t bits = w[wi]; bits; bits &= bits - 1)
      ++counts[wi * 64 + static_cast<std::size_t>(std::countr_zero(bits))];
  ++stage_draws_[si];
}

MonitorLog run_monitoring(const TimingProfile& truth, int M, int S, const PhasePlan& phases,
                          const NoiseSpec& noise, Rng& rng) {
  MonitorLog log;
  for (int t = phases.t_warmup + 1; t <= phases.t_monitor; ++t) {
    const Phase ph = phase_of(t, phases);
    if (ph != Phase::MonitorUpper && ph != Phase::MonitorLower) continue;
    const bool upper = ph == Phase::MonitorUpper;
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) {
        const ActionId f = forward_action(m, s), b = backward_action(m, s);
        log.record(f, t, sample_execution(truth, f, upper ? 0.0 : 1.0, noise, rng), FreezeState::None);
        log.record(b, t, sample_execution(truth, b, upper ? 0.0 : 1.0, noise, rng),
                   upper ? FreezeState::None : FreezeState::Full);
      }
  }
  return log;
}

double cell_ratio(int t, const PhasePlan& phases, double expected) {
  switch (phase_of(t, phases)) {
    case Phase::MonitorLower: return 1.0;
    case Phase::ProgressiveFreeze:
    case Phase::StableFreeze: return actual_freeze_ratio(t, phases, expected);
    default: return 0.0;
  }
}

MaskHistory run_freezing_masks(const std::map<ActionId, double>& expected, const PhasePlan& phases, int M, int S,
                               int n, Rng& rng) {
  MaskHistory h;
  for (int t = 1; t <= phases.t_total; ++t)
    for (int s = 1; s <= S; ++s)
      for (int m = 1; m <= M; ++m) {
        const ActionId node = backward_action(m, s);
        const auto it = expected.find(node);
        const double r = phase_of(t, phases) == Phase::MonitorLower
                             ? 1.0
                             : (it == expected.end() ? 0.0 : cell_ratio(t, phases, it->second));
        h.add(t, node, sample_mask(n, r, rng));
      }
  return h;
}

// ------------------------------------------------------------------ MaskStream

MaskStream::MaskStream(std::vector<double> ratios, PhasePlan phases, int M, int S, int units, std::uint64_t seed)
    : MaskStream(std::move(ratios), phases, M, std::vector<int>(static_cast<std::size_t>(std::max(S, 0)), units), seed) {}

MaskStream::MaskStream(std::vector<double> ratios, PhasePlan phases, int M, std::vector<int> stage_units,
                       std::uint64_t seed)
    : ratios_(std::move(ratios)), phases_(phases), M_(M), S_(static_cast<int>(stage_units.size())),
      units_(std::move(stage_units)), seed_(seed) {
  if (static_cast<int>(ratios_.size()) != M_ * S_) throw std::domain_error("mask stream: ratios must have M*S entries");
  for (int u : units_)
    if (u < 0) throw std::domain_error("mask stream: units must be nonnegative");
  validate_phase_plan(phases_);
  step_prefix_.push_back(0);
}

double MaskStream::ratio(int t, int s, int m) const {
  return cell_ratio(t, phases_, ratios_[static_cast<std::size_t>((s - 1) * M_ + (m - 1))]);
}

int MaskStream::cell_count(int t, int s, int m) const { return mask_count(units(s), ratio(t, s, m)); }

void MaskStream::ensure_prefix(int t) const {
  while (static_cast<int>(step_prefix_.size()) < t) {
    const int tt = static_cast<int>(step_prefix_.size());  // step whose draws we add
    std::uint64_t d = 0;
    for (int s = 1; s <= S_; ++s)
      for (int m = 1; m <= M_; ++m) d += static_cast<std::uint64_t>(cell_count(tt, s, m));
    step_prefix_.push_back(step_prefix_.back() + d);
  }
}

std::uint64_t MaskStream::offset(int t, int s, int m) const {
  if (t < 1 || t > phases_.t_total || s < 1 || s > S_ || m < 1 || m > M_)
    throw std::domain_error("mask stream: cell out of range");
  ensure_prefix(t);
  std::uint64_t off = step_prefix_[static_cast<std::size_t>(t - 1)];
  for (int s2 = 1; s2 <= S_; ++s2)
    for (int m2 = 1; m2 <= M_; ++m2) {
      if (s2 == s && m2 == m) return off;
      off += static_cast<std::uint64_t>(cell_count(t, s2, m2));
    }
  return off;
}

bool MaskStream::stage_step_masks(int t, int s, std::uint64_t* out, int threads) const {
  const int words = words_per_mask(s);
  const int n = units(s);
  std::vector<std::uint64_t> base(static_cast<std::size_t>(M_));
  std::vector<int> counts(static_cast<std::size_t>(M_));
  for (int m = 1; m <= M_; ++m) {
    base[static_cast<std::size_t>(m - 1)] = offset(t, s, m);
    counts[static_cast<std::size_t>(m - 1)] = cell_count(t, s, m);
  }
  std::vector<std::uint64_t> used(static_cast<std::size_t>(M_), 0);
  auto run_cell = [&](int mi, std::uint64_t draw_offset) {
    const int k = counts[static_cast<std::size_t>(mi)];
    std::uint64_t* w = out + static_cast<std::size_t>(mi) * static_cast<std::size_t>(words);
    if (k == 0) {
      std::fill(w, w + words, 0);
      used[static_cast<std::size_t>(mi)] = 0;
      return;
    }
    Rng rng = Rng::at_offset(seed_, draw_offset);
    auto& pool = scratch_pool(n);
    used[static_cast<std::size_t>(mi)] = partial_shuffle(pool.data(), n, k, rng);
    fill_words(pool.data(), k, w, words);
  };
  const int nthreads = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int mi = 0; mi < M_; ++mi) run_cell(mi, base[static_cast<std::size_t>(mi)]);
  // A rejection event inside a cell shifts every later cell: replay them in order.
  bool exact_parallel = true;
  std::uint64_t shift = 0;
  for (int mi = 0; mi < M_; ++mi) {
    if (shift != 0) run_cell(mi, base[static_cast<std::size_t>(mi)] + shift);
    const std::uint64_t extra = used[static_cast<std::size_t>(mi)] - static_cast<std::uint64_t>(counts[static_cast<std::size_t>(mi)]);
    if (extra != 0) {
      exact_parallel = false;
      shift += extra;
    }
  }
  return exact_parallel;
}

}  // namespace pipefreeze
