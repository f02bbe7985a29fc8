// Freeze controller: phases, ramped freeze ratio, exact-count unit masks,
// hybrid reconciliation (Alg. 2), AutoFreeze and APF scores, monitoring and
// the full-horizon mask driver.
// API mirrors proj/include/pipefreeze/freezectl.hpp; ApfState uses
// std::vector<double> where the reference uses Eigen::VectorXd (same
// element-wise arithmetic). Additions for the multi-GPU build: MaskStream
// regenerates any (step, stage, microbatch) cell of the single reference
// stream by counter jump-ahead, in parallel, bit-exactly.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "timing.hpp"
#include "types.hpp"

namespace pipefreeze {

struct PhasePlan {
  int t_warmup{0};
  int t_monitor{0};
  int t_freeze{0};
  int t_total{0};

  int t_mid() const { return t_warmup + (t_monitor - t_warmup + 1) / 2; }
};

void validate_phase_plan(const PhasePlan& plan);

enum class Phase { Warmup, MonitorUpper, MonitorLower, Solve, ProgressiveFreeze, StableFreeze };

std::string to_string(Phase phase);
Phase phase_of(int t, const PhasePlan& plan);
double actual_freeze_ratio(int t, const PhasePlan& plan, double expected_ratio);
double afr_at(int t, const PhasePlan& plan, double expected_ratio);

class FreezeMask {
 public:
  FreezeMask() = default;
  explicit FreezeMask(int n_params) : n_(n_params), words_(static_cast<std::size_t>((n_params + 63) / 64), 0) {}

  int size() const { return n_; }
  bool test(int i) const { return (words_[static_cast<std::size_t>(i >> 6)] >> (i & 63)) & 1u; }
  void set(int i) { words_[static_cast<std::size_t>(i >> 6)] |= std::uint64_t{1} << (i & 63); }
  void reset(int i) { words_[static_cast<std::size_t>(i >> 6)] &= ~(std::uint64_t{1} << (i & 63)); }
  int popcount() const;
  std::vector<int> set_indices() const;
  std::vector<int> unset_indices() const;
  const std::vector<std::uint64_t>& words() const { return words_; }
  std::vector<std::uint64_t>& words() { return words_; }

  friend bool operator==(const FreezeMask&, const FreezeMask&) = default;

 private:
  int n_{0};
  std::vector<std::uint64_t> words_;
};

// floor(ratio * n) frozen indices, uniform over subsets of that size.
FreezeMask sample_mask(int n_params, double ratio, Rng& rng);
// Number of frozen units sample_mask draws (= RNG draws consumed, barring rejection).
int mask_count(int n_params, double ratio);

FreezeMask reconcile_mask(const FreezeMask& base, int target_count, Rng& rng);

double autofreeze_score(double norm_prev, double norm_cur);
int autofreeze_select(const std::vector<double>& scores, int frozen_prefix_len, double percentile);

// Dense fp64 vector of the APF state: a std::vector<double> that also takes the element-access
// spelling of the reference's Eigen::VectorXd (v(i), Constant, Zero), so the reference's call
// sites and its own unit suite (tests/test_freezectl.cpp, built by oracle/Makefile product-check)
// compile unchanged against this header; Eigen is not installed here.
struct Vector : std::vector<double> {
  using std::vector<double>::vector;
  Vector() = default;
  Vector(const std::vector<double>& v) : std::vector<double>(v) {}  // NOLINT: implicit, like the reference
  double& operator()(std::size_t i) { return (*this)[i]; }
  double operator()(std::size_t i) const { return (*this)[i]; }
  static Vector Constant(std::size_t n, double v) { return Vector(n, v); }
  static Vector Zero(std::size_t n) { return Vector(n, 0.0); }
  // comma initialiser: v << a, b, c;
  struct CommaInit {
    Vector& v;
    std::size_t i;
    CommaInit& operator,(double x) {
      v.at(i++) = x;
      return *this;
    }
  };
  CommaInit operator<<(double x) {
    at(0) = x;
    return CommaInit{*this, 1};
  }
};

struct ApfState {
  Vector ema;      // E
  Vector ema_abs;  // E_abs
  double alpha{0.9};

  static ApfState zeros(std::size_t n, double alpha = 0.9);
};

Vector apf_update(ApfState& state, const std::vector<double>& delta);
std::vector<int> apf_eligible(const std::vector<double>& scores, double threshold);

struct MaskRecord {
  int step{0};
  int stage{0};
  ActionId action;
  int popcount{0};
  int n_params{0};
};

class MaskHistory {
 public:
  void add(int step, const ActionId& action, const FreezeMask& mask);
  void add_record(const MaskRecord& record) { records_.push_back(record); }
  const std::vector<MaskRecord>& records() const { return records_; }
  const std::vector<std::vector<long>>& stage_counts() const { return stage_counts_; }
  const std::vector<long>& stage_draws() const { return stage_draws_; }

 private:
  std::vector<MaskRecord> records_;
  std::vector<std::vector<long>> stage_counts_;
  std::vector<long> stage_draws_;
};

MonitorLog run_monitoring(const TimingProfile& truth, int num_microbatches, int total_stages,
                          const PhasePlan& phases, const NoiseSpec& noise, Rng& rng);

MaskHistory run_freezing_masks(const std::map<ActionId, double>& expected_ratios, const PhasePlan& phases,
                               int num_microbatches, int total_stages, int params_per_stage, Rng& rng);

// Controller ratio of cell (t, b(m,s)): 1 in MonitorLower, the ramped plan
// ratio in Progressive/Stable, else 0 (proj/src/freezectl.cpp:192-206).
double cell_ratio(int t, const PhasePlan& phases, double expected_ratio);

// Random access into the run_freezing_masks stream (one Rng seeded `seed`,
// cells in t -> s -> m order). Any subset of cells can be generated in
// parallel; results equal the sequential stream bit for bit. Rejection
// sampling inside index_below can in principle consume extra draws (p <= n/2^64
// per draw); generate() detects it and falls back to sequential replay.
class MaskStream {
 public:
  MaskStream(std::vector<double> expected_ratios /* (s-1)*M + (m-1) */, PhasePlan phases,
             int num_microbatches, int total_stages, int units, std::uint64_t seed);
  // Generalisation for stages of different sizes (unit count per stage); with
  // equal counts it is the reference stream.
  MaskStream(std::vector<double> expected_ratios, PhasePlan phases, int num_microbatches,
             std::vector<int> stage_units, std::uint64_t seed);

  // RNG draws consumed by all cells strictly before (t, s, m).
  std::uint64_t offset(int t, int s, int m) const;
  int cell_count(int t, int s, int m) const;  // frozen units in that cell
  double ratio(int t, int s, int m) const;

  // Masks for cells {(t, s, m) : m = 1..M} of one stage, as 64-bit words
  // ([M][words]); threads <= 0 uses all cores. Returns false if a rejection
  // event forced a sequential replay (result is still exact).
  bool stage_step_masks(int t, int s, std::uint64_t* words_out, int threads = 0) const;

  int units(int s = 1) const { return units_[static_cast<std::size_t>(s - 1)]; }
  int words_per_mask(int s = 1) const { return (units(s) + 63) / 64; }

 private:
  void ensure_prefix(int t) const;
  std::vector<double> ratios_;
  PhasePlan phases_;
  int M_, S_;
  std::vector<int> units_;
  std::uint64_t seed_;
  mutable std::vector<std::uint64_t> step_prefix_;  // draws before step t (index t-1)
};

}  // namespace pipefreeze
