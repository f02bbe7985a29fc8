// Per-rank training-step driver: the paper's Alg. 1 with
// the reference's controller semantics. The host side is the C++ pipefreeze
// layer (schedule, DAG, monitoring aggregation, LP, masks); the device side is
// the Stage engine. One instance per GPU/process.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <vector>

#include <cuda_bf16.h>

#include "dag.hpp"
#include "freezectl.hpp"
#include "lp.hpp"
#include "schedule.hpp"
#include "stage.hpp"
#include "timing.hpp"

namespace pf {

struct TrainConfig {
  pipefreeze::PipelineConfig pipeline;
  int rank = 0;
  pipefreeze::PhasePlan phases{2, 8, 10, 20};
  double r_max = 0.8;
  double lr = 1e-3;
  uint64_t seed = 42;
  bool apf = false;
  float apf_alpha = 0.9f;
  float apf_threshold = 1e-4f;
  int apf_every = 1;
  int device = 0;
  int mask_threads = 0;
  // Hybrid TimelyFreeze + APF (paper Alg. 2): in the freezing phases each cell's
  // mask is reconcile_mask(APF base set, floor(AFR * units)); a unit joins the
  // base set when at least this fraction of its elements is APF-eligible.
  bool hybrid = false;
  float hybrid_unit_fraction = 0.5f;
  // optimizer: SGD (reference, sandbox.cpp:250) or AdamW (the paper's optimizer; lr as above)
  OptimCfg optim{};
};

struct StepResult {
  double loss = 0.0;           // mean over microbatches (last stage on this rank; NaN otherwise)
  double batch_ms = 0.0;       // device time from start of the first action to end of the last
  double optimizer_ms = 0.0;
  double predicted_ms = 0.0;   // LP/DAG makespan for this step's ratios (longest path)
  int phase = 0;
  double mean_ratio = 0.0;     // mean realised frozen-unit fraction over this rank's cells
  long long frozen_units = 0;  // sum over cells
  long long total_units = 0;   // units * cells
  double mask_ms = 0.0;        // host time to generate this step's masks
};

class Trainer {
 public:
  Trainer(const ModelConfig& model, const TrainConfig& cfg);
  const TrainConfig& config() const { return cfg_; }
  ~Trainer();

  // host_tokens / host_targets: [M][T] int32 (pinned or pageable) or null to
  // use device-resident synthetic tokens. host_masks: caller-owned frozen-unit
  // masks for every local cell (per local stage, M masks of ceil(units/64) words,
  // FreezeMask::test bit order) instead of the controller's; null = controller.
  int step(int t, const int* host_tokens, const int* host_targets, StepResult* out,
           const uint64_t* host_masks = nullptr);
  // device gradient stamp of the last step (internal counter, 1 for the first step)
  int stamp() const { return stamp_; }

  void set_override(double ratio) {
    override_ratio_ = ratio;
    next_t_ = -1;
  }
  // words of local stage li's masks (ceil(units / 64))
  int mask_words(int li) const;
  void set_plan(const std::vector<double>& ratios);
  bool has_plan() const { return plan_ready_; }
  const std::vector<double>& plan_ratios() const { return plan_ratios_; }
  const pipefreeze::FreezePlan& plan() const { return plan_; }
  const std::vector<double>& action_ms() const { return action_ms_; }
  // start of each action of the last step relative to the step's origin event, recorded when
  // step() began enqueueing (CUDA events)
  const std::vector<double>& action_start_ms() const { return action_start_ms_; }
  const std::vector<pipefreeze::ActionId>& actions() const { return actions_; }
  std::vector<Stage*> local_stages();
  long long tokens_per_step() const;
  double lp_solve_ms() const { return lp_solve_ms_; }
  pipefreeze::TimingProfile measured_profile() const;
  int units_total() const;
  cudaStream_t stream() const { return stream_; }
  bool apf_base_ready() const { return apf_base_ready_; }
  // APF base set of local stage li (hybrid mode) as a unit mask
  pipefreeze::FreezeMask apf_base_mask(int li) const;
  // this step's frozen-unit masks of local stage li: M masks of (words + 1) uint64 each
  const uint64_t* masks_host(int li) const { return masks_host_ + mask_offsets_[static_cast<std::size_t>(li)]; }

  // Multi-rank P2P (NCCL over NVLink). One two-rank communicator and stream per link:
  // a (kind, src rank, dst rank) class of DAG rule-3 edges that crosses ranks
  // (activations s -> s+1, gradients s+1 -> s), so every communicator carries one
  // direction of one edge class and no transfer queues behind another link's. This
  // covers every placement: chains (gpipe / 1f1b), the interleaved ring (rank R-1 ->
  // rank 0) and the ZBV V (activations flow both ways). Plus one world communicator
  // for the monitoring all-reduce at T_m. ids: comm_ids_needed() x 128 bytes, the
  // world id first, then one per link in links() order (same on every rank).
  int init_comm(const void* ids, int nranks, int rank);
  bool distributed() const { return world_comm_ != nullptr; }
  struct Link {
    int kind;      // 0 activations (forward edge), 1 gradients (backward edge)
    int src, dst;  // ranks
    void* comm = nullptr;  // ncclComm_t with src = comm rank 0, dst = comm rank 1
    cudaStream_t stream = nullptr;
  };
  const std::vector<Link>& links() const { return links_; }
  int comm_ids_needed() const { return 1 + static_cast<int>(links_.size()); }

 private:
  int local_index(int stage) const;
  // the host copy of this step's mask of cell (local stage, microbatch) has no frozen unit
  bool cell_dense(int local_stage, int microbatch) const;
  const pipefreeze::MaskStream& mask_stream();
  void solve_plan_from_monitoring();
  void build_masks(int t, pipefreeze::Phase phase, bool controller, uint64_t* out, long long* frozen,
                   long long* total);
  int exchange_monitoring(pipefreeze::TimingProfile* merged);

  Link* link(int kind, int src, int dst);
  std::vector<Link> links_;
  void* world_comm_ = nullptr;  // ncclComm_t over all ranks (monitoring all-reduce)
  cudaStream_t ctl_stream_ = nullptr;
  std::vector<std::vector<__nv_bfloat16*>> x_recv_;   // [local stage][slot] activations from rank_of(s-1)
  std::vector<std::vector<__nv_bfloat16*>> dy_recv_;  // [local stage][slot] gradients from rank_of(s+1)
  std::vector<std::vector<__nv_bfloat16*>> dx_send_;  // [local stage][slot] gradient of the stage input
  // per [local stage][slot]: buffer-reuse guards between compute and comm streams
  std::vector<std::vector<cudaEvent_t>> x_free_ev_, out_sent_ev_, dy_free_ev_, dx_sent_ev_;
  std::vector<cudaEvent_t> comm_ev_;  // data-ready events, pool reused every step

  ModelConfig model_;
  TrainConfig cfg_;
  pipefreeze::RankTimeline timeline_;
  std::unique_ptr<pipefreeze::PipelineDag> dag_;
  std::vector<pipefreeze::IssueOp> program_;   // this rank's issue program (host layer)
  std::vector<pipefreeze::ActionId> actions_;  // program_'s actions
  std::vector<int> stage_ids_;                  // local stages (1-based)
  std::vector<std::unique_ptr<Stage>> stages_;  // parallel to stage_ids_
  std::vector<int> slots_;                      // per local stage
  std::vector<std::vector<__nv_bfloat16*>> grad_bufs_;  // [local stage][slot]: dL/d(stage output)
  cudaStream_t stream_ = nullptr;
  std::vector<cudaEvent_t> ev_;
  cudaEvent_t ev_opt0_ = nullptr, ev_opt1_ = nullptr, ev_origin_ = nullptr;
  int* tokens_dev_ = nullptr;
  int* targets_dev_ = nullptr;
  float* loss_dev_ = nullptr;
  uint64_t* masks_dev_ = nullptr;
  uint64_t* masks_host_ = nullptr;  // pinned
  uint64_t* masks_next_ = nullptr;  // pinned: step next_t_'s masks, built while the previous step ran
  int next_t_ = -1;
  double next_override_ = 0.0;
  bool next_plan_ready_ = false;
  long long next_frozen_ = 0, next_total_ = 0;
  std::vector<long long> mask_offsets_;  // words offset per local stage
  float* loss_host_ = nullptr;           // pinned
  pipefreeze::MonitorLog monitor_;
  bool plan_ready_ = false;
  std::vector<double> plan_ratios_;  // (s-1)*M + (m-1)
  pipefreeze::FreezePlan plan_;
  pipefreeze::TimingProfile plan_profile_;
  double override_ratio_ = -1.0;
  std::vector<double> action_ms_;
  std::vector<double> action_start_ms_;
  std::vector<std::vector<int>> apf_eligible_host_;  // [local stage][unit], last APF step
  bool apf_base_ready_ = false;
  int* apf_pinned_ = nullptr;
  double lp_solve_ms_ = 0.0;
  // Gradient stamps (Stage::unit_stamp): an internal counter that starts at 1 and rises by
  // one every step, independent of the caller's t, so a unit's first dW of a step always
  // overwrites G (which is never memset) and a repeated t cannot accumulate old gradients.
  int stamp_ = 0;
  // The reference mask stream of the current plan. Kept across steps so its step-prefix cache
  // grows incrementally (O(1) amortised per step, not O(t)); rebuilt when the plan changes.
  std::unique_ptr<pipefreeze::MaskStream> mask_stream_;
};

}  // namespace pf
