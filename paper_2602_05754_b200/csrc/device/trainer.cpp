#include "trainer.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include <nccl.h>

namespace pf {

using namespace pipefreeze;

namespace {

#define PF_TRY(expr)              \
  do {                            \
    const int _rc = (expr);       \
    if (_rc != PF_OK) return _rc; \
  } while (0)
#define PF_CUDA(expr)                              \
  do {                                             \
    if ((expr) != cudaSuccess) return PF_ERR_CUDA; \
  } while (0)

// Layers [begin, end) of virtual stage s (1-based) out of S: the first L % S
// stages take one extra layer (e.g. 40 layers / 16 stages = 8 x 3 + 8 x 2).
StageSpec stage_spec(const ModelConfig& m, int s, int S) {
  const int base = m.layers / S, extra = m.layers % S;
  StageSpec sp;
  sp.stage = s;
  sp.layer_begin = (s - 1) * base + std::min(s - 1, extra);
  sp.layer_end = sp.layer_begin + base + (s - 1 < extra ? 1 : 0);
  sp.first = s == 1;
  sp.last = s == S;
  return sp;
}

int units_of(int rows, int cols) { return ((rows + 127) / 128) * ((cols + 127) / 128); }

// Unit count of a stage without allocating it (same matrix lists as LlamaStage / VitStage).
int stage_units(const ModelConfig& m, const StageSpec& sp) {
  const int mlp_in = m.family == 1 ? m.ffn : 2 * m.ffn;  // ViT fc1 vs LLaMA gate|up
  const int per_layer = units_of(m.qkv_dim(), m.hidden) + units_of(m.hidden, m.attn_dim()) +
                        units_of(mlp_in, m.hidden) + units_of(m.hidden, m.ffn);
  int u = (sp.layer_end - sp.layer_begin) * per_layer + (sp.last ? units_of(m.vocab, m.hidden) : 0);
  if (m.family == 1 && sp.first) u += units_of(m.hidden, m.patch_dim());  // patch embedding
  return u;
}

}  // namespace

Trainer::Trainer(const ModelConfig& model, const TrainConfig& cfg) : model_(model), cfg_(cfg) {
  cudaSetDevice(cfg.device);
  timeline_ = build_schedule(cfg.pipeline);
  dag_ = std::make_unique<PipelineDag>(build_dag(timeline_));
  validate_phase_plan(cfg.phases);
  const int S = cfg.pipeline.total_stages();
  const int M = cfg.pipeline.num_microbatches;
  if (cfg.rank < 0 || cfg.rank >= cfg.pipeline.num_ranks) throw std::invalid_argument("trainer: rank out of range");
  if (model.layers < S) throw std::invalid_argument("trainer: fewer layers than pipeline stages");
  // the rank's issue program (libpf_host): actions in schedule order + their cross-rank P2P
  program_ = issue_program(cfg.pipeline, cfg.rank);
  for (const auto& op : program_) actions_.push_back(op.action);
  for (int s = 1; s <= S; ++s)
    if (stage_to_rank(cfg.pipeline, s) == cfg.rank) stage_ids_.push_back(s);
  // cross-rank edge classes of DAG rule 3 (dag.cpp:90-93): one P2P link each
  for (int s = 1; s < S; ++s) {
    const int a = stage_to_rank(cfg.pipeline, s), b = stage_to_rank(cfg.pipeline, s + 1);
    if (a == b) continue;
    for (const Link& l : {Link{0, a, b}, Link{1, b, a}}) {
      bool seen = false;
      for (const Link& x : links_) seen |= x.kind == l.kind && x.src == l.src && x.dst == l.dst;
      if (!seen) links_.push_back(l);
    }
  }
  // in-flight microbatches per stage = slot count; a slot is held from F until the
  // action that last reads it: b, or w when the backward is split
  const bool split = splits_weight_grad(cfg.pipeline);
  const ActionKind release = split ? ActionKind::Weight : ActionKind::Backward;
  for (int s : stage_ids_) {
    int live = 0, peak = 0;
    for (const auto& a : actions_) {
      if (a.stage != s) continue;
      live += a.kind == ActionKind::Forward ? 1 : (a.kind == release ? -1 : 0);
      peak = std::max(peak, live);
    }
    slots_.push_back(std::max(1, peak));
  }
  for (std::size_t i = 0; i < stage_ids_.size(); ++i)
    stages_.push_back(make_stage(model, stage_spec(model, stage_ids_[i], S), slots_[i], cfg.seed, cfg.device, split));
  const long long T = model.tokens();
  auto act_alloc = [&]() {
    __nv_bfloat16* p = nullptr;
    if (cudaMalloc(&p, static_cast<size_t>(T) * model.hidden * 2) != cudaSuccess)
      throw std::runtime_error("trainer: cudaMalloc failed");
    return p;
  };
  x_recv_.resize(stage_ids_.size());
  dy_recv_.resize(stage_ids_.size());
  dx_send_.resize(stage_ids_.size());
  for (std::size_t i = 0; i < stage_ids_.size(); ++i) {
    const int s = stage_ids_[i];
    for (int k = 0; k < slots_[i]; ++k) {
      if (s > 1 && local_index(s - 1) < 0) {
        x_recv_[i].push_back(act_alloc());
        dx_send_[i].push_back(act_alloc());
      }
      if (s < S && local_index(s + 1) < 0) dy_recv_[i].push_back(act_alloc());
    }
  }
  grad_bufs_.resize(stage_ids_.size());
  for (std::size_t i = 0; i < stage_ids_.size(); ++i)
    for (int k = 0; k < slots_[i]; ++k) {
      __nv_bfloat16* p = nullptr;
      if (cudaMalloc(&p, static_cast<size_t>(T) * model.hidden * 2) != cudaSuccess)
        throw std::runtime_error("trainer: cudaMalloc failed");
      grad_bufs_[i].push_back(p);
    }
  if (cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking) != cudaSuccess)
    throw std::runtime_error("trainer: stream creation failed");
  ev_.resize(2 * actions_.size());
  for (auto& e : ev_) cudaEventCreate(&e);
  cudaEventCreate(&ev_opt0_);
  cudaEventCreate(&ev_origin_);
  cudaEventCreate(&ev_opt1_);
  cudaMalloc(&tokens_dev_, static_cast<size_t>(M) * T * 4);
  cudaMalloc(&targets_dev_, static_cast<size_t>(M) * T * 4);
  cudaMalloc(&loss_dev_, 4);
  launch_random_tokens(tokens_dev_, static_cast<long long>(M) * T, model.vocab, cfg.seed * 31 + 1, stream_);
  launch_random_tokens(targets_dev_, static_cast<long long>(M) * T, model.vocab, cfg.seed * 31 + 2, stream_);
  long long words = 0;
  for (auto& st : stages_) {
    mask_offsets_.push_back(words);
    words += static_cast<long long>(M) * (st->words() + 1);  // +1 pad word per mask (K5 reads one past)
  }
  mask_offsets_.push_back(words);
  cudaMalloc(&masks_dev_, static_cast<size_t>(std::max<long long>(words, 1)) * 8);
  cudaMallocHost(&masks_host_, static_cast<size_t>(std::max<long long>(words, 1)) * 8);
  std::memset(masks_host_, 0, static_cast<size_t>(std::max<long long>(words, 1)) * 8);
  cudaMallocHost(&masks_next_, static_cast<size_t>(std::max<long long>(words, 1)) * 8);
  std::memset(masks_next_, 0, static_cast<size_t>(std::max<long long>(words, 1)) * 8);
  cudaMallocHost(&loss_host_, 4);
  plan_ratios_.assign(static_cast<std::size_t>(S * M), 0.0);
  if (cudaStreamSynchronize(stream_) != cudaSuccess) throw std::runtime_error("trainer: setup failed");
}

Trainer::~Trainer() {
  cudaSetDevice(cfg_.device);
  if (stream_) cudaStreamSynchronize(stream_);
  stages_.clear();
  for (auto& v : grad_bufs_)
    for (auto* p : v) cudaFree(p);
  for (auto* vv : {&x_recv_, &dy_recv_, &dx_send_})
    for (auto& v : *vv)
      for (auto* p : v) cudaFree(p);
  for (auto& e : comm_ev_) cudaEventDestroy(e);
  for (auto* vv : {&x_free_ev_, &out_sent_ev_, &dy_free_ev_, &dx_sent_ev_})
    for (auto& v : *vv)
      for (auto e : v) cudaEventDestroy(e);
  for (auto& l : links_) {
    if (l.comm) ncclCommDestroy(static_cast<ncclComm_t>(l.comm));
    if (l.stream) cudaStreamDestroy(l.stream);
  }
  if (world_comm_) ncclCommDestroy(static_cast<ncclComm_t>(world_comm_));
  if (ctl_stream_) cudaStreamDestroy(ctl_stream_);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (ev_opt0_) cudaEventDestroy(ev_opt0_);
  if (ev_origin_) cudaEventDestroy(ev_origin_);
  if (ev_opt1_) cudaEventDestroy(ev_opt1_);
  cudaFree(tokens_dev_);
  cudaFree(targets_dev_);
  cudaFree(loss_dev_);
  cudaFree(masks_dev_);
  cudaFreeHost(masks_host_);
  cudaFreeHost(masks_next_);
  cudaFreeHost(loss_host_);
  if (apf_pinned_) cudaFreeHost(apf_pinned_);
  if (stream_) cudaStreamDestroy(stream_);
}

int Trainer::local_index(int stage) const {
  for (std::size_t i = 0; i < stage_ids_.size(); ++i)
    if (stage_ids_[i] == stage) return static_cast<int>(i);
  return -1;
}

std::vector<Stage*> Trainer::local_stages() {
  std::vector<Stage*> out;
  for (auto& s : stages_) out.push_back(s.get());
  return out;
}

long long Trainer::tokens_per_step() const {
  return static_cast<long long>(model_.tokens()) * cfg_.pipeline.num_microbatches;
}

int Trainer::units_total() const {
  int u = 0;
  for (const auto& s : stages_) u += s->units();
  return u;
}

void Trainer::set_plan(const std::vector<double>& ratios) {
  const int S = cfg_.pipeline.total_stages(), M = cfg_.pipeline.num_microbatches;
  if (static_cast<int>(ratios.size()) != S * M) throw std::invalid_argument("set_plan: need M*S ratios");
  plan_ratios_ = ratios;
  plan_ready_ = true;
  mask_stream_.reset();
  next_t_ = -1;  // prefetched masks used the old plan
}

int Trainer::mask_words(int li) const { return stages_[static_cast<std::size_t>(li)]->words(); }

const MaskStream& Trainer::mask_stream() {
  if (!mask_stream_) {
    const int S = cfg_.pipeline.total_stages(), M = cfg_.pipeline.num_microbatches;
    std::vector<int> units_all;
    for (int s = 1; s <= S; ++s) units_all.push_back(stage_units(model_, stage_spec(model_, s, S)));
    mask_stream_ = std::make_unique<MaskStream>(plan_ratios_, cfg_.phases, M, units_all, cfg_.seed);
  }
  return *mask_stream_;
}

namespace {
// splitmix64 finaliser over non-overlapping (t, s, m) fields: per-cell seeds of the
// override / hybrid masks without int overflow or collisions across stages
uint64_t cell_seed(uint64_t seed, uint64_t salt, int t, int s, int m) {
  uint64_t z = seed ^ salt;
  z += (static_cast<uint64_t>(static_cast<uint32_t>(t)) << 32) ^ (static_cast<uint64_t>(s & 0xFFFF) << 16) ^
       static_cast<uint64_t>(m & 0xFFFF);
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // namespace

bool Trainer::cell_dense(int local_stage, int microbatch) const {
  const int words = stages_[static_cast<std::size_t>(local_stage)]->words();
  const uint64_t* w = masks_host_ + mask_offsets_[static_cast<std::size_t>(local_stage)] +
                      static_cast<long long>(microbatch - 1) * (words + 1);
  for (int i = 0; i < words; ++i)
    if (w[i]) return false;
  return true;
}

FreezeMask Trainer::apf_base_mask(int li) const {
  const Stage& st = *stages_[static_cast<std::size_t>(li)];
  FreezeMask base(st.units());
  if (static_cast<std::size_t>(li) >= apf_eligible_host_.size()) return base;
  const auto& elig = apf_eligible_host_[static_cast<std::size_t>(li)];
  for (const auto& m : st.unit_matrices())
    for (int lu = 0; lu < m.units; ++lu) {
      const int rb = lu / m.tiles_n, cb = lu % m.tiles_n;
      const int elems = std::min(128, m.rows - rb * 128) * std::min(128, m.cols - cb * 128);
      const int u = m.unit_offset + lu;
      if (elig[static_cast<std::size_t>(u)] >= cfg_.hybrid_unit_fraction * static_cast<float>(elems)) base.set(u);
    }
  return base;
}

TimingProfile Trainer::measured_profile() const { return plan_profile_.all().empty() ? aggregate_monitoring(monitor_) : plan_profile_; }

Trainer::Link* Trainer::link(int kind, int src, int dst) {
  for (auto& l : links_)
    if (l.kind == kind && l.src == src && l.dst == dst) return &l;
  return nullptr;
}

int Trainer::init_comm(const void* ids, int nranks, int rank) {
  if (nranks != cfg_.pipeline.num_ranks || rank != cfg_.rank || !ids || distributed()) return PF_ERR_INVALID;
  cudaSetDevice(cfg_.device);
  const int n = comm_ids_needed();
  std::vector<ncclUniqueId> u(static_cast<std::size_t>(n));
  std::memcpy(u.data(), ids, static_cast<size_t>(n) * sizeof(ncclUniqueId));
  ncclComm_t w;
  if (ncclCommInitRank(&w, nranks, u[0], rank) != ncclSuccess) return PF_ERR_NCCL;
  world_comm_ = w;
  // every link this rank is an end of, initialised together (no ordering constraints)
  if (ncclGroupStart() != ncclSuccess) return PF_ERR_NCCL;
  for (std::size_t k = 0; k < links_.size(); ++k) {
    Link& l = links_[k];
    if (rank != l.src && rank != l.dst) continue;
    ncclComm_t c;
    if (ncclCommInitRank(&c, 2, u[k + 1], rank == l.src ? 0 : 1) != ncclSuccess) return PF_ERR_NCCL;
    l.comm = c;
  }
  if (ncclGroupEnd() != ncclSuccess) return PF_ERR_NCCL;
  for (auto& l : links_)
    if (l.comm && cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking) != cudaSuccess) return PF_ERR_CUDA;
  if (cudaStreamCreateWithFlags(&ctl_stream_, cudaStreamNonBlocking) != cudaSuccess) return PF_ERR_CUDA;
  for (auto* vv : {&x_free_ev_, &out_sent_ev_, &dy_free_ev_, &dx_sent_ev_}) {
    vv->resize(stage_ids_.size());
    for (std::size_t i = 0; i < stage_ids_.size(); ++i) {
      (*vv)[i].resize(static_cast<std::size_t>(slots_[i]));
      for (auto& e : (*vv)[i])
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return PF_ERR_CUDA;
    }
  }
  return PF_OK;
}

// Alg. 1 at T_m gathers every rank's monitored durations: each
// rank aggregates its own actions, one all-reduce (sum; each node owned by one
// rank) gives every rank the same bounds, so every rank solves the same LP.
int Trainer::exchange_monitoring(TimingProfile* merged) {
  const auto local = aggregate_monitoring(monitor_);
  const std::size_t n = static_cast<std::size_t>(dag_->node_count() - 2);
  std::vector<double> host(2 * n, 0.0);
  for (const auto& [a, b] : local.all()) {
    const int v = dag_->index_of(a) - 1;
    host[static_cast<std::size_t>(v)] = b.w_min;
    host[n + static_cast<std::size_t>(v)] = b.w_max;
  }
  if (distributed()) {
    double* dev = nullptr;
    if (cudaMalloc(&dev, host.size() * sizeof(double)) != cudaSuccess) return PF_ERR_CUDA;
    cudaMemcpyAsync(dev, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, ctl_stream_);
    if (ncclAllReduce(dev, dev, host.size(), ncclFloat64, ncclSum, static_cast<ncclComm_t>(world_comm_),
                      ctl_stream_) != ncclSuccess)
      return PF_ERR_NCCL;
    cudaMemcpyAsync(host.data(), dev, host.size() * sizeof(double), cudaMemcpyDeviceToHost, ctl_stream_);
    cudaStreamSynchronize(ctl_stream_);
    cudaFree(dev);
  }
  TimingProfile p;
  for (int v = 1; v + 1 < dag_->node_count(); ++v)
    p.set_bounds(dag_->action_at(v), {host[static_cast<std::size_t>(v - 1)], host[n + static_cast<std::size_t>(v - 1)]});
  *merged = p;
  return PF_OK;
}

// Alg. 1 line at t = T_m: aggregate the monitored durations into bounds, solve
// the freeze-ratio LP, keep the plan (reference cmd_optimize, pipefreeze.cpp:61-83).
void Trainer::solve_plan_from_monitoring() {
  const auto t0 = std::chrono::steady_clock::now();
  if (exchange_monitoring(&plan_profile_) != PF_OK) throw numerical_error("monitoring exchange failed");
  const auto lp = build_lp(*dag_, plan_profile_, cfg_.r_max);
  const auto sol = solve_lp(lp);
  plan_ = extract_freeze_plan(*dag_, plan_profile_, sol, cfg_.r_max);
  const int S = cfg_.pipeline.total_stages(), M = cfg_.pipeline.num_microbatches;
  for (int s = 1; s <= S; ++s)
    for (int m = 1; m <= M; ++m)
      plan_ratios_[static_cast<std::size_t>((s - 1) * M + (m - 1))] = plan_.ratio_of(freeze_node(cfg_.pipeline, m, s));
  plan_ready_ = true;
  mask_stream_.reset();
  lp_solve_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Masks of step t for every local cell into `out` (masks_host_ layout: per stage, M masks of
// words + 1 pad word), with the frozen / total unit counts.
void Trainer::build_masks(int t, Phase phase, bool controller, uint64_t* out, long long* frozen, long long* total) {
  const int S = cfg_.pipeline.total_stages(), M = cfg_.pipeline.num_microbatches;
  *frozen = 0;
  *total = 0;
  (void)S;
  for (std::size_t li = 0; li < stages_.size(); ++li) {
    const int s = stage_ids_[li];
    const int units = stages_[li]->units();
    const int words = stages_[li]->words();
    std::vector<uint64_t> tmp(static_cast<std::size_t>(M) * static_cast<std::size_t>(words));
    const bool hybrid_cell = controller && cfg_.hybrid && apf_base_ready_ &&
                             (phase == Phase::ProgressiveFreeze || phase == Phase::StableFreeze);
    if (hybrid_cell) {
      // Alg. 2: grow / shrink the APF base set to the cell's exact TimelyFreeze count
      const MaskStream& ms = mask_stream();
      const FreezeMask base = apf_base_mask(static_cast<int>(li));
      for (int m = 1; m <= M; ++m) {
        Rng rng(cell_seed(cfg_.seed, 0x2545f4914f6cdd1dULL, t, s, m));
        const auto mk = reconcile_mask(base, ms.cell_count(t, s, m), rng);
        std::memcpy(tmp.data() + static_cast<std::size_t>(m - 1) * static_cast<std::size_t>(words), mk.words().data(),
                    static_cast<size_t>(words) * 8);
      }
    } else if (controller) {
      mask_stream().stage_step_masks(t, s, tmp.data(), cfg_.mask_threads);
    } else {
      for (int m = 1; m <= M; ++m) {
        Rng rng(cell_seed(cfg_.seed, 0x51ed270b27f2e6a1ULL, t, s, m));
        const auto mk = sample_mask(units, override_ratio_, rng);
        std::memcpy(tmp.data() + static_cast<std::size_t>(m - 1) * static_cast<std::size_t>(words), mk.words().data(),
                    static_cast<size_t>(words) * 8);
      }
    }
    for (int m = 0; m < M; ++m) {
      uint64_t* dst = out + mask_offsets_[li] + static_cast<long long>(m) * (words + 1);
      std::memcpy(dst, tmp.data() + static_cast<std::size_t>(m) * static_cast<std::size_t>(words),
                  static_cast<size_t>(words) * 8);
      dst[words] = 0;
      long long pc = 0;
      for (int w = 0; w < words; ++w) pc += __builtin_popcountll(dst[w]);
      *frozen += pc;
      *total += units;
    }
  }
}

int Trainer::step(int t, const int* host_tokens, const int* host_targets, StepResult* out,
                  const uint64_t* host_masks) {
  cudaSetDevice(cfg_.device);
  const int S = cfg_.pipeline.total_stages(), M = cfg_.pipeline.num_microbatches;
  const int T = model_.tokens();
  StepResult res;
  Phase phase = Phase::StableFreeze;
  const bool controller = override_ratio_ < 0.0 && !host_masks;
  const int stamp = ++stamp_;
  if (controller) {
    phase = phase_of(t, cfg_.phases);
    if (phase == Phase::Solve && !plan_ready_) solve_plan_from_monitoring();
  }
  res.phase = static_cast<int>(phase);

  // ---- masks for this step's cells (host, jump-ahead into the single stream);
  // usually already generated while the previous step ran on the GPU
  const auto tm0 = std::chrono::steady_clock::now();
  if (host_masks) {  // caller-owned masks (reference plan / mask history replay)
    res.frozen_units = res.total_units = 0;
    long long src = 0;
    for (std::size_t li = 0; li < stages_.size(); ++li) {
      const int words = stages_[li]->words();
      const int units = stages_[li]->units();
      for (int m = 0; m < M; ++m) {
        uint64_t* dst = masks_host_ + mask_offsets_[li] + static_cast<long long>(m) * (words + 1);
        std::memcpy(dst, host_masks + src, static_cast<size_t>(words) * 8);
        if (units % 64) dst[words - 1] &= (1ULL << (units % 64)) - 1;  // bits past the last unit are not units
        dst[words] = 0;
        src += words;
        for (int w = 0; w < words; ++w) res.frozen_units += __builtin_popcountll(dst[w]);
        res.total_units += units;
      }
    }
  } else if (next_t_ == t && next_override_ == override_ratio_ && next_plan_ready_ == plan_ready_) {
    std::swap(masks_host_, masks_next_);
    res.frozen_units = next_frozen_;
    res.total_units = next_total_;
  } else {
    build_masks(t, phase, controller, masks_host_, &res.frozen_units, &res.total_units);
  }
  next_t_ = -1;
  res.mean_ratio = res.total_units ? static_cast<double>(res.frozen_units) / static_cast<double>(res.total_units) : 0.0;
  res.mask_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm0).count();

  // step origin: action start times are relative to this event, recorded before the step's
  // first enqueue (a caller that barriers all ranks right before step() gets one time axis)
  PF_CUDA(cudaEventRecord(ev_origin_, stream_));
  PF_CUDA(cudaMemcpyAsync(masks_dev_, masks_host_, static_cast<size_t>(mask_offsets_.back()) * 8,
                          cudaMemcpyHostToDevice, stream_));
  if (host_tokens)
    PF_CUDA(cudaMemcpyAsync(tokens_dev_, host_tokens, static_cast<size_t>(M) * T * 4, cudaMemcpyHostToDevice, stream_));
  if (host_targets)
    PF_CUDA(cudaMemcpyAsync(targets_dev_, host_targets, static_cast<size_t>(M) * T * 4, cudaMemcpyHostToDevice,
                            stream_));
  PF_CUDA(cudaMemsetAsync(loss_dev_, 0, 4, stream_));
  for (auto& st : stages_) PF_TRY(st->zero_dense_grads(stream_));

  // ---- the rank's action list (schedule order), one microbatch action at a time.
  // Remote neighbours (DAG rule-3 edges across ranks) go over NCCL P2P on the
  // activation / gradient streams, ordered against compute with events.
  const size_t act_bytes = static_cast<size_t>(T) * model_.hidden * 2;
  int ev_next = 0;
  auto fresh_event = [&]() -> cudaEvent_t {
    if (ev_next >= static_cast<int>(comm_ev_.size())) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      comm_ev_.push_back(e);
    }
    return comm_ev_[static_cast<std::size_t>(ev_next++)];
  };
  auto after = [&](cudaStream_t waiter, cudaStream_t producer) -> int {
    cudaEvent_t e = fresh_event();
    PF_CUDA(cudaEventRecord(e, producer));
    PF_CUDA(cudaStreamWaitEvent(waiter, e, 0));
    return PF_OK;
  };
  bool needs_comm = false;
  for (std::size_t i = 0; i < stage_ids_.size(); ++i) needs_comm |= !x_recv_[i].empty() || !dy_recv_[i].empty();
  if (needs_comm && !distributed()) return PF_ERR_NCCL;  // init_comm() first
  auto nccl_ok = [](ncclResult_t r) { return r == ncclSuccess ? PF_OK : PF_ERR_NCCL; };
  const int r = cfg_.rank;
  auto comm = [](const Link* l) { return static_cast<ncclComm_t>(l->comm); };
  for (std::size_t i = 0; i < actions_.size(); ++i) {
    const ActionId a = actions_[i];
    const int li = local_index(a.stage);
    const auto ls = static_cast<std::size_t>(li);
    Stage& st = *stages_[ls];
    const int slot = (a.microbatch - 1) % slots_[ls];
    const auto ss = static_cast<std::size_t>(slot);
    const int* tok = tokens_dev_ + static_cast<long long>(a.microbatch - 1) * T;
    const int* tgt = targets_dev_ + static_cast<long long>(a.microbatch - 1) * T;
    const IssueOp& op = program_[i];
    if (a.kind == ActionKind::Forward) {
      const __nv_bfloat16* x_in = nullptr;
      const bool recv_x = op.recv_from >= 0;
      const bool send_y = op.send_to >= 0;
      if (recv_x) {  // f(m, s-1) output over NVLink into this slot's receive buffer
        const Link* l = link(0, op.recv_from, r);
        if (!l || !l->comm) return PF_ERR_NCCL;
        PF_CUDA(cudaStreamWaitEvent(l->stream, x_free_ev_[ls][ss], 0));
        PF_TRY(nccl_ok(ncclRecv(x_recv_[ls][ss], act_bytes, ncclUint8, 0, comm(l), l->stream)));
        PF_TRY(after(stream_, l->stream));
        x_in = x_recv_[ls][ss];
      } else if (a.stage > 1) {
        const int lp = local_index(a.stage - 1);
        x_in = stages_[static_cast<std::size_t>(lp)]->output((a.microbatch - 1) % slots_[static_cast<std::size_t>(lp)]);
      }
      if (send_y) PF_CUDA(cudaStreamWaitEvent(stream_, out_sent_ev_[ls][ss], 0));  // slot output has left
      PF_CUDA(cudaEventRecord(ev_[2 * i], stream_));
      PF_TRY(st.forward(slot, a.microbatch, tok, tgt, x_in, loss_dev_, stream_));
      PF_CUDA(cudaEventRecord(ev_[2 * i + 1], stream_));
      if (recv_x) PF_CUDA(cudaEventRecord(x_free_ev_[ls][ss], stream_));
      if (send_y) {  // to f(m, s+1)
        const Link* l = link(0, r, op.send_to);
        if (!l || !l->comm) return PF_ERR_NCCL;
        PF_TRY(after(l->stream, stream_));
        PF_TRY(nccl_ok(ncclSend(st.output(slot), act_bytes, ncclUint8, 1, comm(l), l->stream)));
        PF_CUDA(cudaEventRecord(out_sent_ev_[ls][ss], l->stream));
      }
    } else if (a.kind == ActionKind::Weight) {  // split backward: dW of the slot's microbatch
      const uint64_t* mw = masks_dev_ + mask_offsets_[ls] + static_cast<long long>(a.microbatch - 1) * (st.words() + 1);
      st.set_dense_cell(cell_dense(ls, a.microbatch));
      PF_CUDA(cudaEventRecord(ev_[2 * i], stream_));
      PF_TRY(st.backward_weight(slot, mw, stamp, stream_));
      PF_CUDA(cudaEventRecord(ev_[2 * i + 1], stream_));
    } else {
      const bool recv_dy = op.recv_from >= 0;
      const bool send_dx = op.send_to >= 0;
      const __nv_bfloat16* dy = nullptr;
      if (recv_dy) {  // b(m, s+1) input gradient
        const Link* l = link(1, op.recv_from, r);
        if (!l || !l->comm) return PF_ERR_NCCL;
        PF_CUDA(cudaStreamWaitEvent(l->stream, dy_free_ev_[ls][ss], 0));
        PF_TRY(nccl_ok(ncclRecv(dy_recv_[ls][ss], act_bytes, ncclUint8, 0, comm(l), l->stream)));
        PF_TRY(after(stream_, l->stream));
        dy = dy_recv_[ls][ss];
      } else if (a.stage < S) {
        dy = grad_bufs_[ls][ss];
      }
      __nv_bfloat16* dx = nullptr;
      if (send_dx) {
        PF_CUDA(cudaStreamWaitEvent(stream_, dx_sent_ev_[ls][ss], 0));
        dx = dx_send_[ls][ss];
      } else if (a.stage > 1) {
        const int lp = local_index(a.stage - 1);
        dx = grad_bufs_[static_cast<std::size_t>(lp)][static_cast<std::size_t>((a.microbatch - 1) %
                                                                               slots_[static_cast<std::size_t>(lp)])];
      }
      const uint64_t* mw = masks_dev_ + mask_offsets_[ls] + static_cast<long long>(a.microbatch - 1) * (st.words() + 1);
      st.set_dense_cell(cell_dense(ls, a.microbatch));
      PF_CUDA(cudaEventRecord(ev_[2 * i], stream_));
      PF_TRY(st.backward(slot, tok, mw, dy, dx, stamp, stream_));
      PF_CUDA(cudaEventRecord(ev_[2 * i + 1], stream_));
      if (recv_dy) PF_CUDA(cudaEventRecord(dy_free_ev_[ls][ss], stream_));
      if (send_dx) {  // to b(m, s-1)
        const Link* l = link(1, r, op.send_to);
        if (!l || !l->comm) return PF_ERR_NCCL;
        PF_TRY(after(l->stream, stream_));
        PF_TRY(nccl_ok(ncclSend(dx, act_bytes, ncclUint8, 1, comm(l), l->stream)));
        PF_CUDA(cudaEventRecord(dx_sent_ev_[ls][ss], l->stream));
      }
    }
  }
  if (distributed()) {  // the step ends when its last transfers have landed
    for (const Link& l : links_)
      if (l.stream) PF_TRY(after(stream_, l.stream));
  }
  // ---- masked optimizer step: theta -= (eta / M) * sum_m U_m . g_m
  PF_CUDA(cudaEventRecord(ev_opt0_, stream_));
  const bool apf_step = cfg_.apf && (t % std::max(1, cfg_.apf_every) == 0);
  OptimCfg oc = cfg_.optim;
  oc.lr = static_cast<float>(cfg_.lr);
  for (auto& st : stages_)
    PF_TRY(st->optimizer_step(oc, M, stamp, apf_step, cfg_.apf_alpha, cfg_.apf_threshold, stream_));
  PF_CUDA(cudaEventRecord(ev_opt1_, stream_));
  PF_CUDA(cudaMemcpyAsync(loss_host_, loss_dev_, 4, cudaMemcpyDeviceToHost, stream_));
  if (apf_step && cfg_.hybrid) {  // per-unit APF eligibility counts for the next steps' base sets
    if (!apf_pinned_) {
      PF_CUDA(cudaMallocHost(&apf_pinned_, static_cast<size_t>(std::max(1, units_total())) * 4));
      apf_eligible_host_.resize(stages_.size());
    }
    int off = 0;
    for (auto& st : stages_) {
      PF_CUDA(cudaMemcpyAsync(apf_pinned_ + off, st->apf_eligible(), static_cast<size_t>(st->units()) * 4,
                              cudaMemcpyDeviceToHost, stream_));
      off += st->units();
    }
  }
  // the next step's masks while this one runs (not in hybrid mode, whose base set comes from
  // this step's APF result, nor across the LP solve, which changes the plan)
  if (!host_masks && !cfg_.hybrid && (!controller || t + 1 <= cfg_.phases.t_total)) {
    const Phase next_phase = controller ? phase_of(t + 1, cfg_.phases) : Phase::StableFreeze;
    if (!(controller && next_phase == Phase::Solve && !plan_ready_)) {
      build_masks(t + 1, next_phase, controller, masks_next_, &next_frozen_, &next_total_);
      next_t_ = t + 1;
      next_override_ = override_ratio_;
      next_plan_ready_ = plan_ready_;
    }
  }
  PF_CUDA(cudaStreamSynchronize(stream_));
  if (apf_step && cfg_.hybrid) {
    int off = 0;
    for (std::size_t li = 0; li < stages_.size(); ++li) {
      apf_eligible_host_[li].assign(apf_pinned_ + off, apf_pinned_ + off + stages_[li]->units());
      off += stages_[li]->units();
    }
    apf_base_ready_ = true;
  }

  action_ms_.assign(actions_.size(), 0.0);
  action_start_ms_.assign(actions_.size(), 0.0);
  for (std::size_t i = 0; i < actions_.size(); ++i) {
    float ms = 0.f, st = 0.f;
    cudaEventElapsedTime(&ms, ev_[2 * i], ev_[2 * i + 1]);
    cudaEventElapsedTime(&st, ev_origin_, ev_[2 * i]);
    action_ms_[i] = ms;
    action_start_ms_[i] = st;
  }
  float bms = 0.f, oms = 0.f;
  if (!actions_.empty()) cudaEventElapsedTime(&bms, ev_[0], ev_[2 * actions_.size() - 1]);
  cudaEventElapsedTime(&oms, ev_opt0_, ev_opt1_);
  res.batch_ms = bms;
  res.optimizer_ms = oms;
  const bool has_last = local_index(S) >= 0;
  res.loss = has_last ? static_cast<double>(*loss_host_) / M : std::nan("");

  // ---- monitoring (Alg. 1): upper bounds unfrozen, lower bounds fully frozen
  if (controller && (phase == Phase::MonitorUpper || phase == Phase::MonitorLower)) {
    for (std::size_t i = 0; i < actions_.size(); ++i) {
      const ActionId a = actions_[i];
      const FreezeState fs = (a == freeze_node(cfg_.pipeline, a.microbatch, a.stage) && phase == Phase::MonitorLower)
                                 ? FreezeState::Full
                                 : FreezeState::None;
      monitor_.record(a, t, action_ms_[i], fs);
    }
  }
  // ---- LP / DAG prediction of this step's batch time
  if (plan_ready_ && !plan_profile_.all().empty()) {
    double scale = 1.0;
    if (controller && phase == Phase::ProgressiveFreeze && cfg_.phases.t_freeze > cfg_.phases.t_monitor)
      scale = std::min(1.0, static_cast<double>(t - cfg_.phases.t_monitor) /
                                (cfg_.phases.t_freeze - cfg_.phases.t_monitor));
    if (!controller || phase == Phase::ProgressiveFreeze || phase == Phase::StableFreeze) {
      FreezePlan p = plan_;
      if (!controller && !host_masks)
        for (auto& [k, r] : p.ratios) r = override_ratio_;
      res.predicted_ms = longest_path_start_times(*dag_, plan_weights(*dag_, plan_profile_, p, scale)).makespan;
    }
  }
  if (out) *out = res;
  return PF_OK;
}

}  // namespace pf
