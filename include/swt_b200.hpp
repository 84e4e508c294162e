// SPDX-License-Identifier: Apache-2.0
//
// swt_b200.hpp — C++ host API of libswt_b200, shaped like the reference
// engine API so a caller of swt::run_step switches by namespace:
//
//   reference                                   here
//   swt::run_step<float>(batch, jp, op, cfg)    swt::b200::run_step(batch, jp, op, cfg)
//     core/include/swt/engine.hpp:116-118         (one-shot context on device 0)
//                                               swt::b200::Engine(opts).run_step(...)
//   swt::Batch<float>        engine.hpp:28-46   swt::b200::Batch
//   swt::JointParams<float>  compute.hpp:13-23  swt::b200::JointParams
//   swt::OutputParams<float> compute.hpp:25-32  swt::b200::OutputParams
//   swt::GradientSet<float>  engine.hpp:49-58   swt::b200::GradientSet
//   swt::EngineConfig        engine.hpp:74-82   swt::b200::EngineConfig
//   swt::StepResult<float>   engine.hpp:84-89   swt::b200::StepResult
//   swt::compute_parallel_iterations engine.hpp:93-94
//   swt::padded_lengths / synth_inputs<float>   bench.hpp:67-81
//   swt::InvalidShapeError … OutOfMemoryError   errors.hpp:12-66
//
// Header-only; everything below the types is a thin call into the C ABI of
// include/swt_b200.h (no CUDA or torch types cross it). Tensors are host
// row-major float buffers with the reference's extents; device-resident
// callers use Engine::run_step_device with raw device pointers.

#pragma once

#include <cstdint>
#include <initializer_list>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "swt_b200.h"

namespace swt::b200 {

// ---- errors (reference core/include/swt/errors.hpp:12-66) ------------------

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidShapeError : Error {
  using Error::Error;
};
struct InvalidInputError : Error {
  using Error::Error;
};
struct NumericalDegeneracyError : Error {
  using Error::Error;
};
struct OutOfMemoryError : Error {
  using Error::Error;
  OutOfMemoryError(const std::string& m, std::string tensor, std::int64_t bytes)
      : Error(m), tensor_(std::move(tensor)), request_bytes_(bytes) {}
  const std::string& tensor() const noexcept { return tensor_; }
  std::int64_t request_bytes() const noexcept { return request_bytes_; }

 private:
  std::string tensor_;
  std::int64_t request_bytes_ = 0;
};
struct CudaError : Error {
  using Error::Error;
};
struct NcclError : Error {
  using Error::Error;
};

inline void check(swtb_status s, const swtb_ctx* ctx = nullptr) {
  if (s == SWTB_OK) return;
  const std::string m = swtb_last_error(ctx);
  switch (s) {
    case SWTB_ERR_SHAPE: throw InvalidShapeError(m);
    case SWTB_ERR_INPUT: throw InvalidInputError(m);
    case SWTB_ERR_NUMERIC: throw NumericalDegeneracyError(m);
    case SWTB_ERR_OOM: {
      std::int64_t bytes = 0;
      char name[64] = {0};
      if (ctx && swtb_last_oom(ctx, &bytes, name, sizeof name) == SWTB_OK)
        throw OutOfMemoryError(m, name, bytes);
      throw OutOfMemoryError(m);
    }
    case SWTB_ERR_CUDA: throw CudaError(m);
    case SWTB_ERR_NCCL: throw NcclError(m);
    default: throw Error(m);
  }
}

// ---- host tensor: rank <= 4, row-major, owning (reference tensor.hpp:152) ---

class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<std::int64_t> shape)
      : shape_(std::move(shape)), data_(size_of(shape_), 0.f) {}
  Tensor(std::initializer_list<std::int64_t> shape)
      : Tensor(std::vector<std::int64_t>(shape)) {}

  std::int64_t rank() const { return std::int64_t(shape_.size()); }
  std::int64_t extent(std::size_t i) const { return shape_.at(i); }
  const std::vector<std::int64_t>& shape() const { return shape_; }
  std::int64_t size() const { return std::int64_t(data_.size()); }
  float* data() { return data_.data(); }
  const float* data() const { return data_.data(); }
  float& operator[](std::int64_t i) { return data_[std::size_t(i)]; }
  float operator[](std::int64_t i) const { return data_[std::size_t(i)]; }

 private:
  static std::size_t size_of(const std::vector<std::int64_t>& s) {
    return std::size_t(std::accumulate(s.begin(), s.end(), std::int64_t(1),
                                       std::multiplies<>()));
  }
  std::vector<std::int64_t> shape_;
  std::vector<float> data_;
};

// ---- reference-shaped types ------------------------------------------------

enum class EngineMode { batched, sample_wise, sample_wise_pr, sample_wise_pr_dp };

enum class Precision {
  bf16 = SWTB_PREC_BF16,
  tf32 = SWTB_PREC_TF32,
  bf16x = SWTB_PREC_BF16X,
  fp16 = SWTB_PREC_FP16
};

struct Batch {
  Tensor acoustic;                   // [B, T, H_A]
  Tensor label;                      // [B, U+1, H_L]
  std::vector<std::int32_t> labels;  // [B, U] flat, zero-padded
  std::vector<std::int64_t> t_len;   // 1 <= t_len[b] <= T
  std::vector<std::int64_t> u_len;   // 0 <= u_len[b] <= U
  // extension (not in swt::Batch): per-sample loss weights w_b >= 0; empty =
  // all 1. Gradients become those of sum_b w_b L_b (losses stay unweighted).
  std::vector<float> sample_weights;

  std::int64_t batch_size() const { return acoustic.extent(0); }
  std::int64_t max_frames() const { return acoustic.extent(1); }
  std::int64_t label_rows() const { return label.extent(1); }
  std::int64_t max_labels() const { return label_rows() - 1; }
  std::int64_t acoustic_dim() const { return acoustic.extent(2); }
  std::int64_t label_dim() const { return label.extent(2); }
};

struct JointParams {
  Tensor w_acoustic;  // [H, H_A]
  Tensor w_label;     // [H, H_L]
  Tensor bias;        // [H]
};

struct OutputParams {
  Tensor w_out;     // [V, H]
  Tensor bias_out;  // [V]
};

struct GradientSet {
  Tensor dw_acoustic;  // [H, H_A]
  Tensor dw_label;     // [H, H_L]
  Tensor dbias;        // [H]
  Tensor dw_out;       // [V, H]
  Tensor dbias_out;    // [V]
  Tensor dacoustic;    // [B, T, H_A], zero in padded regions
  Tensor dlabel;       // [B, U+1, H_L], zero in padded regions
};

struct EngineConfig {
  EngineMode mode = EngineMode::sample_wise;
  std::int64_t mem_budget_bytes = 1'000'000'000;
  int max_parallel = 16;
  int worker_count = 1;
  bool literal_pi_extents = false;
};

struct StepResult {
  float loss = 0;  // sum of per-sample losses, ascending index
  std::vector<float> sample_losses;
  GradientSet grads;
};

struct Options {
  int device = 0;
  Precision precision = Precision::fp16;  // fp32-grade parity at the 16-bit MMA rate
  int rank = 0;
  int nranks = 1;
  const void* nccl_id = nullptr;  // 128-byte ncclUniqueId when nranks > 1
  std::int64_t group_cells = 0;   // 0 = library default
};

// ---- engine ----------------------------------------------------------------

class Engine {
 public:
  explicit Engine(const Options& o = {}) {
    swtb_opts so{o.device, o.rank, o.nranks, o.nccl_id, int(o.precision), o.group_cells};
    swtb_ctx* c = nullptr;
    check(swtb_ctx_create(&so, &c));
    ctx_.reset(c);
  }

  /// swt::run_step on host tensors (the library stages H2D/D2H itself).
  StepResult run_step(const Batch& b, const JointParams& jp, const OutputParams& op,
                      const EngineConfig& cfg = {}) {
    if (b.acoustic.rank() != 3 || b.label.rank() != 3 ||
        b.label.extent(0) != b.batch_size() || jp.w_acoustic.rank() != 2 ||
        op.w_out.rank() != 2)
      throw InvalidShapeError("batch encoding tensors are inconsistent");
    const std::int64_t B = b.batch_size(), T = b.max_frames(), U = b.max_labels();
    const std::int64_t HA = b.acoustic_dim(), HL = b.label_dim();
    const std::int64_t H = op.w_out.extent(1), V = op.w_out.extent(0);
    if (jp.w_acoustic.extent(0) != H || jp.w_acoustic.extent(1) != HA ||
        jp.w_label.extent(0) != H || jp.w_label.extent(1) != HL ||
        jp.bias.size() != H || op.bias_out.size() != V)
      throw InvalidShapeError("parameter extents do not match the batch");
    if (std::int64_t(b.t_len.size()) != B || std::int64_t(b.u_len.size()) != B ||
        std::int64_t(b.labels.size()) != B * U)
      throw InvalidShapeError("batch length/label arrays are inconsistent");
    StepResult r;
    r.sample_losses.assign(std::size_t(B), 0.f);
    GradientSet& g = r.grads;
    g.dw_acoustic = Tensor{H, HA};
    g.dw_label = Tensor{H, HL};
    g.dbias = Tensor{H};
    g.dw_out = Tensor{V, H};
    g.dbias_out = Tensor{V};
    g.dacoustic = Tensor{B, T, HA};
    g.dlabel = Tensor{B, U + 1, HL};
    if (!b.sample_weights.empty() && std::int64_t(b.sample_weights.size()) != B)
      throw InvalidShapeError("sample_weights must have one entry per sample");
    swtb_batch cb{B, T, U, HA, HL, b.acoustic.data(), b.label.data(),
                  b.labels.data(), b.t_len.data(), b.u_len.data(), SWTB_HOST, 0,
                  b.sample_weights.empty() ? nullptr : b.sample_weights.data()};
    swtb_params cp{H, V, jp.w_acoustic.data(), jp.w_label.data(), jp.bias.data(),
                   op.w_out.data(), op.bias_out.data(), SWTB_HOST};
    swtb_cfg cc = c_cfg(cfg);
    swtb_out co{&r.loss, r.sample_losses.data(), g.dw_acoustic.data(),
                g.dw_label.data(), g.dbias.data(), g.dw_out.data(),
                g.dbias_out.data(), g.dacoustic.data(), g.dlabel.data(), SWTB_HOST};
    check(swtb_step(ctx_.get(), &cb, &cp, &cc, &co), ctx_.get());
    return r;
  }

  /// Device-resident variant: every pointer in batch/params/out is device
  /// memory (lengths stay host arrays); no host copies of the data path.
  void run_step_device(swtb_batch batch, swtb_params params, const EngineConfig& cfg,
                       swtb_out out) {
    batch.location = params.location = out.location = SWTB_DEVICE;
    swtb_cfg cc = c_cfg(cfg);
    check(swtb_step(ctx_.get(), &batch, &params, &cc, &out), ctx_.get());
  }

  swtb_stats stats() const {
    swtb_stats s{};
    check(swtb_get_stats(ctx_.get(), &s), ctx_.get());
    return s;
  }
  std::int64_t peak_bytes() const { return swtb_peak_bytes(ctx_.get()); }
  void reset_peak() { swtb_reset_peak(ctx_.get()); }
  // simulated allocation ceiling (reference BenchConfig.alloc_ceiling_bytes)
  void set_alloc_ceiling(std::int64_t bytes) { swtb_set_alloc_ceiling(ctx_.get(), bytes); }
  // bitwise-reproducible theta-grads (default on)
  void set_deterministic(bool on) { swtb_set_deterministic(ctx_.get(), on ? 1 : 0); }
  /// Order each later step after the work enqueued so far on `stream` (a
  /// cudaStream_t that produces device inputs; see swtb_set_caller_stream).
  void set_caller_stream(void* stream, bool enable = true) {
    check(swtb_set_caller_stream(ctx_.get(), stream, enable ? 1 : 0), ctx_.get());
  }
  void* stream() const { return swtb_stream(ctx_.get()); }
  swtb_ctx* handle() const { return ctx_.get(); }

  /// swt::transducer_loss_sample on explicit scores [frames, labels+1, vocab]
  /// (reference core/include/swt/loss.hpp:119-121), f64 host buffers.
  double transducer_loss(const std::vector<double>& scores, std::int64_t frames,
                         std::int64_t labels, std::int64_t vocab,
                         const std::vector<std::int32_t>& y,
                         std::vector<double>* dscores = nullptr) {
    double loss = 0;
    if (dscores) dscores->assign(scores.size(), 0.0);
    check(swtb_transducer_loss(ctx_.get(), scores.data(), frames, labels, vocab,
                               y.empty() ? nullptr : y.data(), &loss,
                               dscores ? dscores->data() : nullptr),
          ctx_.get());
    return loss;
  }

 private:
  static swtb_cfg c_cfg(const EngineConfig& c) {
    return swtb_cfg{int(c.mode), c.mem_budget_bytes, c.max_parallel,
                    c.worker_count, c.literal_pi_extents ? 1 : 0};
  }
  struct Del {
    void operator()(swtb_ctx* c) const { swtb_ctx_destroy(c); }
  };
  std::unique_ptr<swtb_ctx, Del> ctx_;
};

/// One-shot swt::run_step (reference engine.hpp:116-118): creates a context
/// on `opts.device`, runs one step, frees it.
inline StepResult run_step(const Batch& b, const JointParams& jp, const OutputParams& op,
                           const EngineConfig& cfg, const Options& opts = {}) {
  Engine e(opts);
  return e.run_step(b, jp, op, cfg);
}

// ---- context-free helpers ----------------------------------------------------

inline int compute_parallel_iterations(std::int64_t frames, std::int64_t labels,
                                       std::int64_t vocab, std::int64_t budget_bytes) {
  const int r = swtb_parallel_iterations(frames, labels, vocab, budget_bytes);
  if (r < 0) throw InvalidInputError(swtb_last_error(nullptr));
  return r;
}

inline std::pair<std::vector<std::int64_t>, std::vector<std::int64_t>> padded_lengths(
    std::int64_t batch, std::int64_t max_frames, std::int64_t max_labels) {
  std::vector<std::int64_t> t(std::size_t(batch > 0 ? batch : 0)), u(t.size());
  check(swtb_padded_lengths(batch, max_frames, max_labels, t.data(), u.data()));
  return {t, u};
}

struct SynthConfig {
  std::int64_t batch = 1, max_frames = 1, max_labels = 1, joint_dim = 1,
               acoustic_dim = 1, label_dim = 1, vocab = 2;
  std::uint64_t seed = 1;
};

struct SynthInputs {
  Batch batch;
  JointParams jp;
  OutputParams op;
};

/// Bit-identical to swt::synth_inputs<float> (reference bench.cpp:66-115).
inline SynthInputs synth_inputs(const SynthConfig& c) {
  SynthInputs s;
  const std::int64_t B = c.batch, T = c.max_frames, U = c.max_labels, H = c.joint_dim,
                     HA = c.acoustic_dim, HL = c.label_dim, V = c.vocab;
  if (B < 1 || T < 1 || U < 1 || H < 1 || HA < 1 || HL < 1 || V < 2)
    throw InvalidInputError("all benchmark dimensions must be >= 1");
  s.batch.acoustic = Tensor{B, T, HA};
  s.batch.label = Tensor{B, U + 1, HL};
  s.batch.labels.assign(std::size_t(B * U), 0);
  s.batch.t_len.assign(std::size_t(B), 0);
  s.batch.u_len.assign(std::size_t(B), 0);
  s.jp.w_acoustic = Tensor{H, HA};
  s.jp.w_label = Tensor{H, HL};
  s.jp.bias = Tensor{H};
  s.op.w_out = Tensor{V, H};
  s.op.bias_out = Tensor{V};
  swtb_synth_cfg sc{B, T, U, H, HA, HL, V, c.seed};
  check(swtb_synth_inputs(&sc, s.batch.acoustic.data(), s.batch.label.data(),
                          s.batch.labels.data(), s.batch.t_len.data(),
                          s.batch.u_len.data(), s.jp.w_acoustic.data(),
                          s.jp.w_label.data(), s.jp.bias.data(), s.op.w_out.data(),
                          s.op.bias_out.data()));
  return s;
}

}  // namespace swt::b200
