// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY. A thin extern "C" shim that lets the parity tests
// and bench.py's reference arm call the UNMODIFIED reference engine, compiled
// from /root/reference/proj/core/src/*.cpp into oracle/_ref/libswt_ref.so by
// oracle/Makefile. Nothing in paper_2211_16270_b200/ links or loads this.
//
// Wrapped reference entry points:
//   swt::synth_inputs<float>          proj/core/src/bench.cpp:66-115
//   swt::padded_lengths               proj/core/src/bench.cpp:48-64
//   swt::run_step<T>                  proj/core/src/engine.cpp:400-407
//   swt::transducer_loss_sample<T>    proj/core/src/loss.cpp:176-185
//   swt::oracle::enumerate_paths_loss proj/core/src/oracle.cpp:65-85
//   swt::oracle::count_paths          proj/core/src/oracle.cpp:10-22

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "swt/bench.hpp"
#include "swt/engine.hpp"
#include "swt/loss.hpp"
#include "swt/oracle.hpp"

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const swt::InvalidShapeError*>(&e)) return 1;
  if (dynamic_cast<const swt::InvalidInputError*>(&e)) return 2;
  if (dynamic_cast<const swt::NumericalDegeneracyError*>(&e)) return 3;
  if (dynamic_cast<const swt::OutOfMemoryError*>(&e)) return 4;
  return 7;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

template <typename T, typename S>
swt::Tensor<T> make(std::initializer_list<std::int64_t> shape, const S* src,
                    const char* tag) {
  auto t = swt::Tensor<T>::zeros(swt::Shape(shape), tag);
  for (std::int64_t i = 0; i < t.size(); ++i) t.data()[i] = T(src[i]);
  return t;
}

template <typename T, typename D>
void put(const swt::Tensor<T>& t, D* dst) {
  if (!dst) return;
  for (std::int64_t i = 0; i < t.size(); ++i) dst[i] = D(t.data()[i]);
}

template <typename T, typename S>
int run_step_t(int64_t B, int64_t T_, int64_t U, int64_t HA, int64_t HL,
               int64_t H, int64_t V, const S* acoustic, const S* label,
               const int32_t* labels, const int64_t* t_len,
               const int64_t* u_len, const S* wa, const S* wl, const S* bz,
               const S* wo, const S* bo, int mode, int64_t budget,
               int max_parallel, int workers, S* loss, S* sample_losses,
               S* dwa, S* dwl, S* dbz, S* dwo, S* dbo, S* dac, S* dlb) {
  return guard([&] {
    swt::Batch<T> batch;
    batch.acoustic = make<T>({B, T_, HA}, acoustic, "h_acoustic");
    batch.label = make<T>({B, U + 1, HL}, label, "h_label");
    batch.labels.assign(labels, labels + B * U);
    batch.t_len.assign(t_len, t_len + B);
    batch.u_len.assign(u_len, u_len + B);
    swt::JointParams<T> jp{make<T>({H, HA}, wa, "w_acoustic"),
                           make<T>({H, HL}, wl, "w_label"),
                           make<T>({H}, bz, "bias_joint")};
    swt::OutputParams<T> op{make<T>({V, H}, wo, "w_out"),
                            make<T>({V}, bo, "bias_out")};
    swt::EngineConfig cfg;
    cfg.mode = swt::EngineMode(mode);
    cfg.mem_budget_bytes = budget;
    cfg.max_parallel = max_parallel;
    cfg.worker_count = workers;
    const swt::StepResult<T> r = swt::run_step(batch, jp, op, cfg);
    if (loss) *loss = S(r.loss);
    if (sample_losses)
      for (int64_t b = 0; b < B; ++b) sample_losses[b] = S(r.sample_losses[b]);
    put(r.grads.dw_acoustic, dwa);
    put(r.grads.dw_label, dwl);
    put(r.grads.dbias, dbz);
    put(r.grads.dw_out, dwo);
    put(r.grads.dbias_out, dbo);
    put(r.grads.dacoustic, dac);
    put(r.grads.dlabel, dlb);
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_synth_inputs(int64_t B, int64_t T, int64_t U, int64_t H, int64_t HA,
                     int64_t HL, int64_t V, uint64_t seed, float* acoustic,
                     float* label, int32_t* labels, int64_t* t_len,
                     int64_t* u_len, float* wa, float* wl, float* bz,
                     float* wo, float* bo) {
  return guard([&] {
    swt::BenchConfig cfg;
    cfg.batch_size = B;
    cfg.max_frames = T;
    cfg.max_labels = U;
    cfg.joint_dim = H;
    cfg.acoustic_dim = HA;
    cfg.label_dim = HL;
    cfg.vocab = V;
    cfg.seed = seed;
    swt::BenchInputs<float> in = swt::synth_inputs<float>(cfg);
    put(in.batch.acoustic, acoustic);
    put(in.batch.label, label);
    std::memcpy(labels, in.batch.labels.data(), in.batch.labels.size() * 4);
    std::memcpy(t_len, in.batch.t_len.data(), size_t(B) * 8);
    std::memcpy(u_len, in.batch.u_len.data(), size_t(B) * 8);
    put(in.jp.w_acoustic, wa);
    put(in.jp.w_label, wl);
    put(in.jp.bias, bz);
    put(in.op.w_out, wo);
    put(in.op.bias_out, bo);
  });
}

// run_step<float> on float inputs.
int ref_run_step_f32(int64_t B, int64_t T, int64_t U, int64_t HA, int64_t HL,
                     int64_t H, int64_t V, const float* acoustic,
                     const float* label, const int32_t* labels,
                     const int64_t* t_len, const int64_t* u_len,
                     const float* wa, const float* wl, const float* bz,
                     const float* wo, const float* bo, int mode,
                     int64_t budget, int max_parallel, int workers,
                     float* loss, float* sample_losses, float* dwa,
                     float* dwl, float* dbz, float* dwo, float* dbo,
                     float* dac, float* dlb) {
  return run_step_t<float>(B, T, U, HA, HL, H, V, acoustic, label, labels,
                           t_len, u_len, wa, wl, bz, wo, bo, mode, budget,
                           max_parallel, workers, loss, sample_losses, dwa,
                           dwl, dbz, dwo, dbo, dac, dlb);
}

// run_step<double> on double inputs (the parity golden: f32 inputs widened).
int ref_run_step_f64(int64_t B, int64_t T, int64_t U, int64_t HA, int64_t HL,
                     int64_t H, int64_t V, const double* acoustic,
                     const double* label, const int32_t* labels,
                     const int64_t* t_len, const int64_t* u_len,
                     const double* wa, const double* wl, const double* bz,
                     const double* wo, const double* bo, int mode,
                     int64_t budget, int max_parallel, int workers,
                     double* loss, double* sample_losses, double* dwa,
                     double* dwl, double* dbz, double* dwo, double* dbo,
                     double* dac, double* dlb) {
  return run_step_t<double>(B, T, U, HA, HL, H, V, acoustic, label, labels,
                            t_len, u_len, wa, wl, bz, wo, bo, mode, budget,
                            max_parallel, workers, loss, sample_losses, dwa,
                            dwl, dbz, dwo, dbo, dac, dlb);
}

int ref_transducer_loss_f64(const double* scores, int64_t frames,
                            int64_t labels, int64_t vocab, const int32_t* y,
                            double* loss, double* dscores) {
  return guard([&] {
    auto s = make<double>({frames, labels + 1, vocab}, scores, "scores");
    std::vector<int32_t> yy(y, y + labels);
    auto r = swt::transducer_loss_sample(s, swt::LabelSequence(yy));
    *loss = r.value;
    put(r.dscores, dscores);
  });
}

int ref_enumerate_paths_loss(const double* scores, int64_t frames,
                             int64_t labels, int64_t vocab, const int32_t* y,
                             double* loss) {
  return guard([&] {
    auto s = make<double>({frames, labels + 1, vocab}, scores, "scores");
    auto den = swt::log_denominator(s);
    std::vector<int32_t> yy(y, y + labels);
    *loss = swt::oracle::enumerate_paths_loss(s, den, swt::LabelSequence(yy));
  });
}

int64_t ref_count_paths(int64_t frames, int64_t labels) {
  return swt::oracle::count_paths(frames, labels);
}

// swt::padded_lengths (proj/core/src/bench.cpp:48-64): the measurement ramp
int ref_padded_lengths(int64_t B, int64_t T, int64_t U, int64_t* t_len,
                       int64_t* u_len) {
  return guard([&] {
    const swt::SampleLengths s = swt::padded_lengths(B, T, U);
    std::memcpy(t_len, s.t_len.data(), size_t(B) * sizeof(int64_t));
    std::memcpy(u_len, s.u_len.data(), size_t(B) * sizeof(int64_t));
  });
}

int ref_parallel_iterations(int64_t f, int64_t l, int64_t v, int64_t b) {
  int r = -1;
  guard([&] { r = swt::compute_parallel_iterations(f, l, v, b); });
  return r;
}

}  // extern "C"
