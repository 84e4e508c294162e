// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — C++ drop-in parity driver.
//
// Links the UNMODIFIED reference engine (compiled from
// /root/reference/proj/core/src by oracle/Makefile) and libswt_b200 through
// its C++ host API (include/swt_b200.hpp), and runs both on identical inputs
// exactly the way a caller of swt::run_step would after switching namespace:
//
//   auto in  = swt::synth_inputs<float>(cfg);                 // reference
//   auto ref = swt::run_step<double>(widen(in), cfg.engine);  // parity golden
//   auto got = swt::b200::run_step(copy(in), cfg.engine);     // this library
//
// Metric: loss relative error; per gradient tensor
// max|x - y| / max|y|. Bounds per precision as in tests/test_gpu_step.py.
// Also checks that the reference's error taxonomy maps onto the same
// swt::b200 exception types. Prints one JSON line per case; exit 0 iff all
// cases pass. Needs a B200 (the library has no CPU path).

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "swt/bench.hpp"
#include "swt/engine.hpp"
#include "swt_b200.hpp"

namespace b2 = swt::b200;

namespace {

template <typename D, typename S>
swt::Tensor<D> widen(const swt::Tensor<S>& t, const char* tag) {
  auto o = swt::Tensor<D>::zeros(t.shape(), tag);
  for (std::int64_t i = 0; i < t.size(); ++i) o.data()[i] = D(t.data()[i]);
  return o;
}

b2::Tensor to_b2(const swt::Tensor<float>& t) {
  std::vector<std::int64_t> shape;
  for (int i = 0; i < t.shape().rank(); ++i) shape.push_back(t.extent(i));
  b2::Tensor o(shape);
  std::memcpy(o.data(), t.data(), sizeof(float) * size_t(t.size()));
  return o;
}

double rel(const b2::Tensor& x, const swt::Tensor<double>& y) {
  double num = 0, den = 0;
  for (std::int64_t i = 0; i < y.size(); ++i) {
    num = std::max(num, std::fabs(double(x[i]) - y.data()[i]));
    den = std::max(den, std::fabs(y.data()[i]));
  }
  return den > 0 ? num / den : num;
}

struct Case {
  std::string name;
  swt::BenchConfig cfg;
  // optional edits of the synthesized batch (ragged lengths, U_b = 0, ...)
  std::function<void(swt::Batch<float>&)> edit;
};

void zero_padding(swt::Batch<float>& b) {
  const std::int64_t B = b.batch_size(), T = b.max_frames(), U = b.max_labels();
  const std::int64_t HA = b.acoustic_dim(), HL = b.label_dim();
  for (std::int64_t s = 0; s < B; ++s) {
    for (std::int64_t t = b.t_len[s]; t < T; ++t)
      for (std::int64_t h = 0; h < HA; ++h) b.acoustic.data()[(s * T + t) * HA + h] = 0;
    for (std::int64_t u = b.u_len[s] + 1; u <= U; ++u)
      for (std::int64_t h = 0; h < HL; ++h) b.label.data()[(s * (U + 1) + u) * HL + h] = 0;
    for (std::int64_t u = b.u_len[s]; u < U; ++u) b.labels[size_t(s * U + u)] = 0;
  }
}

// mode: the engine mode of both sides (the reference's batched / sample_wise
// engines are the golden for ours; the +PR modes use sample_wise_pr)
int run_case(const Case& c, b2::Precision prec, double tol_loss, double tol_grad,
             b2::EngineMode mode = b2::EngineMode::sample_wise_pr_dp) {
  auto in = swt::synth_inputs<float>(c.cfg);
  if (c.edit) {
    c.edit(in.batch);
    zero_padding(in.batch);
  }
  // golden: the reference engine in f64 on the f32 inputs widened exactly
  swt::Batch<double> bd;
  bd.acoustic = widen<double>(in.batch.acoustic, "h_acoustic");
  bd.label = widen<double>(in.batch.label, "h_label");
  bd.labels = in.batch.labels;
  bd.t_len = in.batch.t_len;
  bd.u_len = in.batch.u_len;
  swt::JointParams<double> jd{widen<double>(in.jp.w_acoustic, "wa"),
                              widen<double>(in.jp.w_label, "wl"),
                              widen<double>(in.jp.bias, "bz")};
  swt::OutputParams<double> od{widen<double>(in.op.w_out, "wo"),
                               widen<double>(in.op.bias_out, "bo")};
  swt::EngineConfig rcfg = c.cfg.engine_config();
  rcfg.mode = mode == b2::EngineMode::batched       ? swt::EngineMode::batched
              : mode == b2::EngineMode::sample_wise ? swt::EngineMode::sample_wise
                                                    : swt::EngineMode::sample_wise_pr;
  const swt::StepResult<double> ref = swt::run_step(bd, jd, od, rcfg);

  // this library through the drop-in host API
  b2::Batch b;
  b.acoustic = to_b2(in.batch.acoustic);
  b.label = to_b2(in.batch.label);
  b.labels = in.batch.labels;
  b.t_len = in.batch.t_len;
  b.u_len = in.batch.u_len;
  b2::JointParams jp{to_b2(in.jp.w_acoustic), to_b2(in.jp.w_label), to_b2(in.jp.bias)};
  b2::OutputParams op{to_b2(in.op.w_out), to_b2(in.op.bias_out)};
  b2::EngineConfig cfg;
  cfg.mode = mode;
  b2::Options opts;
  opts.precision = prec;
  const b2::StepResult got = b2::run_step(b, jp, op, cfg, opts);

  const double el = std::fabs(got.loss - ref.loss) / std::fabs(ref.loss);
  double es = 0;
  for (size_t i = 0; i < ref.sample_losses.size(); ++i)
    es = std::max(es, std::fabs(got.sample_losses[i] - ref.sample_losses[i]) /
                          std::fabs(ref.sample_losses[i]));
  const double e[7] = {rel(got.grads.dw_acoustic, ref.grads.dw_acoustic),
                       rel(got.grads.dw_label, ref.grads.dw_label),
                       rel(got.grads.dbias, ref.grads.dbias),
                       rel(got.grads.dw_out, ref.grads.dw_out),
                       rel(got.grads.dbias_out, ref.grads.dbias_out),
                       rel(got.grads.dacoustic, ref.grads.dacoustic),
                       rel(got.grads.dlabel, ref.grads.dlabel)};
  double eg = 0;
  for (double x : e) eg = std::max(eg, x);
  // padded slots must be exactly zero (reference test_engine.cpp:327-347)
  bool pad_zero = true;
  const std::int64_t T = b.max_frames(), U1 = b.label_rows();
  const std::int64_t HA = b.acoustic_dim(), HL = b.label_dim();
  for (std::int64_t s = 0; s < b.batch_size(); ++s) {
    for (std::int64_t i = (s * T + b.t_len[size_t(s)]) * HA; i < (s + 1) * T * HA; ++i)
      pad_zero &= got.grads.dacoustic[i] == 0.f;
    for (std::int64_t i = (s * U1 + b.u_len[size_t(s)] + 1) * HL; i < (s + 1) * U1 * HL; ++i)
      pad_zero &= got.grads.dlabel[i] == 0.f;
  }
  const bool ok = el <= tol_loss && es <= tol_loss && eg <= tol_grad && pad_zero;
  static const char* pn[] = {"bf16", "tf32", "bf16x", "fp16"};
  static const char* mn[] = {"batched", "sample_wise", "sample_wise_pr", "sample_wise_pr_dp"};
  std::printf(
      "{\"case\": \"%s\", \"mode\": \"%s\", \"precision\": \"%s\", \"loss\": %.9g, \"ref_loss\": %.12g, "
      "\"loss_rel\": %.3g, \"sample_loss_rel\": %.3g, \"grad_rel\": {\"dw_acoustic\": %.3g, "
      "\"dw_label\": %.3g, \"dbias\": %.3g, \"dw_out\": %.3g, \"dbias_out\": %.3g, "
      "\"dacoustic\": %.3g, \"dlabel\": %.3g}, \"padding_zero\": %s, \"tol\": [%g, %g], "
      "\"pass\": %s}\n",
      c.name.c_str(), mn[int(mode)], pn[int(prec)], got.loss, ref.loss, el, es, e[0], e[1], e[2], e[3], e[4],
      e[5], e[6], pad_zero ? "true" : "false", tol_loss, tol_grad, ok ? "true" : "false");
  std::fflush(stdout);
  return ok ? 0 : 1;
}

template <class Ex, class F>
int expect_throw(const char* what, F&& f) {
  try {
    f();
  } catch (const Ex&) {
    std::printf("{\"error_case\": \"%s\", \"pass\": true}\n", what);
    return 0;
  } catch (const std::exception& e) {
    std::printf("{\"error_case\": \"%s\", \"pass\": false, \"got\": \"%s\"}\n", what, e.what());
    return 1;
  }
  std::printf("{\"error_case\": \"%s\", \"pass\": false, \"got\": \"no throw\"}\n", what);
  return 1;
}

swt::BenchConfig bc(std::int64_t B, std::int64_t T, std::int64_t U, std::int64_t V,
                    std::int64_t H, std::int64_t HA = 0, std::int64_t HL = 0) {
  swt::BenchConfig c;
  c.batch_size = B;
  c.max_frames = T;
  c.max_labels = U;
  c.vocab = V;
  c.joint_dim = H;
  c.acoustic_dim = HA ? HA : H;
  c.label_dim = HL ? HL : H;
  c.seed = 1;
  return c;
}

}  // namespace

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::strcmp(argv[1], "--quick") == 0;
  std::vector<Case> cases = {
      {"c1", bc(1, 50, 10, 32, 64), nullptr},
      {"c1_B4", bc(4, 50, 10, 32, 64), nullptr},
      {"ragged_HA_HL", bc(5, 37, 9, 45, 40, 26, 27),
       [](swt::Batch<float>& b) {
         const std::int64_t t[5] = {1, 37, 20, 5, 33}, u[5] = {0, 9, 3, 9, 1};
         for (int i = 0; i < 5; ++i) {
           b.t_len[size_t(i)] = t[i];
           b.u_len[size_t(i)] = u[i];
           for (int k = 0; k < u[i]; ++k)  // valid ids in [1, V=45)
             b.labels[size_t(i * 9 + k)] = 1 + (i * 7 + k * 3) % 44;
         }
       }},
      {"U_much_greater_than_T", bc(2, 3, 40, 11, 32), nullptr},
  };
  if (!quick) cases.push_back({"c2_B4", bc(4, 200, 50, 512, 256), nullptr});
  int fails = 0;
  for (const Case& c : cases) {
    fails += run_case(c, b2::Precision::fp16, 1e-4, 1e-3);
    fails += run_case(c, b2::Precision::tf32, 1e-4, 1e-3);
    fails += run_case(c, b2::Precision::bf16x, 1e-4, 5e-3);
    fails += run_case(c, b2::Precision::bf16, 5e-4, 3e-2);
  }
  // engine modes: our batched comparator and padded sample-wise engine
  // against the reference's run_batched / sample_wise engines
  for (const Case& c : {cases[1], cases[2]})
    for (b2::EngineMode m : {b2::EngineMode::batched, b2::EngineMode::sample_wise})
      fails += run_case(c, b2::Precision::tf32, 1e-4, 1e-3, m);
  // OOM simulation (reference acceptance.cpp:415-447): a ceiling of half
  // the analytic batched 4D footprint fails batched, not the sample-wise
  // engines; the refused tensor is named
  {
    swt::BenchConfig oc = bc(16, 50, 10, 128, 64);
    oc.seed = 22;
    const swt::LatticeDims dims{oc.max_frames, oc.max_labels + 1, oc.joint_dim,
                                oc.acoustic_dim, oc.label_dim, oc.vocab};
    const std::int64_t ceiling =
        oc.batch_size * swt::lattice_trio_bytes(dims, swt::Precision::f32) / 2;
    auto in = swt::synth_inputs<float>(oc);
    b2::Batch b{to_b2(in.batch.acoustic), to_b2(in.batch.label), in.batch.labels,
                in.batch.t_len, in.batch.u_len};
    b2::JointParams jp{to_b2(in.jp.w_acoustic), to_b2(in.jp.w_label), to_b2(in.jp.bias)};
    b2::OutputParams op{to_b2(in.op.w_out), to_b2(in.op.bias_out)};
    bool ok = true;
    std::string tensor;
    std::int64_t req = 0;
    {
      b2::Engine eng;
      eng.set_alloc_ceiling(ceiling);
      b2::EngineConfig cfg;
      cfg.mode = b2::EngineMode::batched;
      try {
        eng.run_step(b, jp, op, cfg);
        ok = false;
      } catch (const b2::OutOfMemoryError& e) {
        tensor = e.tensor();
        req = e.request_bytes();
        ok &= !tensor.empty() && req > 0;
      }
    }
    for (b2::EngineMode m : {b2::EngineMode::sample_wise, b2::EngineMode::sample_wise_pr,
                             b2::EngineMode::sample_wise_pr_dp}) {
      b2::Engine eng;
      eng.set_alloc_ceiling(ceiling);
      b2::EngineConfig cfg;
      cfg.mode = m;
      try {
        eng.run_step(b, jp, op, cfg);
      } catch (const std::exception& e) {
        std::printf("{\"oom_case_error\": \"%s\"}\n", e.what());
        ok = false;
      }
    }
    std::printf("{\"oom_simulation\": {\"ceiling\": %lld, \"batched_refused\": \"%s\", "
                "\"request_bytes\": %lld}, \"pass\": %s}\n",
                (long long)ceiling, tensor.c_str(), (long long)req, ok ? "true" : "false");
    fails += ok ? 0 : 1;
  }
  // error taxonomy: the reference's exceptions, raised by the same inputs
  {
    auto in = swt::synth_inputs<float>(bc(2, 8, 3, 16, 32));
    b2::Batch b{to_b2(in.batch.acoustic), to_b2(in.batch.label), in.batch.labels,
                in.batch.t_len, in.batch.u_len};
    b2::JointParams jp{to_b2(in.jp.w_acoustic), to_b2(in.jp.w_label), to_b2(in.jp.bias)};
    b2::OutputParams op{to_b2(in.op.w_out), to_b2(in.op.bias_out)};
    b2::EngineConfig cfg;
    b2::Engine eng;
    fails += expect_throw<b2::InvalidInputError>("label_out_of_range", [&] {
      b2::Batch bb = b;
      bb.labels[0] = 16;
      eng.run_step(bb, jp, op, cfg);
    });
    fails += expect_throw<b2::InvalidInputError>("length_out_of_range", [&] {
      b2::Batch bb = b;
      bb.t_len[0] = 9;
      eng.run_step(bb, jp, op, cfg);
    });
    fails += expect_throw<b2::InvalidInputError>("max_parallel_not_pow2", [&] {
      b2::EngineConfig c2;
      c2.mode = b2::EngineMode::sample_wise_pr_dp;
      c2.max_parallel = 3;
      eng.run_step(b, jp, op, c2);
    });
    fails += expect_throw<b2::InvalidShapeError>("param_shape_mismatch", [&] {
      b2::JointParams j2{b2::Tensor{32, 7}, to_b2(in.jp.w_label), to_b2(in.jp.bias)};
      eng.run_step(b, j2, op, cfg);
    });
    fails += expect_throw<b2::InvalidInputError>("pi_bad_extent",
                                                 [] { b2::compute_parallel_iterations(0, 1, 1, 1); });
    // Eq. 9 and the padding ramp agree with the reference
    bool eq = true;
    for (auto [f, l, v] : {std::tuple{500, 101, 4096}, {232, 47, 4096}, {50, 11, 4096}, {1000, 201, 1024}})
      eq &= b2::compute_parallel_iterations(f, l, v, 1'000'000'000) ==
            swt::compute_parallel_iterations(f, l, v, 1'000'000'000);
    const auto [tl, ul] = b2::padded_lengths(1024, 1000, 200);
    const auto rl = swt::padded_lengths(1024, 1000, 200);
    eq &= tl == rl.t_len && ul == rl.u_len;
    std::printf("{\"helpers_match_reference\": %s}\n", eq ? "true" : "false");
    fails += eq ? 0 : 1;
  }
  std::printf("{\"failures\": %d}\n", fails);
  return fails ? 1 : 0;
}
