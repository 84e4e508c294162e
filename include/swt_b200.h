/* SPDX-License-Identifier: Apache-2.0
 *
 * libswt_b200 — C ABI of the B200-native sample-wise transducer
 * loss-and-gradient engine (arXiv 2211.16270, Algorithm 1 lines 5-12).
 *
 * This header is the drop-in boundary. Each entry point names the reference
 * interface it replaces (paths relative to the reference tree, proj/...):
 *
 *   swtb_step                  <- swt::run_step<T>
 *                                 core/include/swt/engine.hpp:116-118,
 *                                 dispatch core/src/engine.cpp:400-407
 *   swtb_parallel_iterations   <- swt::compute_parallel_iterations
 *                                 core/include/swt/engine.hpp:93-94,
 *                                 core/src/engine.cpp:31-50
 *   swtb_padded_lengths        <- swt::padded_lengths
 *                                 core/include/swt/bench.hpp:67-68,
 *                                 core/src/bench.cpp:48-64
 *   swtb_synth_inputs          <- swt::synth_inputs<float>
 *                                 core/include/swt/bench.hpp:80-81,
 *                                 core/src/bench.cpp:66-115
 *   swtb_transducer_loss       <- swt::transducer_loss_sample<T>
 *                                 core/include/swt/loss.hpp:119-121,
 *                                 core/src/loss.cpp:176-185
 *                                 (f^W on caller-supplied scores)
 *   swtb_last_error            <- the what() of the swt::Error thrown
 *                                 (core/include/swt/errors.hpp:12-66)
 *   swtb_set_alloc_ceiling     <- swt::AllocationTracker::set_ceiling /
 *                                 CeilingGuard (core/include/swt/tensor.hpp:
 *                                 115-140; BenchConfig.alloc_ceiling_bytes,
 *                                 core/include/swt/bench.hpp:31)
 *   swtb_last_oom              <- OutOfMemoryError::tensor() /
 *                                 request_bytes() (errors.hpp:37-53)
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *   - Every call returns an swtb_status; nothing throws across the ABI.
 *     Status codes map one-to-one onto the reference exception types
 *     (swt::InvalidShapeError, InvalidInputError, NumericalDegeneracyError,
 *     OutOfMemoryError); the C++ header swt_b200.hpp rethrows them.
 *   - Layouts are the reference's: row-major, lattice cell (t,u) at
 *     t*(U+1)+u, blank id 0, labels int32 [B, U] zero-padded, lengths int64.
 *   - Buffers may be host or device memory (swtb_batch.location /
 *     swtb_out.location). There is no CPU compute path: without a usable
 *     sm_100 GPU, swtb_ctx_create fails with SWTB_ERR_CUDA.
 */
#ifndef SWT_B200_H_
#define SWT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWTB_ABI_VERSION 3

typedef enum {
  SWTB_OK = 0,
  SWTB_ERR_SHAPE = 1,     /* swt::InvalidShapeError */
  SWTB_ERR_INPUT = 2,     /* swt::InvalidInputError */
  SWTB_ERR_NUMERIC = 3,   /* swt::NumericalDegeneracyError */
  SWTB_ERR_OOM = 4,       /* swt::OutOfMemoryError */
  SWTB_ERR_CUDA = 5,      /* CUDA runtime / no sm_100 device */
  SWTB_ERR_NCCL = 6,      /* NCCL failure (multi-GPU) */
  SWTB_ERR_INTERNAL = 7
} swtb_status;

/* Engine modes, numbered like swt::EngineMode (engine.hpp:16-21); all four
 * give the same losses and gradients (engine.hpp:108-112), with the
 * reference's memory behaviour:
 *   BATCHED            run_batched (engine.cpp:245-323): the whole shard at
 *                      the padded extents (T, U+1) in one pass, every
 *                      intermediate materialized in HBM -- joint [cells, H],
 *                      scores [cells, V] fp32, log_den / alpha / beta,
 *                      dscores [cells, V] -- stage by stage. Device memory
 *                      grows with B (the paper's baseline).
 *   SAMPLE_WISE        padded extents, streamed in launch groups: memory
 *                      bounded by the group, not by B.
 *   SAMPLE_WISE_PR(_DP) true (T_b, U_b+1) extents (padding removal), groups
 *                      of many samples per launch (dynamic parallelism);
 *                      _DP checks max_parallel exactly like engine.cpp:336-339.
 * Under an allocation ceiling (swtb_set_alloc_ceiling) the sample-wise
 * modes shrink their groups, down to one sample, until the workspace fits. */
typedef enum {
  SWTB_MODE_BATCHED = 0,
  SWTB_MODE_SAMPLE_WISE = 1,
  SWTB_MODE_SAMPLE_WISE_PR = 2,
  SWTB_MODE_SAMPLE_WISE_PR_DP = 3
} swtb_mode;

/* Arithmetic of the output-layer GEMMs (f^O forward, logit recompute, dz,
 * dW_O); every accumulator is f32 in TMEM.
 *   BF16   operands rounded to bf16 (fastest; bf16 parity bound)
 *   TF32   operands rounded to tf32, and W_O carried as a tf32 (hi, lo) pair
 *          in the GEMMs that read it (f32-grade weights; fp32/TF32 bound)
 *   BF16X  bf16 operands with W_O as a bf16 (hi, lo) pair: removes the
 *          systematic part of the bf16 error at 2 MMAs per weight k-step
 *   FP16   fp16 operands (11-bit significand, the tf32 grade, at the bf16
 *          MMA rate); W_O as an fp16 (hi, lo) pair in the f^O forward only,
 *          whose logits feed the lattice (their rounding error is the one
 *          every cell shares). fp32/TF32 bound. z = tanh(...) and dh lie in
 *          [-1, 1]; W_O entries are assumed within fp16 range (|w| < 65504;
 *          entries below 2^-14 lose relative precision, not the bound)
 * Joint-network GEMMs always use split-bf16 (hi, lo) operands (f32-grade);
 * the lattice recursion accumulates in f64 with f32 transcendentals. */
typedef enum {
  SWTB_PREC_BF16 = 0,
  SWTB_PREC_TF32 = 1,
  SWTB_PREC_BF16X = 2,
  SWTB_PREC_FP16 = 3
} swtb_precision;

typedef enum { SWTB_HOST = 0, SWTB_DEVICE = 1 } swtb_location;

typedef struct swtb_ctx swtb_ctx;

typedef struct {
  int device;             /* CUDA ordinal this context drives */
  int rank;               /* this process's rank among nranks */
  int nranks;             /* >1: samples b with b % nranks == rank are
                             processed here; theta-grads and sample losses
                             are summed across ranks with one NCCL
                             all-reduce */
  const void* nccl_id;    /* 128-byte ncclUniqueId for nranks > 1; NULL =
                             shard-only: no collective, the outputs hold this
                             rank's partial sums (the caller reduces). With
                             nranks = 1 an id makes a single-rank
                             communicator: the all-reduce path runs on one
                             GPU (tests) */
  int precision;          /* swtb_precision */
  int64_t group_cells;    /* lattice cells packed per launch group
                             (0 = default); bounds the workspace */
} swtb_opts;

/* Mirrors swt::Batch<float> (engine.hpp:28-46). */
typedef struct {
  int64_t B, T, U, H_A, H_L; /* U = max labels; label rows = U + 1 */
  const float* acoustic;     /* [B, T, H_A], zero past t_len[b]       */
  const float* label;        /* [B, U+1, H_L], zero past u_len[b]+1   */
  const int32_t* labels;     /* [B, U], zero past u_len[b]            */
  const int64_t* t_len;      /* [B], 1 <= t_len[b] <= T (host memory)  */
  const int64_t* u_len;      /* [B], 0 <= u_len[b] <= U (host memory)  */
  int location;              /* swtb_location of acoustic/label/labels.
                                SWTB_HOST: page-locked (pinned/registered)
                                buffers are copied by async DMA on a copy
                                stream; pageable ones (a plain std::vector)
                                through pinned staging rings filled and
                                drained by the library's worker threads —
                                either way overlapped with the compute */
  int shard_local;           /* 0: per-sample tensors (acoustic, label,
                                labels here; dacoustic, dlabel in swtb_out)
                                hold all B samples, index b. 1: they hold only
                                the samples this rank owns (b % nranks ==
                                rank), in ascending b: slot (b - rank) /
                                nranks — a rank stages 1/nranks of the batch.
                                t_len / u_len always cover all B samples. */
  const float* sample_weights; /* [B] per-sample loss weights w_b >= 0 (host
                                memory), or NULL (all 1). The gradients are
                                those of sum_b w_b L_b (dh^A / dh^L slots and
                                theta-grads); loss and sample_losses stay the
                                unweighted L_b. For the encoder hand-off with
                                per-sample upstream gradients (Algorithm 1
                                lines 13-14); not part of swt::Batch. */
} swtb_batch;

/* Mirrors swt::JointParams / OutputParams (compute.hpp:13-32). */
typedef struct {
  int64_t H, V;
  const float* w_acoustic; /* [H, H_A] */
  const float* w_label;    /* [H, H_L] */
  const float* bias;       /* [H]      */
  const float* w_out;      /* [V, H]   */
  const float* bias_out;   /* [V]      */
  int location;
} swtb_params;

/* Mirrors swt::EngineConfig (engine.hpp:74-82). */
typedef struct {
  int mode; /* swtb_mode */
  int64_t mem_budget_bytes;
  int max_parallel;
  int worker_count;
  int literal_pi_extents;
} swtb_cfg;

/* Mirrors swt::StepResult<float> / GradientSet<float> (engine.hpp:49-58,
 * 84-89). Outputs are overwritten (not accumulated). Under nranks > 1 every
 * rank receives the summed theta-grads, all B sample losses and the total
 * loss; dacoustic/dlabel slots are written only for the samples this rank
 * owns (b % nranks == rank; padding rows zero). With host buffers the other
 * samples' slots are left untouched; with device buffers they are zero. */
typedef struct {
  float* loss;          /* [1]: sum of sample losses, ascending b */
  float* sample_losses; /* [B] */
  float* dw_acoustic;   /* [H, H_A] */
  float* dw_label;      /* [H, H_L] */
  float* dbias;         /* [H] */
  float* dw_out;        /* [V, H] */
  float* dbias_out;     /* [V] */
  float* dacoustic;     /* [B, T, H_A], zero in padded frames */
  float* dlabel;        /* [B, U+1, H_L], zero in padded rows */
  int location;
} swtb_out;

/* Timing/introspection of the last swtb_step on this context. */
typedef struct {
  int64_t groups;          /* launch groups (packed sample sets) */
  int64_t cells;           /* valid lattice cells processed here */
  int64_t tiles;           /* 128-cell tiles (16 t x 8 u) launched */
  int64_t kernel_launches; /* CUDA kernels this step launched */
  int parallel_iterations; /* Eq. 9 PI the reference would use */
  int64_t peak_bytes;      /* device high-water mark of this step */
  int64_t h2d_bytes;       /* host->device bytes copied by this step */
  int64_t d2h_bytes;       /* device->host bytes copied by this step */
  int64_t logits_stored;   /* 1: dh from the forward's stored fp16 logits
                              (x slab); 0: logit-recompute GEMM */
  int64_t active_tiles;    /* fp16: tiles the backward GEMMs walked (their dh
                              is not all zero); -1: every tile (dense) */
} swtb_stats;

int swtb_abi_version(void);

swtb_status swtb_ctx_create(const swtb_opts* opts, swtb_ctx** out);
void swtb_ctx_destroy(swtb_ctx* ctx);

/* Error text of the last failing call on ctx (or of the last failing
 * context-free call when ctx is NULL). Never NULL. */
const char* swtb_last_error(const swtb_ctx* ctx);

/* The CUDA stream (cudaStream_t) every kernel of ctx is launched on. */
void* swtb_stream(swtb_ctx* ctx);

/* Stream-ordering contract. swtb_step is host-synchronous: when it returns,
 * every output is written and none of its kernels is in flight, so callers
 * may read or reuse the outputs on any stream. Device inputs must be
 * complete when the step starts: inputs written by asynchronous work on a
 * caller stream are ordered by passing that stream (cudaStream_t; NULL is
 * the legacy default stream) with enable = 1 — every later step of ctx
 * first makes its own (non-blocking) stream wait for the caller stream's
 * work enqueued so far (an event, no host sync). enable = 0 clears it;
 * without it the caller must synchronize before the call. */
swtb_status swtb_set_caller_stream(swtb_ctx* ctx, void* stream, int enable);

swtb_status swtb_step(swtb_ctx* ctx, const swtb_batch* batch,
                      const swtb_params* params, const swtb_cfg* cfg,
                      swtb_out* out);

swtb_status swtb_get_stats(const swtb_ctx* ctx, swtb_stats* stats);

/* Device memory high-water mark since the last reset (cudaMemPool
 * UsedMemHigh of the context's pool plus its fixed workspace). */
int64_t swtb_peak_bytes(const swtb_ctx* ctx);
void swtb_reset_peak(swtb_ctx* ctx);

/* Bitwise-reproducible steps (default on; the reference's acceptance
 * criterion 10): split-K partial sums of the theta-grads are reduced in a
 * fixed order instead of by fp32 atomics. Off: atomics (about 1 % faster,
 * results vary in the last bits between runs). SWTB_DETERMINISTIC=0 in the
 * environment sets the default off. */
void swtb_set_deterministic(swtb_ctx* ctx, int on);

/* Simulated device-memory ceiling in bytes for this context's allocations
 * (0 = off, the default): an allocation that would push the live bytes past
 * it fails the step with SWTB_ERR_OOM, naming the tensor. */
void swtb_set_alloc_ceiling(swtb_ctx* ctx, int64_t bytes);
/* The tensor name (NUL-terminated, truncated to tensor_cap bytes) and
 * request size of the last allocation refused on ctx; SWTB_ERR_INPUT if
 * none was refused. */
swtb_status swtb_last_oom(const swtb_ctx* ctx, int64_t* request_bytes,
                          char* tensor, int64_t tensor_cap);

/* Live per-stage timing: when enabled, every kernel the engine launches is
 * bracketed by CUDA events on the context stream and its duration is
 * accumulated per stage (read back after each synchronizing swtb_step). */
typedef enum {
  SWTB_STAGE_PREP = 0,      /* parameter conversion, gathers, z slab       */
  SWTB_STAGE_JOINT_FWD = 1, /* P_A / P_L projections (tcgen05 tf32)        */
  SWTB_STAGE_OUT_FWD = 2,   /* f^O forward + log-softmax epilogue          */
  SWTB_STAGE_LATTICE = 3,   /* alpha/beta wavefront                        */
  SWTB_STAGE_OUT_DH = 4,    /* logit recompute + dh epilogue               */
  SWTB_STAGE_OUT_DZ = 5,    /* dz = dh W_O + tanh gate / lattice sums      */
  SWTB_STAGE_OUT_DW = 6,    /* dW_O += dh^T z (split-K)                    */
  SWTB_STAGE_JOINT_BWD = 7, /* ga/gl reduction + joint backward GEMMs      */
  SWTB_STAGE_COMM = 8,      /* NCCL all-reduce                             */
  SWTB_STAGE_WAIT = 9,      /* engine stream waiting on the wavefront      */
  SWTB_STAGE_OTHER = 10,    /* memsets, copies, outputs outside the above  */
  SWTB_NUM_STAGES = 11
} swtb_stage;

void swtb_set_profiling(swtb_ctx* ctx, int enable);
/* ms[SWTB_NUM_STAGES], launches[SWTB_NUM_STAGES] accumulated since the last
 * reset; reset != 0 clears them after reading. */
swtb_status swtb_get_profile(swtb_ctx* ctx, double* ms, int64_t* launches,
                             int reset);

/* ncclGetUniqueId for multi-GPU contexts (128 bytes written to out). */
swtb_status swtb_nccl_unique_id(void* out);

/* f^W alone on caller-supplied scores (host memory, float64 in/out, the
 * reference's transducer_loss_sample<double> signature):
 *   scores [frames, labels+1, vocab], y [labels]
 *   -> *loss = -beta[0,0], dscores [frames, labels+1, vocab]
 * Runs the same GPU kernels as swtb_step: log-sum-exp in f32, the alpha/beta
 * recursion in f64 with f32 log-add-exp corrections. Accuracy is therefore
 * ~1e-6 relative (loss and dscores), not f64's: the reference's f64 unit
 * tests (1e-9..1e-12, test_loss.cpp:84-148) pass at 1e-6. */
swtb_status swtb_transducer_loss(swtb_ctx* ctx, const double* scores,
                                 int64_t frames, int64_t labels,
                                 int64_t vocab, const int32_t* y,
                                 double* loss, double* dscores);

/* Eq. 9: 2^clamp(floor(log2(budget / (4*frames*labels*vocab))), 0, 4).
 * Returns -1 (and sets swtb_last_error(NULL)) when an extent is < 1. */
int swtb_parallel_iterations(int64_t frames, int64_t labels, int64_t vocab,
                             int64_t budget_bytes);

/* Benchmark padding ramp (t_len, u_len out, [batch] each). */
swtb_status swtb_padded_lengths(int64_t batch, int64_t max_frames,
                                int64_t max_labels, int64_t* t_len,
                                int64_t* u_len);

/* Bit-identical to swt::synth_inputs<float> (mt19937_64, seed, draw order,
 * padding ramp, zeroed padding). All outputs are host buffers of the
 * batch/params shapes above. */
typedef struct {
  int64_t B, T, U, H, H_A, H_L, V;
  uint64_t seed;
} swtb_synth_cfg;

swtb_status swtb_synth_inputs(const swtb_synth_cfg* cfg, float* acoustic,
                              float* label, int32_t* labels, int64_t* t_len,
                              int64_t* u_len, float* w_acoustic,
                              float* w_label, float* bias, float* w_out,
                              float* bias_out);

/* ---- testing hook -------------------------------------------------------
 * One tcgen05 GEMM of the engine's core, on caller DEVICE buffers:
 *   out[m, n] (=|+=) sum_k A(m, k) * B(n, k)
 * A is [M, K] row-major (a_mn = 0) or [K, M] (a_mn = 1); B is [N, K]
 * (b_mn = 0) or [K, N] (b_mn = 1); elements bf16 (precision 0) or fp32 read
 * as tf32 (precision 1); lda/ldb in elements. accumulate = 1 adds with
 * split-K atomics. Runs on the context's stream and synchronizes. */
swtb_status swtb_debug_gemm(swtb_ctx* ctx, int precision, int a_mn, int b_mn,
                            const void* A, int64_t lda, const void* B,
                            int64_t ldb, int64_t M, int64_t N, int64_t K,
                            float* out, int64_t ldo, int accumulate);

#ifdef __cplusplus
}
#endif

#endif /* SWT_B200_H_ */
