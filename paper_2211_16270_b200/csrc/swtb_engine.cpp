// SPDX-License-Identifier: Apache-2.0
//
// libswt_b200 host engine: the B200 replacement of swt::run_step /
// run_sample_wise (reference proj/core/src/engine.cpp:325-407) behind the C
// ABI declared in include/swt_b200.h.
//
// One call = one training step over the batch shard this rank owns:
//   1. validate exactly like validate_step_inputs (engine.cpp:72-96) and the
//      label checks of loss.cpp:14-27; DP mode checks max_parallel
//      (engine.cpp:336-339) and records Eq. 9's PI (engine.cpp:31-50);
//   2. pack owned samples (b % nranks == rank, ascending b) into launch
//      groups of <= group_cells lattice cells, each cropped to its true
//      (T_b, U_b+1) extents (padding removal) and tiled into 16x8-cell tiles
//      (dynamic parallelism = many samples per launch);
//   3. per group, on one CUDA stream: gather -> joint projections (tcgen05
//      tf32) -> z slab -> f^O forward + log-softmax epilogue (tcgen05) ->
//      alpha/beta wavefront -> logit recompute + dh epilogue -> dz GEMM +
//      tanh-gate/lattice-sum epilogue -> dW_O split-K GEMM -> ga/gl
//      reduction -> joint backward GEMMs;
//   4. theta-grads and sample losses live in one fp32 buffer that is summed
//      across ranks with a single ncclAllReduce, then copied out.
// All per-sample intermediates live in a grow-only workspace sized by the
// largest group, so device memory is bounded by group_cells, not by B.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <memory>
#include <string>
#include <vector>

#include "../../include/swt_b200.h"
#include "swtb_kernels.h"

namespace {

using namespace swtb;

struct SwtbError : std::runtime_error {
  swtb_status status;
  SwtbError(swtb_status s, const std::string& m)
      : std::runtime_error(m), status(s) {}
};

[[noreturn]] void fail(swtb_status s, const std::string& m) {
  throw SwtbError(s, m);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    fail(SWTB_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  if (e != cudaSuccess)
    fail(SWTB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// NCCL is resolved at run time, only for multi-GPU contexts: an NCCL that
// is already loaded in the process (e.g. torch's) is reused, so libswt_b200
// never drags a second libnccl into a host application.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t,
                             ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h) {
      n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
      n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!n.get_unique_id || !n.comm_init_rank || !n.all_reduce || !n.comm_destroy)
    fail(SWTB_ERR_NCCL, "libnccl.so.2 could not be loaded");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(SWTB_ERR_NCCL, std::string(what) + ": " +
                            (nccl().error_string ? nccl().error_string(r) : "error"));
}

long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

thread_local std::string g_last_error = "";

// Grow-only device buffer with byte accounting.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// Copies between device memory and PAGEABLE host memory (a drop-in caller's
// plain host tensors). cudaMemcpyAsync from/to pageable memory returns only
// after the driver has staged the bytes, so issued from the engine thread it
// would hold back every kernel launch behind 2.5 GB of host copies. Instead
// a worker thread moves the bytes through a ring of pinned slots: H2D =
// memcpy into a slot, async copy out of it; D2H = async copy into a slot,
// memcpy out once it landed. Jobs run in submission order on the worker;
// the engine thread waits only for what its next launch needs.
class PinnedRing {
 public:
  PinnedRing(int device, size_t slot_bytes, int slots) : device_(device) {
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    slots_.resize(size_t(slots));
    for (Slot& sl : slots_) {
      CK(cudaHostAlloc(&sl.ptr, slot_bytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
    }
    slot_bytes_ = slot_bytes;
    worker_ = std::thread([this] { loop(); });
  }
  ~PinnedRing() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    worker_.join();
    for (Slot& sl : slots_) {
      cudaEventDestroy(sl.ev);
      cudaFreeHost(sl.ptr);
    }
    cudaStreamDestroy(stream_);
  }
  cudaStream_t stream() const { return stream_; }
  // queue a job (runs on the worker, in order); returns its sequence number
  long long post(std::function<void(PinnedRing&)> f) {
    std::lock_guard<std::mutex> lk(mu_);
    jobs_.push_back(std::move(f));
    cv_.notify_all();
    return ++posted_;
  }
  // block until job `seq` has run (rethrows a worker failure)
  void wait(long long seq) {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ >= seq || err_; });
    if (err_) {
      std::exception_ptr e = err_;
      err_ = nullptr;
      done_ = posted_;
      jobs_.clear();
      std::rethrow_exception(e);
    }
  }
  void wait_all() { wait(posted_); }
  // --- called from jobs (worker thread) ---
  void h2d(void* dst, const void* src, size_t n) {
    for (size_t o = 0; o < n; o += slot_bytes_) {
      const size_t k = std::min(slot_bytes_, n - o);
      Slot& sl = next_slot();
      std::memcpy(sl.ptr, static_cast<const char*>(src) + o, k);
      CK(cudaMemcpyAsync(static_cast<char*>(dst) + o, sl.ptr, k, cudaMemcpyHostToDevice, stream_));
      CK(cudaEventRecord(sl.ev, stream_));
    }
  }
  void d2h(void* dst, const void* src, size_t n) {
    for (size_t o = 0; o < n; o += slot_bytes_) {
      const size_t k = std::min(slot_bytes_, n - o);
      Slot& sl = next_slot();
      CK(cudaMemcpyAsync(sl.ptr, static_cast<const char*>(src) + o, k, cudaMemcpyDeviceToHost,
                         stream_));
      CK(cudaEventRecord(sl.ev, stream_));
      sl.out = static_cast<char*>(dst) + o;
      sl.out_n = k;
    }
  }
  // finish every pending D2H (memcpy the landed slots out)
  void drain() {
    for (size_t i = 0; i < slots_.size(); ++i) settle(slots_[(cur_ + i) % slots_.size()]);
  }

 private:
  struct Slot {
    void* ptr = nullptr;
    cudaEvent_t ev = nullptr;
    char* out = nullptr;  // pending D2H destination
    size_t out_n = 0;
  };
  void settle(Slot& sl) {
    CK(cudaEventSynchronize(sl.ev));
    if (sl.out) {
      std::memcpy(sl.out, sl.ptr, sl.out_n);
      sl.out = nullptr;
    }
  }
  Slot& next_slot() {  // oldest slot: its last copy has finished (and is drained)
    Slot& sl = slots_[cur_];
    cur_ = (cur_ + 1) % slots_.size();
    settle(sl);
    return sl;
  }
  void loop() {
    cudaSetDevice(device_);
    for (;;) {
      std::function<void(PinnedRing&)> f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (jobs_.empty()) return;  // stop requested, queue drained
        f = std::move(jobs_.front());
        jobs_.pop_front();
      }
      std::exception_ptr e;
      try {
        if (!err_) f(*this);
      } catch (...) {
        e = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (e && !err_) err_ = e;
        ++done_;
      }
      done_cv_.notify_all();
    }
  }
  int device_;
  cudaStream_t stream_ = nullptr;
  std::vector<Slot> slots_;
  size_t slot_bytes_ = 0;
  size_t cur_ = 0;
  std::thread worker_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::function<void(PinnedRing&)>> jobs_;
  long long posted_ = 0, done_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
};

bool is_pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

struct swtb_ctx {
  int device = 0;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  Prec prec = Prec::kBF16;
  bool split_w = false;  // W_O as a (hi, lo) pair in the f^O forward
  bool split_w_bwd = false;  // ... and in the recompute + dz GEMMs
  // fp16: the f^O forward runs on the single fp16 W_O and corrects each
  // label row's logits by zbar_u . W_lo^T (zmean_kernel + a small GEMM
  // folded into a per-row bias): the rounding error every frame of the row
  // would repeat, at 1 MMA per k-step instead of the (hi, lo) pair's 2
  bool fwd_corr = false;
  // SWTB_STORE_X=1 (16-bit operand modes, an alternative pipeline, off by
  // default): the f^O forward also stores the logits as the fp16 x slab
  // (block-relative, see FwdLseArgs) and the backward forms dh from it
  // elementwise, in place (x_to_dh_kernel), instead of recomputing the
  // logits with a second output-layer GEMM. Same-box A/B at c4:
  // the forward's x stores (+15 ms) and the HBM-bound dh pass (~4 B/element,
  // 114-150 ms) cost what the recompute GEMM (~144 ms) saves, for +0.7 GB.
  bool store_x = [] {
    const char* e = std::getenv("SWTB_STORE_X");
    return e && std::atoi(e) == 1;
  }();
  // fp16 mode: the backward (logit recompute, dz, dW_O) walks only the tiles
  // whose dh is not all zero — a tile where every cell's occupancy alpha *
  // beta / P is below 2^-26 has every dh term below fp16's smallest
  // subnormal / 2, so its dh rows round to exactly 0 and contribute nothing.
  // SWTB_SKIP_ZERO_TILES=0: every tile (dense).
  bool skip_zero_tiles = [] {
    const char* e = std::getenv("SWTB_SKIP_ZERO_TILES");
    return !(e && std::atoi(e) == 0);
  }();
  long long group_cells = 1 << 20;
  // the backward of a group runs over sub-slabs of at most this many dh-slab
  // bytes (the dh slab is the largest workspace buffer). 1.6 GB: one
  // sub-slab per part at c4 (fewer, longer backward GEMM launches; A/B
  // 1000 MB -> 1600 MB: -10 ms/step for +0.6 GB)
  long long bwd_slab_bytes = [] {  // SWTB_BWD_SLAB_MB overrides (experiments)
    const char* e = std::getenv("SWTB_BWD_SLAB_MB");
    const long long v = e ? std::atoll(e) : 1600;
    return (v > 0 ? v : 1600) << 20;
  }();
  // bitwise-reproducible theta-grads: split-K partials + ordered reductions
  // instead of fp32 atomics (SWTB_DETERMINISTIC=0 restores the atomics)
  bool deterministic = [] {
    const char* e = std::getenv("SWTB_DETERMINISTIC");
    return !(e && std::atoi(e) == 0);
  }();
  // groups per joint-network batch (SWTB_JOINT_BATCH overrides). 8 since
  // the zero-tile skip and the deferred tail (A/B at c4: 4 groups 423.4 ms,
  // 8 groups 419.1 ms, +0.3 GB)
  int joint_batch = [] {
    const char* e = std::getenv("SWTB_JOINT_BATCH");
    const int v = e ? std::atoi(e) : 8;
    return v < 1 ? 1 : v;
  }();
  cudaStream_t stream = nullptr;
  // the alpha/beta wavefront of one part of a group runs here, overlapped
  // with the GEMMs of the other part on `stream`
  cudaStream_t lat_stream = nullptr;
  // host-buffer steps: per-group H2D of inputs / D2H of dh^A, dh^L slots run
  // here, overlapped with the compute of other groups
  cudaStream_t cp_stream = nullptr;
  // swtb_set_caller_stream: each step's stream first waits for this one
  cudaStream_t caller = nullptr;  // may be the legacy default stream (0)
  bool has_caller = false;
  cudaEvent_t ev_caller = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done;
  // the step plan depends only on lengths and shapes: reused (with its
  // device descriptor blob) while they repeat
  std::shared_ptr<void> plan_cache;
  std::vector<int64_t> plan_key;
  const void* plan_blob_dev = nullptr;
  void events(std::vector<cudaEvent_t>& v, size_t n) {
    while (v.size() < n) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      v.push_back(e);
    }
  }
  static constexpr int kMaxParts = 4;  // parts a launch group is cut into
  cudaEvent_t ev_fwd[kMaxParts] = {}, ev_lat[kMaxParts] = {};
  std::string last_error;
  swtb_stats stats{};
  long long live_bytes = 0, peak_bytes = 0;

  // named workspace buffers
  std::vector<DevBuf*> all;
  DevBuf in_acoustic, in_label, in_labels;  // device copies of host inputs
  DevBuf p_wa, p_wl, p_bz, p_wo, p_bo;      // parameter operands
  DevBuf theta, bad;                        // accumulators
  DevBuf out_dacoustic, out_dlabel;         // device outputs (host-out path)
  DevBuf desc;                              // group descriptors
  DevBuf ha, hl, pa, pl, ga, gl, zs, dhs, parta, partl;
  DevBuf xoff;         // x slab: per-32-column block maxima of the logits
  DevBuf tflags, tlist;  // zero-tile skip: per-tile active flags, per-part active lists
  DevBuf lmp;            // ... and log2 of each cell's largest softmax probability
  DevBuf zbar, cbias;  // fp16 forward correction: per-label-row mean z, bias rows
  DevBuf weights;      // per-sample loss weights
  const void* cbias_zeroed = nullptr;  // cbias allocation whose pad columns are zero
  size_t cbias_zeroed_bytes = 0;
  DevBuf lse, lpb, lpy, alpha, beta, logz, eb, ey;
  DevBuf scores;  // batched comparator: materialized fp32 logits
  DevBuf split_ws;  // deterministic split-K partials
  DevBuf dw_acc;    // deterministic dW_O / db_O accumulator slices
  // f^W op
  DevBuf op_scores, op_y, op_dscores, op_sd;
  // pageable host buffers: pinned staging rings with their worker threads
  // (created on first use; inputs and outputs on separate rings / streams)
  std::unique_ptr<PinnedRing> ring_in, ring_out;
  PinnedRing& ring(std::unique_ptr<PinnedRing>& r) {
    if (!r) r = std::make_unique<PinnedRing>(device, size_t(32) << 20, 6);
    return *r;
  }
  // live per-stage timing
  bool prof = false;
  double prof_ms[SWTB_NUM_STAGES] = {0};
  int64_t prof_n[SWTB_NUM_STAGES] = {0};
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  size_t ev_next = 0;
  int cur_stage = -1;
  cudaEvent_t cur_start = nullptr;

  cudaEvent_t take_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  // Mark the start of a stage (closing the previous one).
  void stage(int st_id, int launches = 1) {
    if (!prof) return;
    if (cur_stage >= 0) end_stage();
    cur_stage = st_id;
    cur_start = take_event();
    CK(cudaEventRecord(cur_start, stream));
    prof_n[st_id] += launches;
  }
  void end_stage() {
    if (!prof || cur_stage < 0) return;
    cudaEvent_t e = take_event();
    CK(cudaEventRecord(e, stream));
    ev_used.push_back({cur_stage, {cur_start, e}});
    cur_stage = -1;
  }
  // Time one launch on another stream (outside the stage sequence).
  void side_begin(cudaStream_t s, cudaEvent_t* e0) {
    if (!prof) return;
    *e0 = take_event();
    CK(cudaEventRecord(*e0, s));
  }
  void side_end(int st_id, cudaStream_t s, cudaEvent_t e0) {
    if (!prof) return;
    cudaEvent_t e1 = take_event();
    CK(cudaEventRecord(e1, s));
    ev_used.push_back({st_id, {e0, e1}});
    prof_n[st_id] += 1;
  }
  // After a stream sync: fold elapsed times into the per-stage totals.
  void collect() {
    if (!prof) return;
    end_stage();
    // the closing event was recorded after the step's stream sync: wait for
    // it (on a shared GPU the record itself can lag)
    CK(cudaStreamSynchronize(stream));
    for (auto& u : ev_used) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, u.second.first, u.second.second));
      prof_ms[u.first] += ms;
    }
    ev_used.clear();
    ev_next = 0;
  }

  swtb_ctx() {
    all = {&in_acoustic, &in_label, &in_labels, &p_wa,    &p_wl,  &p_bz,
           &p_wo,        &p_bo,     &theta,     &bad,     &out_dacoustic,
           &out_dlabel,  &desc,     &ha,        &hl,      &pa,    &pl,
           &ga,          &gl,       &zs,        &dhs,     &parta, &partl,
           &lse,         &lpb,      &lpy,       &alpha,   &beta,  &logz, &eb, &ey,
           &op_scores,   &op_y,     &op_dscores, &op_sd, &scores, &split_ws, &dw_acc,
           &zbar,        &cbias,    &weights,  &xoff,   &tflags, &tlist, &lmp};
  }

  // Simulated allocation ceiling (reference AllocationTracker::on_alloc,
  // tensor.cpp:12-25): 0 = off. The last refusal is kept for swtb_last_oom.
  long long alloc_ceiling = 0;
  std::string oom_tensor;
  long long oom_bytes = 0;

  void* need(DevBuf& b, size_t bytes, const char* tag = "workspace") {
    bytes = std::max<size_t>(round_up(std::max<size_t>(bytes, 16), 256), 256);
    if (b.bytes >= bytes) return b.ptr;
    const long long live_after = live_bytes - (long long)b.bytes;
    if (alloc_ceiling > 0 && live_after + (long long)bytes > alloc_ceiling) {
      oom_tensor = tag;
      oom_bytes = (long long)bytes;
      fail(SWTB_ERR_OOM, "allocation of tensor '" + std::string(tag) + "' (" +
                             std::to_string(bytes) + " bytes) exceeds ceiling " +
                             std::to_string(alloc_ceiling) + " with " +
                             std::to_string(live_after) + " bytes live");
    }
    if (b.ptr) {
      CK(cudaStreamSynchronize(stream));
      CK(cudaFree(b.ptr));
      live_bytes -= b.bytes;
      b.ptr = nullptr;
      b.bytes = 0;
    }
    cudaError_t e = cudaMalloc(&b.ptr, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      b.ptr = nullptr;
      oom_tensor = tag;
      oom_bytes = (long long)bytes;
      fail(SWTB_ERR_OOM, "device allocation of tensor '" + std::string(tag) + "' (" +
                             std::to_string(bytes) + " bytes) failed: " +
                             cudaGetErrorString(e));
    }
    b.bytes = bytes;
    live_bytes += bytes;
    peak_bytes = std::max(peak_bytes, live_bytes);
    return b.ptr;
  }
  // Release a buffer (the batched comparator's materialized tensors are not
  // kept across steps).
  void drop(DevBuf& b) noexcept {
    if (!b.ptr) return;
    cudaStreamSynchronize(stream);
    cudaFree(b.ptr);
    live_bytes -= b.bytes;
    b.ptr = nullptr;
    b.bytes = 0;
  }

  ~swtb_ctx() {
    ring_in.reset();
    ring_out.reset();
    if (stream) cudaStreamSynchronize(stream);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (DevBuf* b : all)
      if (b->ptr) cudaFree(b->ptr);
    if (comm) nccl().comm_destroy(comm);
    for (int i = 0; i < kMaxParts; ++i) {
      if (ev_fwd[i]) cudaEventDestroy(ev_fwd[i]);
      if (ev_lat[i]) cudaEventDestroy(ev_lat[i]);
    }
    for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_done) cudaEventDestroy(e);
    if (ev_caller) cudaEventDestroy(ev_caller);
    if (cp_stream) cudaStreamDestroy(cp_stream);
    if (lat_stream) cudaStreamDestroy(lat_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// ---------------------------------------------------------------------------
// Reference-equivalent helpers (no GPU needed)

// Eq. 9 — reference proj/core/src/engine.cpp:31-50.
int parallel_iterations(long long frames, long long labels, long long vocab,
                        long long budget) {
  if (frames < 1 || labels < 1 || vocab < 1)
    fail(SWTB_ERR_INPUT, "parallel-iteration extents must be >= 1");
  const unsigned __int128 base = (unsigned __int128)4 * frames * labels * vocab;
  if (budget <= 0 || base > (unsigned __int128)budget) return 1;
  int e = 0;
  unsigned __int128 cur = base;
  while (e < 4 && cur * 2 <= (unsigned __int128)budget) {
    cur *= 2;
    ++e;
  }
  return 1 << e;
}

// Benchmark padding ramp — reference proj/core/src/bench.cpp:48-64.
void padded_lengths(long long B, long long T, long long U, int64_t* t_len,
                    int64_t* u_len) {
  for (long long b = 0; b < B; ++b) {
    const double ramp = B == 1 ? 0.0 : double(b) / double(B - 1);
    t_len[b] = std::max<long long>(1, std::llround(double(T) * (1.0 - 0.093 * ramp)));
    u_len[b] = std::max<long long>(1, std::llround(double(U) * (1.0 - 0.458 * ramp)));
  }
}

// ---------------------------------------------------------------------------
// Step planning

struct Group {
  std::vector<SampleDesc> samples;
  std::vector<TileDesc> tiles;
  std::vector<long long> a_src, l_src;  // source rows for packed rows
  std::vector<long long> a_dst, l_dst;  // dh^A / dh^L output rows
  std::vector<int> l_info;              // per label row: (sample's first P_A row, T_b)
  std::vector<int> a_sample, l_sample;
  long long R_A = 0, R_L = 0, lat = 0, cells = 0;
  long long ra0 = 0, rl0 = 0;  // first row of this group in its joint batch
  int jb = 0;                  // joint batch
  int max_U1 = 1;
  // offsets into the descriptor upload (bytes)
  size_t off_samples, off_tiles, off_asrc, off_lsrc, off_asmp, off_lsmp;
};

// Consecutive groups whose joint-network GEMMs (projections forward, dh^A /
// dh^L / dW_A / dW_L backward) run as one batch: a few big GEMMs instead of
// many small ones per group.
struct JBatch {
  int g0 = 0, g1 = 0;  // groups [g0, g1)
  long long R_A = 0, R_L = 0;
  std::vector<long long> a_src, l_src, a_dst, l_dst;
  std::vector<int> l_info;
  size_t off_asrc = 0, off_lsrc = 0, off_adst = 0, off_ldst = 0, off_linfo = 0;
};

// Where sample b lives in a per-sample tensor: its batch index b (full
// layout), or its rank-local slot (b - rank) / nranks (the shard-local
// layout: only this rank's samples, in ascending b).
struct SlotMap {
  int rank = 0, nranks = 1;
  bool local = false;
  long long operator()(long long b) const { return local ? (b - rank) / nranks : b; }
};
// samples rank `rank` owns of a batch of B (b % nranks == rank)
inline long long owned_samples(long long B, int rank, int nranks) {
  return rank < B ? (B - rank + nranks - 1) / nranks : 0;
}

struct Plan {
  std::vector<Group> groups;
  std::vector<JBatch> batches;
  long long max_R_A = 0, max_R_L = 0, max_tiles = 0, max_lat = 0,
            max_samples = 0;
  long long cells = 0, tiles = 0;
  std::vector<char> blob;
};

// pad: tile every sample over the batch's padded extents (T, U+1) instead of
// its true (T_b, U_b+1) -- the reference's modes without padding removal
// (engine.cpp:182-198, 245-323); only the true sub-lattice is valid.
// in_slot / out_slot / lab_slot: where a sample's input rows, dh^A / dh^L
// output rows and labels live (full batch layout or rank-local slots).
Plan make_plan(const swtb_batch& bt, int rank, int nranks, long long budget,
               int joint_batch, bool pad, SlotMap in_slot, SlotMap out_slot,
               SlotMap lab_slot) {
  Plan p;
  const long long U1max = bt.U + 1;
  const long long slack = lat_slack(int(U1max));
  Group g;
  g.lat = slack;
  JBatch jb;
  auto close_batch = [&] {
    if (jb.g1 == jb.g0) return;
    p.max_R_A = std::max(p.max_R_A, jb.R_A);
    p.max_R_L = std::max(p.max_R_L, jb.R_L);
    p.batches.push_back(std::move(jb));
    jb = JBatch();
    jb.g0 = jb.g1 = int(p.groups.size());
  };
  auto flush = [&] {
    if (g.samples.empty()) return;
    g.lat += slack;
    g.jb = int(p.batches.size());
    jb.a_src.insert(jb.a_src.end(), g.a_src.begin(), g.a_src.end());
    jb.l_src.insert(jb.l_src.end(), g.l_src.begin(), g.l_src.end());
    jb.a_dst.insert(jb.a_dst.end(), g.a_dst.begin(), g.a_dst.end());
    jb.l_dst.insert(jb.l_dst.end(), g.l_dst.begin(), g.l_dst.end());
    jb.l_info.insert(jb.l_info.end(), g.l_info.begin(), g.l_info.end());
    jb.R_A += g.R_A;
    jb.R_L += g.R_L;
    ++jb.g1;
    p.max_tiles = std::max<long long>(p.max_tiles, (long long)g.tiles.size());
    p.max_lat = std::max(p.max_lat, g.lat);
    p.max_samples = std::max<long long>(p.max_samples, (long long)g.samples.size());
    p.groups.push_back(std::move(g));
    if (jb.g1 - jb.g0 >= joint_batch) close_batch();
    g = Group();
    g.lat = slack;
    g.ra0 = jb.R_A;
    g.rl0 = jb.R_L;
  };
  for (long long b = rank; b < bt.B; b += nranks) {
    const int T = int(bt.t_len[b]);
    const int U1 = int(bt.u_len[b]) + 1;
    const int Tt = pad ? int(bt.T) : T, Ut = pad ? int(U1max) : U1;
    const long long cells = (long long)Tt * Ut;  // cells the GEMMs process
    if (!g.samples.empty() && g.cells + cells > budget) flush();
    SampleDesc sd{};
    sd.T = T;
    sd.U1 = U1;
    sd.a_row0 = int(g.ra0 + g.R_A);  // rows of the joint batch's buffers
    sd.l_row0 = int(g.rl0 + g.R_L);
    sd.lat = g.lat;
    sd.lab = lab_slot(b) * bt.U;
    sd.b = int(b);
    sd.tile0 = int(g.tiles.size());
    sd.n_tb = (Tt + kTileT - 1) / kTileT;
    sd.n_ub = (Ut + kTileU - 1) / kTileU;
    const int s = int(g.samples.size());
    for (int tb = 0; tb < sd.n_tb; ++tb)
      for (int ub = 0; ub < sd.n_ub; ++ub)
        g.tiles.push_back(TileDesc{s, tb * kTileT, ub * kTileU, 0});
    for (int t = 0; t < T; ++t) {
      g.a_src.push_back(in_slot(b) * bt.T + t);
      g.a_dst.push_back(out_slot(b) * bt.T + t);
      g.a_sample.push_back(s);
    }
    for (int u = 0; u < U1; ++u) {
      g.l_src.push_back(in_slot(b) * U1max + u);
      g.l_dst.push_back(out_slot(b) * U1max + u);
      g.l_info.push_back(sd.a_row0);
      g.l_info.push_back(T);
      g.l_sample.push_back(s);
    }
    g.R_A += T;
    g.R_L += U1;
    g.lat += skew_size(T, U1);
    g.cells += cells;
    g.max_U1 = std::max(g.max_U1, U1);
    g.samples.push_back(sd);
    p.cells += (long long)T * U1;
    p.tiles += (long long)sd.n_tb * sd.n_ub;
  }
  flush();
  close_batch();
  // one descriptor blob for the whole step (single H2D copy)
  size_t off = 0;
  auto put = [&](size_t bytes) {
    const size_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  };
  for (Group& gr : p.groups) {
    gr.off_samples = put(gr.samples.size() * sizeof(SampleDesc));
    gr.off_tiles = put(gr.tiles.size() * sizeof(TileDesc));
    gr.off_asrc = put(gr.a_src.size() * sizeof(long long));
    gr.off_lsrc = put(gr.l_src.size() * sizeof(long long));
    gr.off_asmp = put(gr.a_sample.size() * sizeof(int));
    gr.off_lsmp = put(gr.l_sample.size() * sizeof(int));
  }
  for (JBatch& b : p.batches) {
    b.off_asrc = put(b.a_src.size() * sizeof(long long));
    b.off_lsrc = put(b.l_src.size() * sizeof(long long));
    b.off_adst = put(b.a_dst.size() * sizeof(long long));
    b.off_ldst = put(b.l_dst.size() * sizeof(long long));
    b.off_linfo = put(b.l_info.size() * sizeof(int));
  }
  p.blob.assign(std::max<size_t>(off, 256), 0);
  for (Group& gr : p.groups) {
    std::memcpy(p.blob.data() + gr.off_samples, gr.samples.data(),
                gr.samples.size() * sizeof(SampleDesc));
    std::memcpy(p.blob.data() + gr.off_tiles, gr.tiles.data(),
                gr.tiles.size() * sizeof(TileDesc));
    std::memcpy(p.blob.data() + gr.off_asrc, gr.a_src.data(),
                gr.a_src.size() * sizeof(long long));
    std::memcpy(p.blob.data() + gr.off_lsrc, gr.l_src.data(),
                gr.l_src.size() * sizeof(long long));
    std::memcpy(p.blob.data() + gr.off_asmp, gr.a_sample.data(),
                gr.a_sample.size() * sizeof(int));
    std::memcpy(p.blob.data() + gr.off_lsmp, gr.l_sample.data(),
                gr.l_sample.size() * sizeof(int));
  }
  for (JBatch& b : p.batches) {
    std::memcpy(p.blob.data() + b.off_asrc, b.a_src.data(), b.a_src.size() * sizeof(long long));
    std::memcpy(p.blob.data() + b.off_lsrc, b.l_src.data(), b.l_src.size() * sizeof(long long));
    std::memcpy(p.blob.data() + b.off_adst, b.a_dst.data(), b.a_dst.size() * sizeof(long long));
    std::memcpy(p.blob.data() + b.off_ldst, b.l_dst.data(), b.l_dst.size() * sizeof(long long));
    std::memcpy(p.blob.data() + b.off_linfo, b.l_info.data(), b.l_info.size() * sizeof(int));
  }
  return p;
}

void validate(const swtb_batch& bt, const swtb_params& pr, const swtb_cfg& cfg,
              std::vector<int32_t>& host_labels, cudaStream_t st, int rank,
              int nranks) {
  if (bt.B < 1 || bt.T < 1 || bt.U < 0 || bt.H_A < 1 || bt.H_L < 1)
    fail(SWTB_ERR_SHAPE, "batch encoding tensors are inconsistent");
  if (pr.H < 1 || pr.V < 1)
    fail(SWTB_ERR_SHAPE, "parameter extents do not match the batch");
  if (!bt.acoustic || !bt.label || !bt.t_len || !bt.u_len ||
      (bt.U > 0 && !bt.labels))
    fail(SWTB_ERR_SHAPE, "batch length/label arrays are inconsistent");
  if (!pr.w_acoustic || !pr.w_label || !pr.bias || !pr.w_out || !pr.bias_out)
    fail(SWTB_ERR_SHAPE, "parameter tensors missing");
  for (long long i = 0; i < bt.B; ++i) {
    if (bt.t_len[i] < 1 || bt.t_len[i] > bt.T || bt.u_len[i] < 0 ||
        bt.u_len[i] > bt.U)
      fail(SWTB_ERR_INPUT, "sample lengths outside the padded extents");
  }
  if (cfg.mode < SWTB_MODE_BATCHED || cfg.mode > SWTB_MODE_SAMPLE_WISE_PR_DP)
    fail(SWTB_ERR_INPUT, "unknown engine mode");
  if (cfg.mode == SWTB_MODE_SAMPLE_WISE_PR_DP) {
    if (cfg.max_parallel < 1 || cfg.max_parallel > 16 ||
        !std::has_single_bit(unsigned(cfg.max_parallel)))
      fail(SWTB_ERR_INPUT, "max_parallel must be a power of two in 1..16");
  }
  if (bt.shard_local != 0 && bt.shard_local != 1)
    fail(SWTB_ERR_INPUT, "shard_local must be 0 or 1");
  if (bt.sample_weights)
    for (long long b = 0; b < bt.B; ++b)
      if (!(std::isfinite(bt.sample_weights[b]) && bt.sample_weights[b] >= 0.f))
        fail(SWTB_ERR_INPUT, "sample weights must be finite and >= 0");
  // labels in [1, V) for every emitted position (reference loss.cpp:14-27);
  // shard-local batches hold (and are checked for) this rank's samples only
  const SlotMap lab{rank, nranks, bt.shard_local != 0};
  const long long lab_rows = lab.local ? owned_samples(bt.B, rank, nranks) : bt.B;
  if (bt.U > 0 && lab_rows > 0) {
    host_labels.resize(size_t(lab_rows * bt.U));
    if (bt.location == SWTB_DEVICE) {
      // on the engine stream, which already waits for the caller's stream
      CK(cudaMemcpyAsync(host_labels.data(), bt.labels,
                         host_labels.size() * sizeof(int32_t),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    else
      std::memcpy(host_labels.data(), bt.labels,
                  host_labels.size() * sizeof(int32_t));
    for (long long b = lab.local ? rank : 0; b < bt.B; b += lab.local ? nranks : 1)
      for (long long u = 0; u < bt.u_len[b]; ++u) {
        const int32_t l = host_labels[size_t(lab(b) * bt.U + u)];
        if (l <= 0 || l >= pr.V)
          fail(SWTB_ERR_INPUT, "label id " + std::to_string(l) +
                                   " outside [1, " + std::to_string(pr.V) +
                                   ")");
      }
  }
}

// ---------------------------------------------------------------------------

void run_step(swtb_ctx* c, const swtb_batch& bt, const swtb_params& pr,
              const swtb_cfg& cfg, swtb_out& out) {
  std::vector<int32_t> host_labels;
  CK(cudaSetDevice(c->device));
  if (c->has_caller) {  // inputs may still be in flight on the caller's stream
    CK(cudaEventRecord(c->ev_caller, c->caller));
    CK(cudaStreamWaitEvent(c->stream, c->ev_caller, 0));
  }
  validate(bt, pr, cfg, host_labels, c->stream, c->rank, c->nranks);
  set_gemm_sm_reserve(0);
  cudaStream_t st = c->stream;
  const long long B = bt.B, T = bt.T, U = bt.U, U1max = U + 1;
  const long long H_A = bt.H_A, H_L = bt.H_L, H = pr.H, V = pr.V;
  const bool tf32 = c->prec == Prec::kTF32;
  const int esz = tf32 ? 4 : 2;
  const long long H_pad = round_up(H, 32), V_pad = round_up(V, 32);
  const long long HA_pad = round_up(H_A, 32), HL_pad = round_up(H_L, 32);

  swtb_stats stats{};
  {
    long long mf = 1, ml = 0;
    for (long long b = 0; b < B; ++b) {
      mf = std::max<long long>(mf, bt.t_len[b]);
      ml = std::max<long long>(ml, bt.u_len[b]);
    }
    const long long lab_ext = cfg.literal_pi_extents ? std::max<long long>(ml, 1) : ml + 1;
    int pi = parallel_iterations(mf, lab_ext, V, cfg.mem_budget_bytes > 0 ? cfg.mem_budget_bytes : 1000000000LL);
    if (cfg.mode == SWTB_MODE_SAMPLE_WISE_PR_DP) pi = std::min(pi, cfg.max_parallel);
    else pi = 1;
    stats.parallel_iterations = pi;
  }

  // batched (reference run_batched): one group over the whole shard at the
  // padded extents, every intermediate materialized; sample_wise: padded
  // extents streamed in groups; +PR modes: true extents.
  const bool batched = cfg.mode == SWTB_MODE_BATCHED;
  const bool pad = cfg.mode == SWTB_MODE_BATCHED || cfg.mode == SWTB_MODE_SAMPLE_WISE;
  const bool host_in = bt.location == SWTB_HOST;
  const bool host_out = out.location == SWTB_HOST;
  // The batched comparator's batch-sized tensors stay cached for the next
  // batched step (like every workspace buffer) but are released when the
  // step fails (the reference's are step-scoped RAII tensors) and before a
  // sample-wise step, whose memory must not carry the batched footprint.
  struct BatchedRelease {
    swtb_ctx* c;
    bool on;
    int exc = std::uncaught_exceptions();
    ~BatchedRelease() {
      if (on && std::uncaught_exceptions() > exc) {
        c->drop(c->scores);
        c->drop(c->zs);
        c->drop(c->dhs);
      }
    }
  } batched_release{c, batched};
  if (!batched && c->scores.ptr) {
    c->drop(c->scores);
    c->drop(c->zs);
    c->drop(c->dhs);
  }
  // Per-sample tensors: the caller's layout (shard_local: this rank's
  // samples only), and the device staging of host buffers, which always
  // holds this rank's samples only (a rank stages 1/nranks of the batch).
  const long long B_own = owned_samples(B, c->rank, c->nranks);
  const bool local = bt.shard_local != 0;
  const SlotMap own_slot{c->rank, c->nranks, true};
  const SlotMap user_slot{c->rank, c->nranks, local};
  const SlotMap in_slot = host_in ? own_slot : user_slot;
  const SlotMap out_slot = host_out ? own_slot : user_slot;
  const long long B_lab = local ? B_own : B;  // label rows in the caller's layout
  const long long B_out = out_slot.local ? B_own : B;
  // device bytes that do not depend on the plan (inputs staged from the
  // host, parameter operands, accumulators, host-path outputs)
  auto r256 = [](long long x) { return std::max<long long>(round_up(std::max<long long>(x, 16), 256), 256); };
  const long long fixed_bytes =
      (host_in ? r256(B_own * T * H_A * 4) + r256(B_own * U1max * H_L * 4) + r256(std::max<long long>(B_lab * U, 4) * 4) : r256(16)) +
      (pr.location == SWTB_HOST ? r256((H * H_A + H * H_L + H + V * H + V) * 4 + 256) : 0) +
      r256(V_pad * 4) + r256(V * H_pad * esz * (c->split_w ? 2 : 1)) +
      r256(2 * H * HA_pad * 2) + r256(2 * H * HL_pad * 2) +
      r256((H * H_A + H * H_L + H + V * H + V + B) * 4) + r256(16) +
      (host_out ? r256(B_own * T * H_A * 4) + r256(B_own * U1max * H_L * 4) : 0);
  // workspace of a plan (mirrors the allocations below)
  // x slab: the dh slab holds the whole group (the forward writes x there)
  const bool store_x = c->store_x && !tf32 && !batched && V_pad <= kXMaxLd;
  const bool skip = c->skip_zero_tiles && c->prec == Prec::kFP16 && !batched && !store_x;
  const long long bwd_tiles =
      store_x ? (1LL << 40)
              : std::max<long long>(64, c->bwd_slab_bytes / (128LL * V_pad * esz));
  auto ws_bytes = [&](const Plan& p) {
    const long long rows = p.max_tiles * 128;
    const long long dh_rows = batched ? rows : std::min(rows, bwd_tiles * 128);
    return r256(4 * p.max_R_A * HA_pad * 2) + r256(4 * p.max_R_L * HL_pad * 2) +
           r256(p.max_R_A * H_pad * 4) + r256(p.max_R_L * H_pad * 4) +
           r256(2 * p.max_R_A * H_pad * 2) + r256(2 * p.max_R_L * H_pad * 2) +
           r256(rows * H_pad * esz) + r256(dh_rows * V_pad * esz) +
           (store_x ? r256(rows * round_up(V_pad / 32, 8) * 4) : 0) +
           (skip ? r256(2 * round_up(p.max_tiles + 64, 256)) + r256(round_up(p.max_tiles, 64) * 4 + 256) +
                       r256(p.max_lat * 4)
                 : 0) +
           r256(2 * p.max_tiles * kTileT * H_pad * 4) + r256(2 * p.max_tiles * kTileU * H_pad * 4) +
           (c->fwd_corr && !batched ? r256(p.max_R_L * H_pad * 2) + r256(p.max_R_L * V_pad * 4) : 0) +
           3 * r256(p.max_lat * 4) + 4 * r256(p.max_lat * 8) + r256(p.max_samples * 8) +
           r256((long long)p.blob.size()) + (batched ? r256(rows * V_pad * 4) : 0) +
           (c->deterministic ? r256(4 * (long long)split_workspace_floats(
                                            c->device, int(V), int(H), int(H_A), int(H_L),
                                            std::max(p.max_R_A, p.max_R_L), dh_rows, tf32)) +
                                   r256(4 * (long long)dw_acc_slices(c->device, int(V), dh_rows, tf32) *
                                        (V * H + V))
                             : 0);
  };
  long long budget = batched ? (1LL << 62) : c->group_cells;
  std::vector<int64_t> key = {bt.B, bt.T, bt.U, c->rank, c->nranks, budget,
                              c->joint_batch, int64_t(pad), c->alloc_ceiling,
                              int64_t(in_slot.local), int64_t(out_slot.local), int64_t(local)};
  key.insert(key.end(), bt.t_len, bt.t_len + bt.B);
  key.insert(key.end(), bt.u_len, bt.u_len + bt.B);
  if (!c->plan_cache || key != c->plan_key) {
    auto p = std::make_shared<Plan>(
        make_plan(bt, c->rank, c->nranks, budget, c->joint_batch, pad, in_slot, out_slot,
                  user_slot));
    // Under an allocation ceiling the sample-wise engines stream smaller
    // groups (down to one sample per group) until the workspace fits: device
    // memory is then bounded by the largest sample, not by B. Batched mode
    // never shrinks (it materializes the whole batch, reference behaviour).
    while (!batched && c->alloc_ceiling > 0 && budget > 1 && p->max_samples > 1 &&
           fixed_bytes + ws_bytes(*p) > c->alloc_ceiling) {
      budget /= 2;
      p = std::make_shared<Plan>(
          make_plan(bt, c->rank, c->nranks, budget, c->joint_batch, pad, in_slot, out_slot,
                  user_slot));
    }
    c->plan_cache = p;
    c->plan_key = std::move(key);
    c->plan_blob_dev = nullptr;
  }
  const Plan& plan = *static_cast<const Plan*>(c->plan_cache.get());
  stats.groups = (long long)plan.groups.size();
  stats.cells = plan.cells;
  stats.tiles = plan.tiles;
  const long long launches0 = launch_count();
  long long h2d = 0, d2h = 0;

  // ---- inputs on device ----
  const float* d_ac = bt.acoustic;
  const float* d_lb = bt.label;
  const int32_t* d_labels = bt.labels;
  // The small host copies (labels here, parameters below) are enqueued
  // before the bulk per-group input copies: copies of one direction share
  // the copy engine in submission order, so behind 2.5 GB of inputs they
  // would hold the first kernel back for the whole transfer.
  float* in_a = nullptr;
  float* in_l = nullptr;
  if (host_in) {
    in_a = static_cast<float*>(c->need(c->in_acoustic, size_t(std::max<long long>(1, B_own) * T * H_A) * 4, "acoustic"));
    in_l = static_cast<float*>(c->need(c->in_label, size_t(std::max<long long>(1, B_own) * U1max * H_L) * 4, "label"));
    if (U > 0 && B_lab > 0) {  // labels keep the caller's layout (small)
      int32_t* y = static_cast<int32_t*>(c->need(c->in_labels, size_t(B_lab * U) * 4, "labels"));
      CK(cudaMemcpyAsync(y, bt.labels, size_t(B_lab * U) * 4, cudaMemcpyHostToDevice, st));
      h2d += B_lab * U * 4;
      d_labels = y;
    }
    d_ac = in_a;
    d_lb = in_l;
  }
  // pageable caller buffers go through the pinned staging rings (PinnedRing)
  const bool pageable_in = host_in && (is_pageable(bt.acoustic) || is_pageable(bt.label));
  const bool pageable_out =
      host_out && (is_pageable(out.dacoustic) || is_pageable(out.dlabel));
  std::vector<long long> in_seq;  // ring job of each group's inputs
  // every job of this step has run before the step returns or unwinds (the
  // jobs read and write the caller's buffers)
  struct RingScope {
    swtb_ctx* c;
    int exc = std::uncaught_exceptions();
    ~RingScope() {
      for (auto* r : {c->ring_in.get(), c->ring_out.get()}) {
        if (!r) continue;
        if (std::uncaught_exceptions() > exc) {
          try {
            r->wait_all();
          } catch (...) {
          }
        } else {
          r->wait_all();
        }
      }
    }
  } ring_scope{c};
  auto wait_inputs = [&](size_t gi) {
    if (pageable_in && gi < in_seq.size()) c->ring(c->ring_in).wait(in_seq[gi]);
  };
  auto enqueue_inputs = [&] {
    if (!host_in) return;
    // per group, only the valid rows of each owned sample, on the copy
    // stream: group g+1's inputs stream in while group g computes
    float* a = in_a;
    float* l = in_l;
    c->events(c->ev_in, std::max<size_t>(1, plan.groups.size()));  // a rank may own no sample
    cudaStream_t in_stream = pageable_in ? c->ring(c->ring_in).stream() : c->cp_stream;
    CK(cudaEventRecord(c->ev_in[0], st));  // buffers free, small copies issued first
    CK(cudaStreamWaitEvent(in_stream, c->ev_in[0], 0));
    struct Run {
      void* dst;
      const void* src;
      size_t n;
    };
    std::vector<Run> runs;
    // samples whose slots are consecutive on both sides (host: the caller's
    // layout, device: this rank's staging slots) go as one copy from the
    // first sample's slot to the last one's valid rows: few large copies
    // instead of two per sample (the host-side call rate, not the link,
    // bounded it)
    auto copy_runs = [&](const std::vector<SampleDesc>& ss, float* dst, const float* src,
                         long long slot, long long width, bool acoustic) {
      size_t d0 = 0, h0 = 0, n = 0;
      long long last_d = -2, last_h = -2;
      auto flush = [&] {
        if (n > 0) {
          if (pageable_in)
            runs.push_back({dst + d0, src + h0, n * 4});
          else
            CK(cudaMemcpyAsync(dst + d0, src + h0, n * 4, cudaMemcpyHostToDevice, c->cp_stream));
          h2d += (long long)n * 4;
        }
      };
      for (const SampleDesc& sd : ss) {
        const long long ds = own_slot(sd.b), hs = user_slot(sd.b);
        const size_t len = size_t(acoustic ? sd.T : sd.U1) * width;
        if (ds == last_d + 1 && hs == last_h + 1) {
          n = size_t(ds - (long long)(d0 / size_t(slot * width))) * slot * width + len;
        } else {
          flush();
          d0 = size_t(ds) * slot * width;
          h0 = size_t(hs) * slot * width;
          n = len;
        }
        last_d = ds;
        last_h = hs;
      }
      flush();
    };
    for (size_t gi = 0; gi < plan.groups.size(); ++gi) {
      runs.clear();
      copy_runs(plan.groups[gi].samples, a, bt.acoustic, T, H_A, true);
      copy_runs(plan.groups[gi].samples, l, bt.label, U1max, H_L, false);
      if (pageable_in) {
        cudaEvent_t ev = c->ev_in[gi];
        in_seq.push_back(c->ring(c->ring_in).post([runs, ev](PinnedRing& r) {
          for (const Run& x : runs) r.h2d(x.dst, x.src, x.n);
          CK(cudaEventRecord(ev, r.stream()));
        }));
      } else {
        CK(cudaEventRecord(c->ev_in[gi], c->cp_stream));
      }
    }
  };
  if (U == 0) d_labels = static_cast<int32_t*>(c->need(c->in_labels, 16, "labels"));

  c->stage(SWTB_STAGE_OTHER, 0);
  // ---- parameter operands ----
  const float *pwa = pr.w_acoustic, *pwl = pr.w_label, *pbz = pr.bias,
              *pwo = pr.w_out, *pbo = pr.bias_out;
  if (pr.location == SWTB_HOST) {
    // stage fp32 params in device memory (theta region is reused below)
    const size_t n = size_t(H * H_A + H * H_L + H + V * H + V);
    float* tmp = static_cast<float*>(c->need(c->p_bz, n * 4 + 256, "params"));
    float* q = tmp;
    auto up = [&](const float* src, size_t cnt) {
      CK(cudaMemcpyAsync(q, src, cnt * 4, cudaMemcpyHostToDevice, st));
      const float* r = q;
      q += cnt;
      return r;
    };
    pwa = up(pr.w_acoustic, size_t(H * H_A));
    pwl = up(pr.w_label, size_t(H * H_L));
    pbz = up(pr.bias, size_t(H));
    pwo = up(pr.w_out, size_t(V * H));
    pbo = up(pr.bias_out, size_t(V));
    h2d += (long long)n * 4;
  }
  enqueue_inputs();
  // b_O padded with zeros to a multiple of 32 (epilogues read float4 blocks)
  float* bo_pad = static_cast<float*>(c->need(c->p_bo, size_t(V_pad) * 4, "bias_out"));
  CK(cudaMemsetAsync(bo_pad, 0, size_t(V_pad) * 4, st));
  CK(cudaMemcpyAsync(bo_pad, pbo, size_t(V) * 4, cudaMemcpyDeviceToDevice, st));
  const size_t wo_elems = size_t(V * H_pad);
  void* wo_op = c->need(c->p_wo, wo_elems * esz * (c->split_w ? 2 : 1), "w_out");
  void* wo_lo = c->split_w ? static_cast<char*>(wo_op) + wo_elems * esz : nullptr;
  c->stage(SWTB_STAGE_PREP, 3);
  launch_convert_pad(pwo, V, H, H, wo_op, H_pad, c->prec, st, wo_lo);
  const Mat wo{wo_op, V, H, H_pad}, wo2{wo_lo, V, H, H_pad};
  const Mat* wlo = c->split_w ? &wo2 : nullptr;
  const Mat* wlo_bwd = c->split_w_bwd ? &wo2 : nullptr;
  const bool fwd_corr = c->fwd_corr && !batched;
  const Mat* wlo_fwd = fwd_corr ? nullptr : wlo;
  // joint-network weights as bf16 (hi, lo) split pairs
  using bf16 = __nv_bfloat16;
  bf16* wa_hi = static_cast<bf16*>(c->need(c->p_wa, size_t(2 * H * HA_pad) * 2, "w_acoustic"));
  bf16* wa_lo = wa_hi + H * HA_pad;
  launch_split_rows(pwa, H, H_A, H_A, nullptr, wa_hi, wa_lo, HA_pad, st);
  bf16* wl_hi = static_cast<bf16*>(c->need(c->p_wl, size_t(2 * H * HL_pad) * 2, "w_label"));
  bf16* wl_lo = wl_hi + H * HL_pad;
  launch_split_rows(pwl, H, H_L, H_L, nullptr, wl_hi, wl_lo, HL_pad, st);

  // ---- accumulators ----
  const long long n_dwa = H * H_A, n_dwl = H * H_L, n_dwo = V * H;
  const long long o_dwa = 0, o_dwl = o_dwa + n_dwa, o_dbz = o_dwl + n_dwl,
                  o_dwo = o_dbz + H, o_dbo = o_dwo + n_dwo, o_loss = o_dbo + V,
                  n_theta = o_loss + B;
  float* theta = static_cast<float*>(c->need(c->theta, size_t(n_theta) * 4, "grads"));
  CK(cudaMemsetAsync(theta, 0, size_t(n_theta) * 4, st));
  int* bad = static_cast<int*>(c->need(c->bad, 16, "status"));
  CK(cudaMemsetAsync(bad, 0, 16, st));
  float* d_w = nullptr;  // per-sample loss weights (host array -> device)
  if (bt.sample_weights) {
    d_w = static_cast<float*>(c->need(c->weights, size_t(B) * 4, "sample_weights"));
    CK(cudaMemcpyAsync(d_w, bt.sample_weights, size_t(B) * 4, cudaMemcpyHostToDevice, st));
    h2d += B * 4;
  }

  float* d_dac;
  float* d_dlb;
  if (out.location == SWTB_DEVICE) {
    d_dac = out.dacoustic;
    d_dlb = out.dlabel;
  } else {
    d_dac = static_cast<float*>(c->need(c->out_dacoustic, size_t(std::max<long long>(1, B_own) * T * H_A) * 4, "dacoustic"));
    d_dlb = static_cast<float*>(c->need(c->out_dlabel, size_t(std::max<long long>(1, B_own) * U1max * H_L) * 4, "dlabel"));
  }
  if (B_out > 0) {
    CK(cudaMemsetAsync(d_dac, 0, size_t(B_out * T * H_A) * 4, st));
    CK(cudaMemsetAsync(d_dlb, 0, size_t(B_out * U1max * H_L) * 4, st));
  }

  // ---- workspace ----
  char* desc = static_cast<char*>(c->need(c->desc, plan.blob.size(), "plan"));
  if (c->plan_blob_dev != desc) {  // a new plan, or the buffer moved
    CK(cudaMemcpyAsync(desc, plan.blob.data(), plan.blob.size(), cudaMemcpyHostToDevice, st));
    c->plan_blob_dev = desc;
  }
  const long long rows_max = plan.max_tiles * 128;
  // packed encoder rows: two joint batches' worth (a batch's joint backward
  // runs deferred, after the next batch's rows were packed)
  bf16* ha_base = static_cast<bf16*>(c->need(c->ha, size_t(4 * plan.max_R_A * HA_pad) * 2, "acoustic_rows"));
  bf16* hl_base = static_cast<bf16*>(c->need(c->hl, size_t(4 * plan.max_R_L * HL_pad) * 2, "label_rows"));
  float* pa = static_cast<float*>(c->need(c->pa, size_t(plan.max_R_A * H_pad) * 4, "proj_acoustic"));
  float* pl = static_cast<float*>(c->need(c->pl, size_t(plan.max_R_L * H_pad) * 4, "proj_label"));
  bf16* ga_hi = static_cast<bf16*>(c->need(c->ga, size_t(2 * plan.max_R_A * H_pad) * 2, "gate_acoustic"));
  bf16* ga_lo = ga_hi + plan.max_R_A * H_pad;
  bf16* gl_hi = static_cast<bf16*>(c->need(c->gl, size_t(2 * plan.max_R_L * H_pad) * 2, "gate_label"));
  bf16* gl_lo = gl_hi + plan.max_R_L * H_pad;
  void* zs = c->need(c->zs, size_t(rows_max * H_pad) * esz, "joint");
  const long long dh_rows = batched ? rows_max : std::min(rows_max, bwd_tiles * 128);
  void* dhs = c->need(c->dhs, size_t(dh_rows * V_pad) * esz, "dscores");
  const long long ld_xoff = round_up(V_pad / 32, 8);
  float* xoff = store_x ? static_cast<float*>(c->need(c->xoff, size_t(rows_max * ld_xoff) * 4, "logit_block_max")) : nullptr;
  // zero-tile skip (fp16, sample-wise modes, recompute pipeline)
  uint8_t* tflags_base = nullptr;
  const size_t tf_bytes = size_t(round_up(plan.max_tiles + 64, 256));
  float* lmpv = nullptr;
  int* tlist = nullptr;
  int* tcount = nullptr;
  unsigned long long* tactive = nullptr;
  if (skip) {
    tflags_base = static_cast<uint8_t*>(c->need(c->tflags, 2 * tf_bytes, "tile_flags"));
    lmpv = static_cast<float*>(c->need(c->lmp, size_t(plan.max_lat) * 4, "log_max_prob"));
    // lists [max_tiles] (rounded up to 64 entries: the counts and the 8-byte
    // step total after them stay aligned), kMaxParts counts, the total
    const size_t lbytes = size_t(round_up(plan.max_tiles, 64)) * 4;
    char* tl = static_cast<char*>(c->need(c->tlist, lbytes + 256, "tile_lists"));
    tlist = reinterpret_cast<int*>(tl);
    tcount = reinterpret_cast<int*>(tl + lbytes);
    tactive = reinterpret_cast<unsigned long long*>(tl + lbytes + 128);
    CK(cudaMemsetAsync(tactive, 0, 8, st));
  }
  // the gate partials of two groups (a group's ga/gl sums run deferred,
  // inside the next group's backward)
  const size_t pa_floats = size_t(plan.max_tiles * kTileT * H_pad);
  const size_t pl_floats = size_t(plan.max_tiles * kTileU * H_pad);
  float* parta_base = static_cast<float*>(c->need(c->parta, 2 * pa_floats * 4, "partials_acoustic"));
  float* partl_base = static_cast<float*>(c->need(c->partl, 2 * pl_floats * 4, "partials_label"));
  __half* zbar = fwd_corr ? static_cast<__half*>(c->need(c->zbar, size_t(plan.max_R_L * H_pad) * 2, "zbar")) : nullptr;
  float* cbias = fwd_corr ? static_cast<float*>(c->need(c->cbias, size_t(plan.max_R_L * V_pad) * 4, "bias_rows")) : nullptr;
  if (cbias && (c->cbias_zeroed != cbias || c->cbias_zeroed_bytes != c->cbias.bytes)) {
    // columns [V, V_pad) are staged by the forward epilogue (16-B copies)
    // but never written by the correction GEMM: zero them once
    CK(cudaMemsetAsync(cbias, 0, size_t(plan.max_R_L * V_pad) * 4, st));
    c->cbias_zeroed = cbias;
    c->cbias_zeroed_bytes = c->cbias.bytes;
  }
  float* lse = static_cast<float*>(c->need(c->lse, size_t(plan.max_lat) * 4, "log_den"));
  double* lpb = static_cast<double*>(c->need(c->lpb, size_t(plan.max_lat) * 8, "lp_blank"));
  double* lpy = static_cast<double*>(c->need(c->lpy, size_t(plan.max_lat) * 8, "lp_label"));
  double* alpha = static_cast<double*>(c->need(c->alpha, size_t(plan.max_lat) * 8, "alpha"));
  double* beta = static_cast<double*>(c->need(c->beta, size_t(plan.max_lat) * 8, "beta"));
  double* logz = static_cast<double*>(c->need(c->logz, size_t(plan.max_samples) * 8, "log_z"));
  float* ebv = static_cast<float*>(c->need(c->eb, size_t(plan.max_lat) * 4, "edge_blank"));
  float* eyv = static_cast<float*>(c->need(c->ey, size_t(plan.max_lat) * 4, "edge_label"));
  struct SplitWs {  // the split workspaces are this step's only (thread-local)
    ~SplitWs() {
      set_split_workspace(nullptr, 0);
      set_dw_accumulator(nullptr, 0);
    }
  } split_ws_scope;
  float* dw_acc = nullptr;
  const int dw_slices = dw_acc_slices(c->device, int(V), dh_rows, tf32);
  if (c->deterministic) {
    const size_t n = split_workspace_floats(c->device, int(V), int(H), int(H_A), int(H_L),
                                            std::max(plan.max_R_A, plan.max_R_L), dh_rows, tf32);
    set_split_workspace(static_cast<float*>(c->need(c->split_ws, n * 4, "split_partials")), n);
    const size_t na = size_t(dw_slices) * size_t(V * H + V);
    dw_acc = static_cast<float*>(c->need(c->dw_acc, na * 4, "dw_out_partials"));
    CK(cudaMemsetAsync(dw_acc, 0, na * 4, st));
    set_dw_accumulator(dw_acc, dw_slices);
  }

  const Prec P = c->prec;
  if (host_out) c->events(c->ev_done, plan.groups.size());
  // A group's tail: 9. ga / gl (+ db_Z) from its gate partials; 10. at the
  // joint batch's last group, the joint backward of the batch; then the
  // batch's dh^A / dh^L slots go back to the host. It is deferred into the
  // next group's backward, between its two parts: the engine stream then has
  // work while the second part's wavefront finishes on the lattice stream
  // (group-parity partials / flags and batch-parity packed rows keep the
  // next group from overwriting what the tail reads).
  long long pending = -1;
  auto group_tail = [&](size_t gi) {
    const Group& g = plan.groups[gi];
    const SampleDesc* d_s = reinterpret_cast<const SampleDesc*>(desc + g.off_samples);
    const int* d_asmp = reinterpret_cast<const int*>(desc + g.off_asmp);
    const int* d_lsmp = reinterpret_cast<const int*>(desc + g.off_lsmp);
    const int n_s = int(g.samples.size());
    const int R_A = int(g.R_A), R_L = int(g.R_L);
    const JBatch& jbt = plan.batches[size_t(g.jb)];
    const bool batch_last = int(gi) + 1 == jbt.g1;
    const long long* j_adst = reinterpret_cast<const long long*>(desc + jbt.off_adst);
    const long long* j_ldst = reinterpret_cast<const long long*>(desc + jbt.off_ldst);
    const int JR_A = int(jbt.R_A), JR_L = int(jbt.R_L);
    bf16* ha_hi = ha_base + size_t(g.jb & 1) * 2 * plan.max_R_A * HA_pad;
    bf16* ha_lo = ha_hi + plan.max_R_A * HA_pad;
    bf16* hl_hi = hl_base + size_t(g.jb & 1) * 2 * plan.max_R_L * HL_pad;
    bf16* hl_lo = hl_hi + plan.max_R_L * HL_pad;
    const Mat ha{ha_hi, JR_A, H_A, HA_pad}, ha2{ha_lo, JR_A, H_A, HA_pad};
    const Mat hl{hl_hi, JR_L, H_L, HL_pad}, hl2{hl_lo, JR_L, H_L, HL_pad};
    const Mat wa{wa_hi, H, H_A, HA_pad}, wa2{wa_lo, H, H_A, HA_pad};
    const Mat wl{wl_hi, H, H_L, HL_pad}, wl2{wl_lo, H, H_L, HL_pad};
    float* parta = parta_base + (gi & 1) * pa_floats;
    float* partl = partl_base + (gi & 1) * pl_floats;
    uint8_t* tflags = tflags_base ? tflags_base + (gi & 1) * tf_bytes : nullptr;
    // 9. ga / gl (+ db_Z) of this group, into the joint batch's rows
    c->stage(SWTB_STAGE_JOINT_BWD, 2);
    launch_reduce_partials(parta, partl, d_s, n_s, d_asmp, d_lsmp, int(g.ra0),
                           int(g.rl0), R_A, R_L, int(H), H_pad, ga_hi, ga_lo,
                           gl_hi, gl_lo, theta + o_dbz, st, skip ? tflags : nullptr);
    if (batch_last) {
      const Mat ga{ga_hi, JR_A, H, H_pad}, ga2{ga_lo, JR_A, H, H_pad};
      const Mat gl{gl_hi, JR_L, H, H_pad}, gl2{gl_lo, JR_L, H, H_pad};
      // 10. joint backward of the batch (split bf16 GEMMs, float32-grade):
      //     dh^A = ga W_A (scattered to batch slots), dW_A += ga^T h^A;
      //     same for the label side
      c->stage(SWTB_STAGE_JOINT_BWD, 4);
      gemm_store(Prec::kBF16, false, true, ga, wa, JR_A, int(H_A), int(H), d_dac,
                 H_A, nullptr, j_adst, st, &ga2, &wa2);
      gemm_atomic(Prec::kBF16, true, true, ga, ha, int(H), int(H_A), JR_A,
                  theta + o_dwa, H_A, st, &ga2, &ha2);
      gemm_store(Prec::kBF16, false, true, gl, wl, JR_L, int(H_L), int(H), d_dlb,
                 H_L, nullptr, j_ldst, st, &gl2, &wl2);
      gemm_atomic(Prec::kBF16, true, true, gl, hl, int(H), int(H_L), JR_L,
                  theta + o_dwl, H_L, st, &gl2, &hl2);
    }
    if (host_out && batch_last) {
      // the batch's dh^A / dh^L slots (padding rows included: zero) go back
      // on the copy stream while the next batch computes
      CK(cudaEventRecord(c->ev_done[gi], st));
      if (!pageable_out) CK(cudaStreamWaitEvent(c->cp_stream, c->ev_done[gi], 0));
      // runs of samples whose whole slots are consecutive on both sides
      // (device staging slot, the caller's host slot), one copy per run
      struct Run {
        void* dst;
        const void* src;
        size_t n;
      };
      std::vector<Run> runs;
      long long d0 = -1, h0 = -1, n = 0;
      auto copy_out = [&](float* dst, const float* src, long long cnt) {
        if (pageable_out)
          runs.push_back({dst, src, size_t(cnt) * 4});
        else
          CK(cudaMemcpyAsync(dst, src, size_t(cnt) * 4, cudaMemcpyDeviceToHost, c->cp_stream));
        d2h += cnt * 4;
      };
      auto flush = [&] {
        if (n == 0) return;
        if (out.dacoustic)
          copy_out(out.dacoustic + h0 * T * H_A, d_dac + d0 * T * H_A, n * T * H_A);
        if (out.dlabel)
          copy_out(out.dlabel + h0 * U1max * H_L, d_dlb + d0 * U1max * H_L, n * U1max * H_L);
      };
      for (int bg = jbt.g0; bg < jbt.g1; ++bg)
        for (const SampleDesc& sd : plan.groups[size_t(bg)].samples) {
          const long long ds = own_slot(sd.b), hs = user_slot(sd.b);
          if (n > 0 && ds == d0 + n && hs == h0 + n) {
            ++n;
          } else {
            flush();
            d0 = ds;
            h0 = hs;
            n = 1;
          }
        }
      flush();
      if (pageable_out) {  // the batch's slots drain through the output ring
        cudaEvent_t ev = c->ev_done[gi];
        c->ring(c->ring_out).post([runs, ev](PinnedRing& r) {
          CK(cudaStreamWaitEvent(r.stream(), ev, 0));
          for (const Run& x : runs) r.d2h(x.dst, x.src, x.n);
          r.drain();
        });
      }
    }
  };
  for (size_t gi = 0; gi < plan.groups.size(); ++gi) {
    const Group& g = plan.groups[gi];
    if (host_in) {  // this group's rows are in
      wait_inputs(gi);
      CK(cudaStreamWaitEvent(st, c->ev_in[gi], 0));
    }
    const SampleDesc* d_s = reinterpret_cast<const SampleDesc*>(desc + g.off_samples);
    const TileDesc* d_t = reinterpret_cast<const TileDesc*>(desc + g.off_tiles);
    const int n_s = int(g.samples.size());
    const int n_tiles = int(g.tiles.size());

    const JBatch& jbt = plan.batches[size_t(g.jb)];
    const bool batch_first = int(gi) == jbt.g0;
    const long long* j_asrc = reinterpret_cast<const long long*>(desc + jbt.off_asrc);
    const long long* j_lsrc = reinterpret_cast<const long long*>(desc + jbt.off_lsrc);
    const int* j_linfo = reinterpret_cast<const int*>(desc + jbt.off_linfo);
    const int JR_A = int(jbt.R_A), JR_L = int(jbt.R_L);
    // joint-batch parity packed rows, group parity partials / tile flags
    bf16* ha_hi = ha_base + size_t(g.jb & 1) * 2 * plan.max_R_A * HA_pad;
    bf16* ha_lo = ha_hi + plan.max_R_A * HA_pad;
    bf16* hl_hi = hl_base + size_t(g.jb & 1) * 2 * plan.max_R_L * HL_pad;
    bf16* hl_lo = hl_hi + plan.max_R_L * HL_pad;
    float* parta = parta_base + (gi & 1) * pa_floats;
    float* partl = partl_base + (gi & 1) * pl_floats;
    uint8_t* tflags = tflags_base ? tflags_base + (gi & 1) * tf_bytes : nullptr;
    const Mat ha{ha_hi, JR_A, H_A, HA_pad}, ha2{ha_lo, JR_A, H_A, HA_pad};
    const Mat hl{hl_hi, JR_L, H_L, HL_pad}, hl2{hl_lo, JR_L, H_L, HL_pad};
    const Mat wa{wa_hi, H, H_A, HA_pad}, wa2{wa_lo, H, H_A, HA_pad};
    const Mat wl{wl_hi, H, H_L, HL_pad}, wl2{wl_lo, H, H_L, HL_pad};
    if (batch_first) {
      // the whole joint batch's encoder rows must be on the device
      if (host_in) {
        wait_inputs(size_t(jbt.g1 - 1));
        CK(cudaStreamWaitEvent(st, c->ev_in[size_t(jbt.g1 - 1)], 0));
      }
      // 1. gather valid encoder rows (padding removal) as split bf16 pairs
      c->stage(SWTB_STAGE_PREP, 2);
      launch_split_rows(d_ac, JR_A, H_A, H_A, j_asrc, ha_hi, ha_lo, HA_pad, st);
      launch_split_rows(d_lb, JR_L, H_L, H_L, j_lsrc, hl_hi, hl_lo, HL_pad, st);
      // 2. joint projections P_A = h^A W_A^T + b_Z, P_L = h^L W_L^T
      c->stage(SWTB_STAGE_JOINT_FWD, 2);
      gemm_store(Prec::kBF16, false, false, ha, wa, JR_A, int(H), int(H_A), pa,
                 H_pad, pbz, nullptr, st, &ha2, &wa2);
      gemm_store(Prec::kBF16, false, false, hl, wl, JR_L, int(H), int(H_L), pl,
                 H_pad, nullptr, nullptr, st, &hl2, &wl2);
      if (fwd_corr) {
        // per-label-row logit correction of the single-fp16-W_O forward, for
        // the whole joint batch: bias_rows[r] = b_O + zbar_r . W_lo^T (zbar
        // over 32 evenly spaced frames of the row's sample)
        c->stage(SWTB_STAGE_PREP, 2);
        launch_zmean(pa, pl, H_pad, int(H), j_linfo, JR_L, 32, zbar, H_pad, st);
        gemm_store(Prec::kFP16, false, false, Mat{zbar, JR_L, H, H_pad}, wo2, JR_L, int(V),
                   int(H), cbias, V_pad, bo_pad, nullptr, st);
      }
    }
    if (batched) {
      // Reference run_batched (engine.cpp:245-323), stage-major over the
      // whole shard at the padded extents with every intermediate kept in
      // HBM: joint [cells, H], scores [cells, V] fp32, log_den / alpha /
      // beta, dscores [cells, V]; then dz (+ tanh gate, lattice sums) and
      // dW_O / db_O. The comparator for the sample-wise engine's memory.
      const long long rows = (long long)n_tiles * 128;
      c->stage(SWTB_STAGE_PREP, 1);
      launch_zslab(pa, pl, H_pad, int(H), d_t, d_s, n_tiles, zs, H_pad, P, st);
      float* sc = static_cast<float*>(c->need(c->scores, size_t(rows * V_pad) * 4, "scores"));
      c->stage(SWTB_STAGE_OUT_FWD, 2);
      gemm_store(P, false, false, Mat{zs, rows, H, H_pad}, wo, int(rows), int(V), int(H), sc,
                 V_pad, bo_pad, nullptr, st, nullptr, wlo);
      CK(cudaMemsetAsync(lpb, 0, size_t(g.lat) * 8, st));
      CK(cudaMemsetAsync(lpy, 0, size_t(g.lat) * 8, st));
      launch_tile_scores_lse(sc, V_pad, rows, d_t, d_s, d_labels, int(V), lse, lpb, lpy, st);
      int max_D = 1;
      for (const SampleDesc& sd : g.samples) max_D = std::max(max_D, sd.T + sd.U1 - 1);
      c->stage(SWTB_STAGE_LATTICE, 2);
      launch_lattice(d_s, n_s, d_labels, lpb, lpy, alpha, beta, logz, theta + o_loss,
                     g.max_U1, st);
      launch_edge(d_s, n_s, max_D, lpb, lpy, alpha, beta, logz, lse, ebv, eyv, st, d_w);
      c->stage(SWTB_STAGE_OUT_DH, 1);
      launch_tile_dscores(sc, V_pad, rows, d_t, d_s, d_labels, int(V), V_pad, lse, ebv, eyv,
                          dhs, V_pad, P, bad, st);
      c->stage(SWTB_STAGE_OUT_DZ, 1);
      GateArgs gg{d_t, d_s, zs, H_pad, int(H), parta, partl, H_pad};
      gemm_dz_gate(P, Mat{dhs, rows, V, V_pad}, wo, int(rows), int(V), int(H), gg, st, wlo_bwd);
      c->stage(SWTB_STAGE_OUT_DW, 1);
      gemm_dw_db(P, Mat{dhs, rows, V, V_pad}, Mat{zs, rows, H, H_pad}, int(V), int(H),
                 int(rows), theta + o_dwo, theta + o_dbo, bad, st);
    } else {
      // 3. z slab (tile order)
      c->stage(SWTB_STAGE_PREP, 1);
      launch_zslab(pa, pl, H_pad, int(H), d_t, d_s, n_tiles, zs, H_pad, P, st);

      // 4-8. The group is cut into two parts at a sample boundary near its tile
      //      midpoint. f^O forward of part 0, then of part 1 while part 0's
      //      alpha/beta wavefront runs on the lattice stream; then the backward
      //      of part 0 while part 1's wavefront runs. The persistent GEMMs leave
      //      the wavefront's SM(s) free meanwhile.
      //      (Off-lattice positions of the skewed lp arrays stay zero: the
      //      wavefront reads them unmasked.)
      CK(cudaMemsetAsync(lpb, 0, size_t(g.lat) * 8, st));
      CK(cudaMemsetAsync(lpy, 0, size_t(g.lat) * 8, st));
      if (skip) CK(cudaMemsetAsync(tflags, 0, size_t(n_tiles), st));
      struct Part { int s0, s1, t0, t1, max_U1, max_D; };
      std::vector<Part> parts;
      {
        // up to kMaxParts parts cut at sample boundaries near equal tile counts:
        // part i's wavefront hides behind the forward GEMMs of parts i+1..n
        static const int max_parts = [] {
          const char* e = std::getenv("SWTB_PARTS");  // experiments; default 2
          const int v = e ? std::atoi(e) : 2;
          return std::max(1, std::min(swtb_ctx::kMaxParts, v));
        }();
        const int np = std::min(max_parts, n_s);
        auto mk = [&](int a, int b) {
          Part pt{a, b, g.samples[a].tile0, b < n_s ? g.samples[b].tile0 : n_tiles, 1, 1};
          for (int i = a; i < b; ++i) {
            pt.max_U1 = std::max(pt.max_U1, g.samples[i].U1);
            pt.max_D = std::max(pt.max_D, g.samples[i].T + g.samples[i].U1 - 1);
          }
          return pt;
        };
        // Part 0 is the lead fraction of the tiles (>= 1 sample): its
        // wavefront hides behind the forward of the rest, and the rest's
        // wavefront behind part 0's backward. 0.4 since the zero-tile skip
        // shortened the backward (A/B at c4: 0.25 428 ms, 0.33 426, 0.4 423).
        static const double lead = [] {
          const char* e = std::getenv("SWTB_LEAD");
          const double v = e ? std::atof(e) : 0.4;
          return v > 0.0 && v < 1.0 ? v : 0.4;
        }();
        int a = 0;
        for (int pi = 1; pi <= np && a < n_s; ++pi) {
          int b = n_s;
          if (pi < np) {
            const double f = np == 2 ? lead : double(pi) / np;
            const long long target = (long long)(double(n_tiles) * (pi == 1 ? f : double(pi) / np));
            b = a + 1;
            while (b < n_s - (np - pi) && g.samples[b].tile0 < target) ++b;
          }
          parts.push_back(mk(a, b));
          a = b;
        }
      }
      // SMs the GEMMs leave to wavefronts that may run concurrently: during
      // fwd(i) those of parts < i, during bwd(i) those of parts > i
      std::vector<int> lat_ctas(parts.size());
      for (size_t pi = 0; pi < parts.size(); ++pi)
        lat_ctas[pi] = lattice_launch_ctas(parts[pi].s1 - parts[pi].s0, parts[pi].max_U1);
      auto reserve_range = [&](size_t a, size_t b) {  // max over parts [a, b)
        int r = 0;
        for (size_t i = a; i < b; ++i) r = std::max(r, lat_ctas[i]);
        return r;
      };
      for (size_t pi = 0; pi < parts.size(); ++pi) {
        const Part& pt = parts[pi];
        set_gemm_sm_reserve(reserve_range(0, pi));
        const int prow0 = pt.t0 * 128, prows = (pt.t1 - pt.t0) * 128;
        const void* zp = static_cast<const char*>(zs) + size_t(prow0 * H_pad) * esz;
        c->stage(SWTB_STAGE_OUT_FWD, 1);
        FwdLseArgs fa{d_t + pt.t0, d_s, d_labels, bo_pad, int(V), lse, lpb, lpy};
        fa.lmp = lmpv;
        if (fwd_corr) {
          fa.bias_rows = cbias;
          fa.ld_bias_rows = V_pad;
        }
        if (store_x) {  // the group's x slab rows of this part
          fa.xs = static_cast<char*>(dhs) + size_t(prow0 * V_pad) * 2;
          fa.ld_x = V_pad;
          fa.xoff = xoff + prow0 * ld_xoff;
          fa.ld_xoff = ld_xoff;
        }
        gemm_fwd_lse(P, Mat{zp, prows, H, H_pad}, wo, prows, int(V), int(H), fa, st,
                     wlo_fwd);
        // alpha / beta wavefront of this part, per-sample loss
        c->end_stage();
        CK(cudaEventRecord(c->ev_fwd[pi], st));
        CK(cudaStreamWaitEvent(c->lat_stream, c->ev_fwd[pi], 0));
        cudaEvent_t le0 = nullptr;
        c->side_begin(c->lat_stream, &le0);
        launch_lattice(d_s + pt.s0, pt.s1 - pt.s0, d_labels, lpb, lpy, alpha, beta,
                       logz + pt.s0, theta + o_loss, pt.max_U1, c->lat_stream);
        launch_edge(d_s + pt.s0, pt.s1 - pt.s0, pt.max_D, lpb, lpy, alpha, beta,
                    logz + pt.s0, lse, ebv, eyv, c->lat_stream, d_w, tflags, -26.f, lmpv);
        if (skip)  // this part's active tiles, ascending
          launch_compact_tiles(tflags + pt.t0, pt.t1 - pt.t0, tlist + pt.t0, tcount + pi,
                               tactive, c->lat_stream);
        c->side_end(SWTB_STAGE_LATTICE, c->lat_stream, le0);
        CK(cudaEventRecord(c->ev_lat[pi], c->lat_stream));
      }
      // backward of each part over sub-slabs of at most bwd_tiles tiles (bounds
      // the dh slab): logit recompute + dh epilogue (+ db_O); dz = dh W_O with
      // the tanh gate and lattice-axis partial sums; dW_O += dh^T z (both
      // operands MN-major views of the slabs)
      for (size_t pi = 0; pi < parts.size(); ++pi) {
        const Part& pt = parts[pi];
        if (pi == 1 && pending >= 0) {
          // the previous group's tail fills the gap while this part's
          // wavefront still runs: its GEMMs leave that wavefront's SMs free
          set_gemm_sm_reserve(reserve_range(pi, parts.size()));
          group_tail(size_t(pending));
          pending = -1;
        }
        set_gemm_sm_reserve(reserve_range(pi + 1, parts.size()));
        c->stage(SWTB_STAGE_WAIT, 0);  // time the engine stream idles on it
        CK(cudaStreamWaitEvent(st, c->ev_lat[pi], 0));
        if (skip) {
          // only the part's active tiles (device list, count unknown here):
          // compacted chunks of <= bwd_tiles list entries; z and the
          // epilogues' metadata at the real tiles, dh in list order
          const long long ptiles = pt.t1 - pt.t0;
          const int prow = int(ptiles * 128);
          const void* zpart = static_cast<const char*>(zs) + size_t(pt.t0 * 128 * H_pad) * esz;
          for (long long c0 = 0; c0 < ptiles; c0 += bwd_tiles) {
            const int nt = int(std::min<long long>(bwd_tiles, ptiles - c0));
            const int crows = nt * 128;
            RowMap m;
            m.list = tlist + pt.t0 + c0;
            m.count = tcount + pi;
            m.offset = int(c0);
            m.max = nt;
            c->stage(SWTB_STAGE_OUT_DH, 1);
            BwdDhArgs ba{d_t + pt.t0, d_s, d_labels, bo_pad, int(V), lse, ebv, eyv,
                         dhs, V_pad, bad};
            ba.map = m;
            ba.dh_rows = crows;
            gemm_bwd_dh(P, Mat{zpart, prow, H, H_pad}, wo, prow, int(V), int(H), ba, st,
                        wlo_bwd);
            c->stage(SWTB_STAGE_OUT_DZ, 1);
            GateArgs gg{d_t + pt.t0, d_s, zpart, H_pad, int(H), parta + pt.t0 * kTileT * H_pad,
                        partl + pt.t0 * kTileU * H_pad, H_pad};
            gg.map = m;
            gg.z_rows = prow;
            gemm_dz_gate(P, Mat{dhs, crows, V, V_pad}, wo, crows, int(V), int(H), gg, st,
                         wlo_bwd);
            c->stage(SWTB_STAGE_OUT_DW, 1);
            gemm_dw_db(P, Mat{dhs, crows, V, V_pad}, Mat{zpart, prow, H, H_pad}, int(V), int(H),
                       crows, theta + o_dwo, theta + o_dbo, bad, st, m);
          }
          continue;
        }
        for (long long t0 = pt.t0; t0 < pt.t1; t0 += bwd_tiles) {
          const int nt = int(std::min<long long>(bwd_tiles, pt.t1 - t0));
          const int srows = nt * 128;
          const TileDesc* st_t = d_t + t0;
          const void* zsub = static_cast<const char*>(zs) + size_t(t0 * 128 * H_pad) * esz;
          // store_x: the part's dh is formed in place over its x-slab rows
          void* dh_sub = store_x ? static_cast<void*>(static_cast<char*>(dhs) +
                                                      size_t(t0 * 128 * V_pad) * 2)
                                 : dhs;
          c->stage(SWTB_STAGE_OUT_DH, 1);
          if (store_x) {
            launch_x_to_dh(dh_sub, V_pad, xoff + t0 * 128 * ld_xoff, ld_xoff, srows, st_t, d_s,
                           d_labels, int(V), lse, ebv, eyv, P, bad, st);
          } else {
            BwdDhArgs ba{st_t, d_s, d_labels, bo_pad, int(V), lse, ebv, eyv,
                         dhs, V_pad, bad};
            gemm_bwd_dh(P, Mat{zsub, srows, H, H_pad}, wo, srows, int(V), int(H), ba, st,
                        wlo_bwd);
          }
          c->stage(SWTB_STAGE_OUT_DZ, 1);
          GateArgs gg{st_t, d_s, zsub, H_pad, int(H), parta + t0 * kTileT * H_pad,
                      partl + t0 * kTileU * H_pad, H_pad};
          gemm_dz_gate(P, Mat{dh_sub, srows, V, V_pad}, wo, srows, int(V), int(H), gg,
                       st, wlo_bwd);
          c->stage(SWTB_STAGE_OUT_DW, 1);
          gemm_dw_db(P, Mat{dh_sub, srows, V, V_pad}, Mat{zsub, srows, H, H_pad}, int(V),
                     int(H), srows, theta + o_dwo, theta + o_dbo, bad, st);
        }
      }
      set_gemm_sm_reserve(0);
    }
    // the group's tail (ga/gl sums, joint backward, output copies) runs
    // deferred, inside the next group's backward (or right here)
    if (pending >= 0) group_tail(size_t(pending));
    pending = (long long)gi;
  }
  if (pending >= 0) group_tail(size_t(pending));

  // deterministic dW_O / db_O: the accumulator slices, in slice order
  if (dw_acc) {
    c->stage(SWTB_STAGE_OUT_DW, 2);
    launch_split_reduce(dw_acc, dw_slices, V * H, V * H, theta + o_dwo, st);
    launch_split_reduce(dw_acc + size_t(dw_slices) * V * H, dw_slices, V, V, theta + o_dbo, st);
  }
  // ---- cross-rank reduction: one all-reduce of theta-grads + losses ----
  c->stage(SWTB_STAGE_OTHER, 0);
  if (c->comm) {
    c->stage(SWTB_STAGE_COMM, 0);
    nccl_check(nccl().all_reduce(theta, theta, size_t(n_theta), ncclFloat, ncclSum,
                             c->comm, st),
               "ncclAllReduce");
    c->stage(SWTB_STAGE_OTHER, 0);
  }

  // ---- outputs ----
  std::vector<float> h_loss(static_cast<size_t>(B));
  int h_bad = 0;
  unsigned long long h_active = 0;
  if (skip) CK(cudaMemcpyAsync(&h_active, tactive, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_loss.data(), theta + o_loss, size_t(B) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
  d2h += B * 4 + 4;
  const cudaMemcpyKind k = out.location == SWTB_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  auto cp = [&](float* dst, long long off, long long n) {
    if (!dst) return;
    CK(cudaMemcpyAsync(dst, theta + off, size_t(n) * 4, k, st));
    if (k == cudaMemcpyDeviceToHost) d2h += n * 4;
  };
  cp(out.dw_acoustic, o_dwa, n_dwa);
  cp(out.dw_label, o_dwl, n_dwl);
  cp(out.dbias, o_dbz, H);
  cp(out.dw_out, o_dwo, n_dwo);
  cp(out.dbias_out, o_dbo, V);
  if (host_out) CK(cudaStreamSynchronize(c->cp_stream));
  if (pageable_out) c->ring(c->ring_out).wait_all();
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  c->collect();

  // reference semantics: non-finite log Z / dh -> NumericalDegeneracyError
  double total = 0.0;
  for (long long b = 0; b < B; ++b) {
    if (!std::isfinite(h_loss[size_t(b)]))
      fail(SWTB_ERR_NUMERIC, "no alignment path carries mass (sample " + std::to_string(b) + ")");
    total += double(h_loss[size_t(b)]);
  }
  if (h_bad) fail(SWTB_ERR_NUMERIC, "non-finite output-score gradient");
  if (out.sample_losses) {
    if (out.location == SWTB_DEVICE)
      CK(cudaMemcpy(out.sample_losses, h_loss.data(), size_t(B) * 4, cudaMemcpyHostToDevice));
    else
      std::memcpy(out.sample_losses, h_loss.data(), size_t(B) * 4);
  }
  if (out.loss) {
    // ascending-b sum of the per-sample losses (reference engine.cpp:390-395)
    float acc = 0.f;
    for (long long b = 0; b < B; ++b) acc += h_loss[size_t(b)];
    (void)total;
    if (out.location == SWTB_DEVICE)
      CK(cudaMemcpy(out.loss, &acc, 4, cudaMemcpyHostToDevice));
    else
      *out.loss = acc;
  }
  stats.kernel_launches = launch_count() - launches0;
  stats.h2d_bytes = h2d;
  stats.d2h_bytes = d2h;
  stats.peak_bytes = c->peak_bytes;
  stats.logits_stored = store_x ? 1 : 0;
  stats.active_tiles = skip ? (long long)h_active : -1;
  c->stats = stats;
}

void transducer_loss(swtb_ctx* c, const double* scores, int64_t frames,
                     int64_t labels, int64_t vocab, const int32_t* y,
                     double* loss, double* dscores) {
  if (frames < 1) fail(SWTB_ERR_INPUT, "lattice needs at least one frame");
  if (labels < 0 || vocab < 1) fail(SWTB_ERR_SHAPE, "invalid lattice extents");
  for (int64_t i = 0; i < labels; ++i)
    if (y[i] <= 0 || y[i] >= vocab)
      fail(SWTB_ERR_INPUT, "label id " + std::to_string(y[i]) + " outside [1, " + std::to_string(vocab) + ")");
  CK(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  const int T = int(frames), U1 = int(labels) + 1, V = int(vocab);
  const size_t n = size_t(T) * U1 * V;
  double* d_sc = static_cast<double*>(c->need(c->op_scores, n * 8));
  double* d_ds = static_cast<double*>(c->need(c->op_dscores, n * 8));
  int* d_y = static_cast<int*>(c->need(c->op_y, size_t(U1) * 4));
  SampleDesc sd{};
  sd.T = T;
  sd.U1 = U1;
  const long long slack = lat_slack(U1);
  sd.lat = slack;
  sd.b = 0;
  SampleDesc* d_sd = static_cast<SampleDesc*>(c->need(c->op_sd, sizeof(SampleDesc)));
  const long long L = skew_size(T, U1) + 2 * slack;
  float* lse = static_cast<float*>(c->need(c->lse, size_t(L) * 4));
  double* lpb = static_cast<double*>(c->need(c->lpb, size_t(L) * 8));
  double* lpy = static_cast<double*>(c->need(c->lpy, size_t(L) * 8));
  double* al = static_cast<double*>(c->need(c->alpha, size_t(L) * 8));
  double* be = static_cast<double*>(c->need(c->beta, size_t(L) * 8));
  double* lz = static_cast<double*>(c->need(c->logz, 16));
  float* ls = static_cast<float*>(c->need(c->theta, 16));
  CK(cudaMemcpyAsync(d_sc, scores, n * 8, cudaMemcpyHostToDevice, st));
  if (labels > 0) CK(cudaMemcpyAsync(d_y, y, size_t(labels) * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_sd, &sd, sizeof(sd), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(lpb, 0, size_t(L) * 8, st));
  CK(cudaMemsetAsync(lpy, 0, size_t(L) * 8, st));
  launch_scores_lse(d_sc, T, U1, V, d_y, d_sd, lse, lpb, lpy, st);
  launch_lattice(d_sd, 1, d_y, lpb, lpy, al, be, lz, ls, U1, st);
  launch_scores_grad(d_sc, T, U1, V, d_y, d_sd, lse, al, be, lz, d_ds, st);
  double h_lz = 0;
  CK(cudaMemcpyAsync(&h_lz, lz, 8, cudaMemcpyDeviceToHost, st));
  if (dscores) CK(cudaMemcpyAsync(dscores, d_ds, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (!std::isfinite(h_lz)) fail(SWTB_ERR_NUMERIC, "total path log-probability is not finite");
  *loss = -h_lz * 0.6931471805599453;  // the lattice works in log2 units
  if (dscores)
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(dscores[i])) fail(SWTB_ERR_NUMERIC, "non-finite output-score gradient");
}

template <class F>
swtb_status guarded(swtb_ctx* c, F&& f) {
  try {
    f();
    return SWTB_OK;
  } catch (const SwtbError& e) {
    (c ? c->last_error : g_last_error) = e.what();
    return e.status;
  } catch (const std::exception& e) {
    (c ? c->last_error : g_last_error) = e.what();
    return SWTB_ERR_INTERNAL;
  } catch (...) {
    (c ? c->last_error : g_last_error) = "unknown error";
    return SWTB_ERR_INTERNAL;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int swtb_abi_version(void) { return SWTB_ABI_VERSION; }

swtb_status swtb_ctx_create(const swtb_opts* opts, swtb_ctx** out) {
  if (!out) return SWTB_ERR_INPUT;
  *out = nullptr;
  swtb_ctx* c = nullptr;
  swtb_status s = guarded(nullptr, [&] {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      fail(SWTB_ERR_CUDA, "no CUDA device available (libswt_b200 has no CPU path)");
    }
    const int dev = opts ? opts->device : 0;
    if (dev < 0 || dev >= ndev) fail(SWTB_ERR_INPUT, "device ordinal out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
      fail(SWTB_ERR_CUDA, std::string("libswt_b200 is built for sm_100a; device is ") + prop.name);
    c = new swtb_ctx();
    c->device = dev;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->lat_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->cp_stream, cudaStreamNonBlocking));
    for (int i = 0; i < swtb_ctx::kMaxParts; ++i) {
      CK(cudaEventCreateWithFlags(&c->ev_fwd[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_lat[i], cudaEventDisableTiming));
    }
    if (opts) {
      if (opts->precision < SWTB_PREC_BF16 || opts->precision > SWTB_PREC_FP16)
        fail(SWTB_ERR_INPUT, "unknown precision");
      c->prec = opts->precision == SWTB_PREC_TF32   ? Prec::kTF32
                : opts->precision == SWTB_PREC_FP16 ? Prec::kFP16
                                                    : Prec::kBF16;
      c->split_w = opts->precision != SWTB_PREC_BF16;
      // fp16: the (hi, lo) W_O pair only in the f^O forward (the lattice's
      // logits); recompute and dz read the single fp16 W_O
      c->split_w_bwd = c->split_w && opts->precision != SWTB_PREC_FP16;
      c->fwd_corr = opts->precision == SWTB_PREC_FP16 && [] {
        const char* e = std::getenv("SWTB_FWD_CORR");  // 0 = (hi, lo) forward (A/B)
        return !(e && std::atoi(e) == 0);
      }();
      if (opts->group_cells > 0) {
        c->group_cells = opts->group_cells;
      } else if (const char* e = std::getenv("SWTB_GROUP_CELLS")) {  // experiments
        if (std::atoll(e) > 0) c->group_cells = std::atoll(e);
      }
      c->rank = opts->rank;
      c->nranks = opts->nranks < 1 ? 1 : opts->nranks;
      if (c->rank < 0 || c->rank >= c->nranks) fail(SWTB_ERR_INPUT, "rank outside [0, nranks)");
      // no id: shard-only, no collective; an id with nranks = 1 runs the
      // collective path on a single-rank communicator
      if (opts->nccl_id) {
        ncclUniqueId id;
        std::memcpy(&id, opts->nccl_id, sizeof(id));
        nccl_check(nccl().comm_init_rank(&c->comm, c->nranks, id, c->rank), "ncclCommInitRank");
      }
    }
  });
  if (s != SWTB_OK) {
    delete c;
    return s;
  }
  *out = c;
  return SWTB_OK;
}

void swtb_ctx_destroy(swtb_ctx* ctx) { delete ctx; }

const char* swtb_last_error(const swtb_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_last_error.c_str();
}

void* swtb_stream(swtb_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

swtb_status swtb_set_caller_stream(swtb_ctx* ctx, void* stream, int enable) {
  if (!ctx) return SWTB_ERR_INPUT;
  return guarded(ctx, [&] {
    CK(cudaSetDevice(ctx->device));
    if (!ctx->ev_caller) CK(cudaEventCreateWithFlags(&ctx->ev_caller, cudaEventDisableTiming));
    ctx->caller = static_cast<cudaStream_t>(stream);
    ctx->has_caller = enable != 0;
  });
}

swtb_status swtb_step(swtb_ctx* ctx, const swtb_batch* batch,
                      const swtb_params* params, const swtb_cfg* cfg,
                      swtb_out* out) {
  if (!ctx) return SWTB_ERR_INPUT;
  return guarded(ctx, [&] {
    if (!batch || !params || !cfg || !out) fail(SWTB_ERR_INPUT, "null argument");
    swtb_out o = *out;
    run_step(ctx, *batch, *params, *cfg, o);
  });
}

swtb_status swtb_get_stats(const swtb_ctx* ctx, swtb_stats* stats) {
  if (!ctx || !stats) return SWTB_ERR_INPUT;
  *stats = ctx->stats;
  return SWTB_OK;
}

int64_t swtb_peak_bytes(const swtb_ctx* ctx) { return ctx ? ctx->peak_bytes : 0; }

void swtb_set_alloc_ceiling(swtb_ctx* ctx, int64_t bytes) {
  if (ctx) ctx->alloc_ceiling = bytes > 0 ? bytes : 0;
}

swtb_status swtb_last_oom(const swtb_ctx* ctx, int64_t* request_bytes,
                          char* tensor, int64_t tensor_cap) {
  if (!ctx || ctx->oom_tensor.empty()) return SWTB_ERR_INPUT;
  if (request_bytes) *request_bytes = ctx->oom_bytes;
  if (tensor && tensor_cap > 0) {
    const size_t n = std::min<size_t>(ctx->oom_tensor.size(), size_t(tensor_cap - 1));
    std::memcpy(tensor, ctx->oom_tensor.data(), n);
    tensor[n] = 0;
  }
  return SWTB_OK;
}

void swtb_set_deterministic(swtb_ctx* ctx, int on) {
  if (ctx) ctx->deterministic = on != 0;
}

void swtb_reset_peak(swtb_ctx* ctx) {
  if (ctx) ctx->peak_bytes = ctx->live_bytes;
}

swtb_status swtb_transducer_loss(swtb_ctx* ctx, const double* scores,
                                 int64_t frames, int64_t labels, int64_t vocab,
                                 const int32_t* y, double* loss,
                                 double* dscores) {
  if (!ctx || !scores || !loss) return SWTB_ERR_INPUT;
  return guarded(ctx, [&] {
    transducer_loss(ctx, scores, frames, labels, vocab, y, loss, dscores);
  });
}

int swtb_parallel_iterations(int64_t frames, int64_t labels, int64_t vocab,
                             int64_t budget_bytes) {
  int r = -1;
  guarded(nullptr, [&] { r = parallel_iterations(frames, labels, vocab, budget_bytes); });
  return r;
}

swtb_status swtb_padded_lengths(int64_t batch, int64_t max_frames,
                                int64_t max_labels, int64_t* t_len,
                                int64_t* u_len) {
  return guarded(nullptr, [&] {
    if (batch < 1 || max_frames < 1 || max_labels < 1)
      fail(SWTB_ERR_INPUT, "all benchmark dimensions must be >= 1");
    padded_lengths(batch, max_frames, max_labels, t_len, u_len);
  });
}

// Reference proj/core/src/bench.cpp:66-115 with the Rng of
// proj/core/include/swt/rng.hpp:14-37 (std::mt19937_64 is fully specified by
// the C++ standard, so identical seeds give identical streams).
swtb_status swtb_synth_inputs(const swtb_synth_cfg* cfg, float* acoustic,
                              float* label, int32_t* labels, int64_t* t_len,
                              int64_t* u_len, float* w_acoustic,
                              float* w_label, float* bias, float* w_out,
                              float* bias_out) {
  return guarded(nullptr, [&] {
    if (!cfg) fail(SWTB_ERR_INPUT, "null config");
    const long long B = cfg->B, T = cfg->T, U = cfg->U, H = cfg->H,
                    HA = cfg->H_A, HL = cfg->H_L, V = cfg->V;
    if (B < 1 || T < 1 || U < 1 || H < 1 || HA < 1 || HL < 1)
      fail(SWTB_ERR_INPUT, "all benchmark dimensions must be >= 1");
    if (V < 2) fail(SWTB_ERR_INPUT, "vocabulary must hold blank plus one label");
    padded_lengths(B, T, U, t_len, u_len);
    std::mt19937_64 gen(cfg->seed);
    auto unit = [&] { return double(gen() >> 11) * 0x1.0p-53; };
    auto fill = [&](float* p, long long n) {
      for (long long i = 0; i < n; ++i) p[i] = float(-0.1 + 0.2 * unit());
    };
    fill(acoustic, B * T * HA);
    for (long long b = 0; b < B; ++b)
      std::fill(acoustic + (b * T + t_len[b]) * HA, acoustic + (b + 1) * T * HA, 0.f);
    const long long R = U + 1;
    fill(label, B * R * HL);
    for (long long b = 0; b < B; ++b)
      std::fill(label + (b * R + u_len[b] + 1) * HL, label + (b + 1) * R * HL, 0.f);
    fill(w_acoustic, H * HA);
    fill(w_label, H * HL);
    fill(bias, H);
    fill(w_out, V * H);
    fill(bias_out, V);
    std::fill(labels, labels + B * U, 0);
    for (long long b = 0; b < B; ++b)
      for (long long i = 0; i < u_len[b]; ++i)
        labels[b * U + i] = int32_t(1 + int64_t(gen() % uint64_t(V - 1)));
  });
}

void swtb_set_profiling(swtb_ctx* ctx, int enable) {
  if (ctx) ctx->prof = enable != 0;
}

swtb_status swtb_get_profile(swtb_ctx* ctx, double* ms, int64_t* launches,
                             int reset) {
  if (!ctx) return SWTB_ERR_INPUT;
  for (int i = 0; i < SWTB_NUM_STAGES; ++i) {
    if (ms) ms[i] = ctx->prof_ms[i];
    if (launches) launches[i] = ctx->prof_n[i];
    if (reset) {
      ctx->prof_ms[i] = 0;
      ctx->prof_n[i] = 0;
    }
  }
  return SWTB_OK;
}

swtb_status swtb_nccl_unique_id(void* out) {
  return guarded(nullptr, [&] {
    if (!out) fail(SWTB_ERR_INPUT, "null output");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}

swtb_status swtb_debug_gemm(swtb_ctx* ctx, int precision, int a_mn, int b_mn,
                            const void* A, int64_t lda, const void* B,
                            int64_t ldb, int64_t M, int64_t N, int64_t K,
                            float* out, int64_t ldo, int accumulate) {
  if (!ctx) return SWTB_ERR_INPUT;
  return guarded(ctx, [&] {
    CK(cudaSetDevice(ctx->device));
    const Prec p = precision == SWTB_PREC_TF32   ? Prec::kTF32
                   : precision == SWTB_PREC_FP16 ? Prec::kFP16
                                                 : Prec::kBF16;
    if (p == Prec::kFP16 && accumulate) fail(SWTB_ERR_INPUT, "fp16 debug GEMM: store only");
    const Mat a{A, a_mn ? K : M, a_mn ? M : K, lda};
    const Mat b{B, b_mn ? K : N, b_mn ? N : K, ldb};
    if (accumulate)
      gemm_atomic(p, a_mn != 0, b_mn != 0, a, b, int(M), int(N), int(K), out,
                  ldo, ctx->stream);
    else
      gemm_store(p, a_mn != 0, b_mn != 0, a, b, int(M), int(N), int(K), out,
                 ldo, nullptr, nullptr, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
