// SPDX-License-Identifier: Apache-2.0
//
// Host-side declarations of the libswt_b200 kernel launchers. Everything the
// engine (swtb_engine.cpp) launches goes through these; no kernel is launched
// anywhere else.

#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace swtb {

// One sample of a launch group (arrays of these live in device memory).
struct SampleDesc {
  int T;          // valid frames T_b
  int U1;         // valid label rows U_b + 1
  int a_row0;     // first packed acoustic row (P_A / ga / ha_pack)
  int l_row0;     // first packed label row   (P_L / gl / hl_pack)
  long long lat;  // offset of the sample's diagonal-major lattice arrays
  long long lab;  // offset of the sample's labels (b * U)
  int b;          // batch index
  int tile0;      // first 128-cell tile of the sample
  int n_tb;       // tiles along t (16 frames each)
  int n_ub;       // tiles along u (8 label rows each)
};

// A 128-cell tile: frames [t0, t0+16) x label rows [u0, u0+8) of sample s.
// Cell r of the tile is (t0 + r/8, u0 + r%8).
struct TileDesc {
  int s, t0, u0, pad;
};

constexpr int kTileT = 16;
constexpr int kTileU = 8;

// Lattice value convention: lp_blank / lp_label, alpha, beta and logZ are
// kept in log2 units (bits = nats * log2 e), so the wavefront's log-add-exp
// is log2(2^a + 2^b) = max + log2(1 + 2^-|a-b|), straight MUFU ex2 / lg2 with
// no scaling; lse stays in nats. Consumers convert (x * ln 2) where needed.
//
// Diagonal-major ("skewed") lattice index: the cells of anti-diagonal
// d = t + u are contiguous, so the wavefront kernel reads/writes coalesced.
// Diagonals are `lat_pitch(U1)` floats apart (U1 rounded up to 4), so every
// diagonal starts 16-byte aligned and a run of diagonals can be moved by one
// bulk copy.
__host__ __device__ inline int lat_pitch(int U1) { return (U1 + 3) & ~3; }
__host__ __device__ inline long long skew(long long lat, int U1, int t, int u) {
  return lat + (long long)(t + u) * lat_pitch(U1) + u;
}
__host__ __device__ inline long long skew_size(int T, int U1) {
  return (long long)(T + U1 - 1) * lat_pitch(U1);
}
// Diagonals per bulk-copied chunk of the warp wavefront kernel, and the slack
// (in diagonals of the group's widest pitch) kept before the first and after
// the last sample of a group's lattice arrays, so a chunk that straddles a
// sample's ends still reads inside the allocation.
constexpr int kLatChunk = 8;
__host__ __device__ inline long long lat_slack(int max_U1) {
  return (long long)kLatChunk * lat_pitch(max_U1);
}

// Operand view of a row-major 2D buffer for TMA: `rows` x `cols` valid
// elements, leading dimension `ld` elements (ld * elem % 16 == 0).
struct Mat {
  const void* ptr;
  long long rows, cols, ld;
};

// A device-built list of active 128-row tiles (tile indices, ascending)
// that a row-mapped GEMM walks instead of every tile: entries
// list[0, n), n = clamp(*count - offset, 0, max) (gemm.cuh, kRowMap);
// list == nullptr: every tile.
struct RowMap {
  const int* list = nullptr;
  const int* count = nullptr;
  int offset = 0;
  int max = 0;
};

// operand element format of the output-layer GEMMs (and their slabs)
enum class Prec { kBF16 = 0, kTF32 = 1, kFP16 = 2 };

int num_sms(int device);
// kernels this thread has launched through the launchers below
long long launch_count();
// Persistent GEMMs launched by this thread use (#SMs - n) CTAs until reset.
void set_gemm_sm_reserve(int n);
// Deterministic accumulation: while set, split-K GEMMs (gemm_atomic,
// gemm_dw_db) and the db_Z column sums store per-split partials in `ws` and
// add them to their outputs in a fixed order (no fp32 atomics), so repeated
// steps are bitwise identical. nullptr restores the atomic form.
void set_split_workspace(float* ws, size_t floats);
// floats the workspace needs (worst case over SM reserves) when the joint
// GEMMs reduce over <= K_joint rows and dW_O over <= K_dw slab rows
size_t split_workspace_floats(int device, int V, int H, int H_A, int H_L,
                              long long K_joint, long long K_dw, bool tf32);
void launch_split_reduce(const float* part, int S, long long n, long long stride,
                         float* out, cudaStream_t st);
// Deterministic dW_O / db_O: while set, gemm_dw_db adds split s's partial
// into slice s of `acc` ([slices][V][H] then [slices][V], zeroed by the
// caller) with plain read-modify-writes (each element has one owner per
// launch); the caller reduces the slices once per step in a fixed order.
void set_dw_accumulator(float* acc, int slices);
// slices a step needs: the largest split count of its dW_O launches
int dw_acc_slices(int device, int V, long long K_dw, bool tf32);

// ---- elementwise / gather ----
void launch_convert_pad(const float* src, long long rows, long long cols,
                        long long src_ld, void* dst, long long dst_ld,
                        Prec prec, cudaStream_t st, void* dst_lo = nullptr);
void launch_zslab(const float* pa, const float* pl, long long ldp, int H,
                  const TileDesc* tiles, const SampleDesc* samples,
                  int n_tiles, void* z, long long ldz, Prec prec,
                  cudaStream_t st);
void launch_lattice(const SampleDesc* samples, int n_samples,
                    const int* labels, const double* lpb, const double* lpy,
                    double* alpha, double* beta, double* logz,
                    float* loss_out /* [B] indexed by sample.b */,
                    int max_U1, cudaStream_t st);
// Per-cell logit-gradient scalars (so overwrites lse in place; eb, ey):
// run after both sweeps of the samples' lattices. weights: optional
// per-sample loss weights [B] (>= 0, indexed by sample.b) scaling dh.
// tile_flags (optional, zeroed by the caller): flag[tile] = 1 for every
// 128-cell tile of the samples holding a cell whose log2 bound on |dh|,
// log2(alpha beta / P) + lmp (lmp: log2 of the cell's largest softmax
// probability, FwdLseArgs.lmp; 0 when null), exceeds thr — the tiles whose
// dh is not all zero.
void launch_edge(const SampleDesc* samples, int n_samples, int max_D,
                 const double* lpb, const double* lpy, const double* alpha,
                 const double* beta, const double* logz, float* lse_so,
                 float* eb, float* ey, cudaStream_t st,
                 const float* weights = nullptr, uint8_t* tile_flags = nullptr,
                 float thr = 0.f, const float* lmp = nullptr);
// list[0, n) = ascending indices of the nonzero flags[0, n_flags); *count = n;
// *total += n (optional). One CTA, on st.
void launch_compact_tiles(const uint8_t* flags, int n_flags, int* list, int* count,
                          unsigned long long* total, cudaStream_t st);
// CTAs (= SMs it may occupy) one launch_lattice of this shape uses.
int lattice_launch_ctas(int n_samples, int max_U1);
// ga/gl are emitted as bf16 (hi, lo) pairs for the split joint GEMMs.
// Rows [ra0, ra0 + R_A) / [rl0, rl0 + R_L) of the joint batch's ga / gl.
void launch_reduce_partials(const float* part_a, const float* part_l,
                            const SampleDesc* samples, int n_samples,
                            const int* row_sample_a, const int* row_sample_l,
                            int ra0, int rl0, int R_A, int R_L, int H, long long ldp,
                            __nv_bfloat16* ga_hi, __nv_bfloat16* ga_lo,
                            __nv_bfloat16* gl_hi, __nv_bfloat16* gl_lo,
                            float* dbias, cudaStream_t st,
                            const uint8_t* active = nullptr);
// zbar[r, :] = mean over min(T_b, nsamp) evenly spaced frames of
// tanh(P_A[a0 + t] + P_L[r]) for the R label rows of a joint batch
// (row_info[2r] = a0, the sample's first P_A row; row_info[2r+1] = T_b);
// fp16, ldz >= H columns, zero beyond H: the fp16 forward's correction input.
void launch_zmean(const float* pa, const float* pl, long long ldp, int H,
                  const int* row_info, int R, int nsamp, __half* zbar, long long ldz,
                  cudaStream_t st);
// dst[r, c] = split(src[row_src ? row_src[r] : r, c]) for c < cols, else 0.
void launch_split_rows(const float* src, long long rows, long long cols,
                       long long src_ld, const long long* row_src,
                       __nv_bfloat16* hi, __nv_bfloat16* lo, long long dst_ld,
                       cudaStream_t st);

// ---- GEMM-based stages (all tcgen05) ----
// C[m, n] = A[m, :] . B[n, :]; fp32 store (+ bias[n]) into out[row_map(m)].
// With A_lo/B_lo (bf16 only) the operands are (hi, lo) split pairs and the
// kernel forms hi*hi + hi*lo + lo*hi: float32-grade joint-network GEMMs.
void gemm_store(Prec prec, bool a_mn, bool b_mn, const Mat& A, const Mat& B,
                int M, int N, int K, float* out, long long ldo,
                const float* bias, const long long* row_map, cudaStream_t st,
                const Mat* A_lo = nullptr, const Mat* B_lo = nullptr);
// out[m, n] += C[m, n] via split-K fp32 atomics.
void gemm_atomic(Prec prec, bool a_mn, bool b_mn, const Mat& A, const Mat& B,
                 int M, int N, int K, float* out, long long ldo,
                 cudaStream_t st, const Mat* A_lo = nullptr,
                 const Mat* B_lo = nullptr);

// dW_O += dh^T z and db_O += column sums of dh (tensor-core row sums of the
// MN-major dh^T operand), split-K over the slab rows; CTA pairs.
void gemm_dw_db(Prec prec, const Mat& dh, const Mat& z, int V, int H, int rows,
                float* dw_out, float* db_out, int* bad, cudaStream_t st,
                const RowMap& map = RowMap{});

struct FwdLseArgs {
  const TileDesc* tiles;
  const SampleDesc* samples;
  const int* labels;
  const float* bias_out;
  int V;
  float* lse;
  double* lpb;  // log-probabilities of the blank / label edges (f64: the
  double* lpy;  // wavefront accumulates in f64 and reads them directly)
  // optional per-label-row bias [joint-batch label rows][ld_bias_rows]
  // (b_O + the row's W_O-rounding correction); bias_out when null
  const float* bias_rows = nullptr;
  long long ld_bias_rows = 0;
  // optional x slab (16-bit operand modes): x[row, v] = h[row, v] - m[row,
  // v / 32] as fp16, rows in tile order, in 8-row strips of 8 ld_x elements
  // (the bytes the strip's rows occupy in the row-major dh slab, ld = ld_x):
  // inside a strip, the 16-B piece of row rr holding columns [8 k, 8 k + 8)
  // sits at piece index 8 k + rr (so 8 rows' pieces are one 128-B line); m, the maxima
  // of the 32-column blocks, in xoff [rows][ld_xoff] (ld_xoff a multiple of
  // 8), block b at slot 8 (b / 8) + 4 (b % 2) + (b % 8) / 2: each epilogue
  // thread writes its column half's 4 blocks of a 256-column chunk at once
  void* xs = nullptr;
  long long ld_x = 0;
  float* xoff = nullptr;
  long long ld_xoff = 0;
  // optional: log2 of the cell's largest softmax probability, (max_v h -
  // lse) log2 e, at the skewed lattice index (the zero-tile test's bound)
  float* lmp = nullptr;
};
// w_lo: optional low half of a split W_O (the GEMM then adds z * W_lo^T)
void gemm_fwd_lse(Prec prec, const Mat& z, const Mat& w_out, int rows, int V,
                  int H, const FwdLseArgs& a, cudaStream_t st,
                  const Mat* w_lo = nullptr);

struct BwdDhArgs {
  const TileDesc* tiles;
  const SampleDesc* samples;
  const int* labels;
  const float* bias_out;
  int V;
  const float* so;  // per-cell scalars from edge_kernel (skewed layout)
  const float* eb;
  const float* ey;
  void* dh;
  long long ld_dh;
  int* bad;
  // active tiles only (fp16 zero-tile skip): z rows of the listed tiles are
  // read, dh is written in list order (compacted slab rows, dh_rows of them;
  // 0 = the GEMM's rows)
  RowMap map;
  long long dh_rows = 0;
};
void gemm_bwd_dh(Prec prec, const Mat& z, const Mat& w_out, int rows, int V,
                 int H, const BwdDhArgs& a, cudaStream_t st,
                 const Mat* w_lo = nullptr);

// largest x slab row pitch (elements) launch_x_to_dh handles (registers
// hold a whole 8-row strip per CTA)
constexpr long long kXMaxLd = 4096;
// dh from the forward's x slab, in place (fp16 x -> dh in the operand
// precision, same 2-byte slots): dh[row, v] = 2^((x + xoff) log2 e + s) with
// the blank / label edge columns replaced by eb / ey and padded cells 0 —
// the values gemm_bwd_dh's epilogue forms from recomputed logits.
void launch_x_to_dh(void* xs, long long ld_x, const float* xoff, long long ld_xoff,
                    long long rows, const TileDesc* tiles, const SampleDesc* samples,
                    const int* labels, int V, const float* so, const float* eb,
                    const float* ey, Prec prec, int* bad, cudaStream_t st);

struct GateArgs {
  const TileDesc* tiles;
  const SampleDesc* samples;
  const void* z;
  long long ld_z;
  int H;
  float* part_a;  // [n_tiles][16][ldp]
  float* part_l;  // [n_tiles][8][ldp]
  long long ldp;
  // active tiles only: dh rows compacted (list order), z / partials at the
  // real tiles; z_rows = rows of the z view (the part), 0 = the GEMM's rows
  RowMap map;
  long long z_rows = 0;
};
void gemm_dz_gate(Prec prec, const Mat& dh, const Mat& w_out, int rows, int V,
                  int H, const GateArgs& a, cudaStream_t st,
                  const Mat* w_lo = nullptr);

// ---- batched comparator: passes over materialized fp32 scores ----
// rows in tile order (cell r of tile k = row 128 k + r), ld floats apart.
void launch_tile_scores_lse(const float* scores, long long ld, long long rows,
                            const TileDesc* tiles, const SampleDesc* samples,
                            const int* labels, int V, float* lse, double* lpb,
                            double* lpy, cudaStream_t st);
// dh in the GEMM operand precision, columns [V, V_pad) and padded cells 0.
void launch_tile_dscores(const float* scores, long long ld, long long rows,
                         const TileDesc* tiles, const SampleDesc* samples,
                         const int* labels, int V, long long V_pad,
                         const float* so, const float* eb, const float* ey,
                         void* dh, long long ld_dh, Prec prec, int* bad,
                         cudaStream_t st);

// ---- f^W on explicit scores (swtb_transducer_loss) ----
void launch_scores_lse(const double* scores, int T, int U1, int V,
                       const int* y, const SampleDesc* sd, float* lse,
                       double* lpb, double* lpy, cudaStream_t st);
void launch_scores_grad(const double* scores, int T, int U1, int V,
                        const int* y, const SampleDesc* sd, const float* lse,
                        const double* alpha, const double* beta,
                        const double* logz, double* dscores, cudaStream_t st);

}  // namespace swtb
