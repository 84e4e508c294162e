// SPDX-License-Identifier: Apache-2.0
//
// libswt_b200 device code: the GEMM epilogues that carry the transducer
// math, plus the non-GEMM kernels of the per-group pipeline.
//
// Reference semantics (paths relative to the reference tree, proj/core/):
//   joint forward  z = tanh(W_A a + W_L l + b)        src/compute.cpp:45-67
//   output forward h = W_O z + b_O                    src/compute.cpp:69-90
//   log-softmax    lse = max + log sum exp(h - max)   include/swt/tensor.hpp:397-405
//   alpha/beta     log-space recursions               src/loss.cpp:41-81
//   loss           -beta[0,0]                         src/loss.cpp:155-162
//   dh             occ*softmax - blank/label edges    src/loss.cpp:83-132
//   output bwd     dz = dh W_O, dW_O += dh^T z, db_O  src/compute.cpp:92-122
//   joint bwd      g = dz (1-z^2), ga/gl sums, ...    src/compute.cpp:124-192

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm.cuh"
#include "swtb_kernels.h"

namespace swtb {

namespace {

constexpr double kNegInfD = -__builtin_huge_val();
constexpr double kL2Ed = 1.4426950408889634;  // log2(e)
constexpr double kLn2d = 0.6931471805599453;   // ln(2)

__device__ __forceinline__ float round_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Operand element formats of the output-layer GEMMs (Prec): 0 bf16,
// 1 fp32 read as tf32, 2 fp16. pack2 / bits give the 16-bit formats' raw
// storage (two elements per 32-bit word, low half first).
template <int kFmt>
struct OpElem;
template <>
struct OpElem<0> {
  using T = __nv_bfloat16;
  __device__ static T cvt(float x) { return __float2bfloat16_rn(x); }
  __device__ static float back(T x) { return __bfloat162float(x); }
  __device__ static uint32_t pack2(float a, float b) {
    __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&p);
  }
  __device__ static unsigned short bits(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
  __device__ static float2 unpack2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  }
};
template <>
struct OpElem<1> {
  using T = float;
  __device__ static T cvt(float x) { return round_tf32(x); }
  __device__ static float back(T x) { return x; }
};
template <>
struct OpElem<2> {
  using T = __half;
  __device__ static T cvt(float x) { return __float2half_rn(x); }
  __device__ static float back(T x) { return __half2float(x); }
  __device__ static uint32_t pack2(float a, float b) {
    __half2 p = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&p);
  }
  __device__ static unsigned short bits(float x) {
    return __half_as_ushort(__float2half_rn(x));
  }
  __device__ static float2 unpack2(uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
};

struct CellInfo {
  int t, u, s;
  bool valid;
};

__device__ __forceinline__ CellInfo cell_of(const TileDesc* tiles,
                                            const SampleDesc* samples,
                                            int m0, int row, SampleDesc& sd) {
  const TileDesc td = tiles[m0 / kGemmBM];
  sd = samples[td.s];
  CellInfo c;
  c.t = td.t0 + row / kTileU;
  c.u = td.u0 + row % kTileU;
  c.s = td.s;
  c.valid = c.t < sd.T && c.u < sd.U1;
  return c;
}

// ---------------------------------------------------------------------------
// Epilogues

struct EpiNoSmem {
  static constexpr int kSmemBytes = 0;
  __device__ void setup(uint8_t*, int, const CUtensorMap*) {}
  __device__ void prefetch(const GemmUnit&, int) {}
  __device__ void finish(uint8_t*, int) {}
};

// bias (padded to a multiple of 32 floats) added to 32 accumulator columns
__device__ __forceinline__ void add_bias32(float (&v)[32], const float* bias) {
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 b = __ldg(b4 + q);
    v[4 * q] += b.x;
    v[4 * q + 1] += b.y;
    v[4 * q + 2] += b.z;
    v[4 * q + 3] += b.w;
  }
}

// out[row_map(m), n] = acc (+ bias[n])
template <int BN, bool F16 = false>
struct EpiStore : EpiNoSmem {
  static constexpr bool kF16 = F16;
  float* out;
  long long ldo;
  int M, N;
  const float* bias;
  const long long* row_map;
  long long orow;
  bool live;

  __device__ void begin(const GemmUnit& g, int row) {
    const int m = g.m0 + row;
    live = m < M;
    orow = live ? (row_map ? row_map[m] : (long long)m) : 0;
  }
  __device__ void chunk(const GemmUnit&, int n0, int, int half, uint32_t taddr) {
#pragma unroll 1
    for (int c = 32 * half; c < BN && n0 + c < N; c += 64) {
      float v[32];
      tmem_ld32(taddr + c, v);
      if (!live) continue;
      float* dst = out + orow * ldo + n0 + c;
      const int nv = min(32, N - (n0 + c));
      if (bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) v[j] += bias[n0 + c + j];
      }
      if (nv == 32 && (ldo % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) dst[j] = v[j];
      }
    }
  }
  __device__ void end(const GemmUnit&, int) {}
};

// out[m, n] += acc   (split-K partial sums; fp32 vector reductions in L2).
// Deterministic form (split_stride > 0): split s stores its partial to
// out + s * split_stride and an ordered reduction adds the splits later, so
// repeated steps are bitwise identical (reference acceptance criterion 10).
template <int BN>
struct EpiAtomic : EpiNoSmem {
  float* out;
  long long ldo;
  int M, N;
  long long split_stride = 0;
  bool split_accumulate = false;  // deterministic form: += into the slice
  bool live;
  int m;

  __device__ void begin(const GemmUnit& g, int row) {
    m = g.m0 + row;
    live = m < M;
  }
  __device__ void chunk(const GemmUnit& g, int n0, int, int half, uint32_t taddr) {
#pragma unroll 1
    for (int c = 32 * half; c < BN && n0 + c < N; c += 64) {
      float v[32];
      tmem_ld32(taddr + c, v);
      if (!live) continue;
      float* dst = out + g.split * split_stride + (long long)m * ldo + n0 + c;
      const int nv = min(32, N - (n0 + c));
      if (split_stride) {
        if (nv == 32 && (ldo % 4) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (split_accumulate) {
              const float4 p = *reinterpret_cast<const float4*>(dst + j);
              o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
            }
            *reinterpret_cast<float4*>(dst + j) = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) dst[j] = split_accumulate ? dst[j] + v[j] : v[j];
        }
      } else if (nv == 32 && (ldo % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          atomicAdd(reinterpret_cast<float4*>(dst + j),
                    make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) atomicAdd(dst + j, v[j]);
      }
    }
  }
  __device__ void end(const GemmUnit&, int) {}
};

// dW_O += dh^T z (EpiAtomic) plus db_O: the GEMM also runs the all-ones
// MMA on A = dh^T, so TMEM holds sum over the unit's cells of dh[cell, v]
// for each row v — the reference's db_O accumulation (compute.cpp:118-121)
// on the tensor core instead of column sums in the dh epilogue.
template <int BN, bool F16 = false>
struct EpiAtomicDb : EpiAtomic<BN> {
  static constexpr int kOnesCols = 16;
  static constexpr bool kF16 = F16;
  // one N chunk per unit: the two chunk units of a (row group, split) run
  // concurrently, so the dh rows come from DRAM once (with whole-row units
  // each unit re-streamed its dh rows once per chunk: 1.7x the bytes)
  static constexpr bool kChunkUnits = true;
  // K = slab rows: only the listed (active) tiles' rows; dh compacted, z real
  static constexpr int kRowMap = 3;
  RowMap map;
  float* db;
  long long db_stride = 0;  // deterministic form: per-split partial rows
  int* bad;
  __device__ void ones(const GemmUnit& g, int row, int half, uint32_t taddr) {
    const float v = tmem_ld1(taddr);  // warp-collective: both halves load
    const int m = g.m0 + row;
    if (half == 0 && m < this->M) {
      if (db_stride)
        db[g.split * db_stride + m] += v;  // per-split accumulator slice
      else
        atomicAdd(db + m, v);
      if (!isfinite(v)) atomicOr(bad, 1);
    }
  }
};

// Forward f^O epilogue: bias, online log-sum-exp over the whole vocabulary
// row, gathers of the blank and next-label logits. Writes 3 floats per
// lattice cell (lse, lp_blank, lp_label); the logits never leave TMEM. The
// two column halves of a row are merged through shared memory at row end.
template <int BN, bool F16 = false, bool kStoreX = false>
struct EpiFwdLse {
  // per-label-row biases (a.bias_rows): the chunk's 8 rows x BN columns are
  // staged in shared memory by cp.async one chunk ahead (double-buffered):
  // a tile's 128 cells use 8 label rows, so every bias value is read by 16
  // threads — from L2 directly the loads stalled the epilogue. Each column
  // half (the 4 warps taking the even / odd 32-column blocks) stages its own
  // 8 x BN/2 columns and syncs on its own 128-thread barrier, so the halves
  // do not wait for each other.
  static constexpr int kPartBytes = 2 * 128 * 16;
  static constexpr int kBiasPitch = BN / 2 + 4;  // floats; +16 B: conflict-free rows
  static constexpr int kBiasBuf = 2 * kTileU * kBiasPitch * 4;  // both halves
  // kStoreX: the logits leave the kernel as fp16 block-relative values
  // x = h - max(block of 32 columns) plus the block maxima, so the backward
  // forms dh elementwise (x_to_dh_kernel) instead of recomputing the logits
  // with a second GEMM. x goes straight from registers to HBM in the strip-
  // interleaved layout (FwdLseArgs): every warp store instruction writes four
  // whole 128-B lines, no shared-memory staging.
  static constexpr int kSmemBytes = kPartBytes + 2 * kBiasBuf;
  static constexpr bool kF16 = F16;
  static constexpr bool kEarlyRelease = true;
  FwdLseArgs a;  // a.bias_out padded to a multiple of 32 floats
  float mx, sum, hb, hy;
  int y, half, tid;
  bool valid;
  long long idx;
  float4* part;  // [2 parity][128 rows] (m, s, hb, hy) of half 1
  int units;
  uint32_t bsm;  // the two staged bias-row buffers
  int kc;        // chunks processed by this CTA
  long long cur_r0, cur_rmax, nxt_r0, nxt_rmax;  // tile's label rows, clamp
  bool nxt_ok;
  // the next unit's row state, loaded one unit ahead (prefetch): begin()
  // then finds it in registers instead of waiting on a chain of dependent
  // loads (tile -> sample -> label, lattice index)
  int n_y;
  bool n_valid, have_next;
  long long n_idx;

  __device__ void load_row(const GemmUnit& g, int row, bool& o_valid, int& o_y,
                           long long& o_idx) {
    SampleDesc sd;
    const CellInfo c = cell_of(a.tiles, a.samples, g.m0, row, sd);
    o_valid = c.valid;
    o_y = (c.valid && c.u < sd.U1 - 1) ? a.labels[sd.lab + c.u] : -1;
    o_idx = c.valid ? skew(sd.lat, sd.U1, c.t, c.u) : 0;
  }

  __device__ void tile_rows(const GemmUnit& g, long long& r0, long long& rmax) {
    const TileDesc td = a.tiles[g.m0 / kGemmBM];
    const SampleDesc sd = a.samples[td.s];
    r0 = sd.l_row0 + td.u0;
    rmax = sd.l_row0 + sd.U1 - 1;
  }
  // this thread's share (2 x 16 B) of its half's bias rows [r0, r0 + 8) x
  // (the half's BN/2 columns of [n0, n0 + BN): blocks 32 half + 64 k)
  __device__ uint32_t hbuf(int buf) const {
    return bsm + buf * kBiasBuf + half * (kBiasBuf / 2);
  }
  __device__ void issue(long long r0, long long rmax, int n0, int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int f = (tid & 127) + 128 * i;
      const int r = f / (BN / 8), c4 = f % (BN / 8);  // c4: float4 of the half
      const uint32_t dst = hbuf(buf) + (r * kBiasPitch + c4 * 4) * 4;
      const long long srow = r0 + r < rmax ? r0 + r : rmax;
      const int col = n0 + 32 * half + 64 * (c4 >> 3) + 4 * (c4 & 7);
      if (col < a.ld_bias_rows)
        cp_async16(dst, a.bias_rows + srow * a.ld_bias_rows + col);
    }
    cp_async_commit();
  }
  __device__ void prefetch(const GemmUnit& gn, int row) {
    load_row(gn, row, n_valid, n_y, n_idx);
    have_next = true;
    if (a.bias_rows) {
      tile_rows(gn, nxt_r0, nxt_rmax);
      nxt_ok = true;
    }
  }
  int xk;                    // x blocks this thread stored in the current chunk
  float xo[BN / 64];         // block maxima of the current chunk
  __device__ void setup(uint8_t* smem, int t, const CUtensorMap*) {
    part = reinterpret_cast<float4*>(smem);
    bsm = smem_u32(smem + kPartBytes);
    tid = t;
    half = tid >> 7;
    units = 0;
    kc = 0;
    nxt_ok = false;
    have_next = false;
  }
  __device__ void begin(const GemmUnit& g, int row) {
    if (have_next) {
      valid = n_valid;
      y = n_y;
      idx = n_idx;
      have_next = false;
      if (a.bias_rows) {  // prefetch() loaded the tile's label rows too
        cur_r0 = nxt_r0;
        cur_rmax = nxt_rmax;
      }
    } else {
      load_row(g, row, valid, y, idx);
      if (a.bias_rows) tile_rows(g, cur_r0, cur_rmax);
    }
    if (a.bias_rows) nxt_ok = false;  // set again by prefetch() if a next unit exists
    mx = -INFINITY;
    sum = 0.f;
    hb = 0.f;
    hy = 0.f;
  }
  template <class Rel>
  __device__ void chunk(const GemmUnit& g, int n0, int row, int hf, uint32_t taddr, Rel&& rel) {
    constexpr float kL2E = 1.4426950408889634f;
    const float2 l2e2 = make_float2(kL2E, kL2E);
    uint32_t bs = 0;  // this row's staged bias row (shared address)
    if (a.bias_rows) {
      if (kc == 0) issue(cur_r0, cur_rmax, n0, 0);  // the CTA's first chunk
      cp_async_wait_all();  // this chunk's rows (issued a chunk ahead)
      half_bar(half);       // ... from every thread of the half; its other buffer is free
      if (n0 + BN < a.V)
        issue(cur_r0, cur_rmax, n0 + BN, (kc + 1) & 1);
      else if (nxt_ok)
        issue(nxt_r0, nxt_rmax, 0, (kc + 1) & 1);
      bs = hbuf(kc & 1) + (row & (kTileU - 1)) * kBiasPitch * 4;
      ++kc;
    }
    xk = 0;
    tmem_blocks<BN>(taddr, hf, a.V - n0, [&](int c, float (&v)[32]) {
      const int base = n0 + c;
      const float4* b4 = reinterpret_cast<const float4*>(a.bias_out + base);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        // c = 32 half + 64 k: the half's staged columns 32 k + 4 q
        const float4 b = bs ? lds_v4(bs + ((c >> 6) * 32 + 4 * q) * 4) : __ldg(b4 + q);
        const float2 x0 = add2(make_float2(v[4 * q], v[4 * q + 1]), make_float2(b.x, b.y));
        const float2 x1 = add2(make_float2(v[4 * q + 2], v[4 * q + 3]), make_float2(b.z, b.w));
        v[4 * q] = x0.x;
        v[4 * q + 1] = x0.y;
        v[4 * q + 2] = x1.x;
        v[4 * q + 3] = x1.y;
      }
      if (base + 32 > a.V) {  // vocabulary tail (warp-uniform)
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (base + j >= a.V) v[j] = -INFINITY;
      }
      if (base == 0) hb = v[0];
      if ((unsigned)(y - base) < 32u) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (base + j == y) hy = v[j];
      }
      float m[11];
#pragma unroll
      for (int k = 0; k < 10; ++k) m[k] = max3(v[3 * k], v[3 * k + 1], v[3 * k + 2]);
      m[10] = fmaxf(v[30], v[31]);
      const float bm = max3(max3(m[0], m[1], m[2]), max3(m[3], m[4], m[5]),
                            max3(max3(m[6], m[7], m[8]), m[9], m[10]));
      if constexpr (kStoreX) store_x(g, row, base, v, bm);
      const float nm = fmaxf(mx, bm);
      const float2 nml = make_float2(-nm * kL2E, -nm * kL2E);
      float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 e0 = fma2(make_float2(v[4 * q], v[4 * q + 1]), l2e2, nml);
        const float2 e1 = fma2(make_float2(v[4 * q + 2], v[4 * q + 3]), l2e2, nml);
        s0 = add2(s0, make_float2(ex2(e0.x), ex2(e0.y)));
        s1 = add2(s1, make_float2(ex2(e1.x), ex2(e1.y)));
      }
      const float2 st = add2(s0, s1);
      const float carry = (mx == -INFINITY) ? 0.f : sum * ex2(fmaf(mx, kL2E, nml.x));
      sum = carry + (st.x + st.y);
      mx = nm;
    }, rel);
    if constexpr (kStoreX) {
      // this thread's BN/64 block maxima of the chunk, one vector store; slot
      // order per chunk: the half's blocks (launch_x_to_dh's xoff layout)
      float4* o = reinterpret_cast<float4*>(a.xoff + (long long)(g.m0 + row) * a.ld_xoff +
                                            (n0 / BN) * (BN / 32) + hf * (BN / 64));
      static_assert(BN / 64 == 4, "one float4 of maxima per chunk and half");
      *o = make_float4(xo[0], xo[1], xo[2], xo[3]);
    }
  }
  __device__ void end(const GemmUnit&, int row) {
    const uint32_t p = smem_u32(part + (units & 1) * 128 + row);
    if (half == 1) sts_v4(p, mx, sum, hb, hy);
    // only the two warps of this TMEM lane quarter (one per column half)
    // exchange: a 64-thread named barrier instead of all 256 epilogue threads
    named_bar_sync(4 + (row >> 5), 64);
    if (half == 0 && valid) {
      const float4 o = lds_v4(p);
      const float m = fmaxf(mx, o.x);
      const float s = (mx == -INFINITY ? 0.f : sum * __expf(mx - m)) +
                      (o.x == -INFINITY ? 0.f : o.y * __expf(o.x - m));
      const float l = m + logf(s);
      a.lse[idx] = l;
      if (a.lmp) a.lmp[idx] = (m - l) * 1.4426950408889634f;  // log2 max_v softmax
      // lattice operands in log2 units (bits), see swtb_kernels.h
      a.lpb[idx] = double(hb - l) * kL2Ed;
      if (y >= 0) a.lpy[idx] = double((((y >> 5) & 1) ? o.w : hy) - l) * kL2Ed;
    }
    ++units;
  }
  // x = h - bm for the block's 32 columns of this row: four 16-B pieces,
  // piece q of block cb of row r at strip r / 8, slot (4 cb + q) 8 + r % 8
  __device__ void store_x(const GemmUnit& g, int row, int base, const float (&v)[32],
                          float bm) {
    const float b = bm == -INFINITY ? 0.f : bm;
    const long long r = (long long)g.m0 + row;
    uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(a.xs) + (r >> 3) * (16 * a.ld_x)) +
                 (base >> 5) * 32 + (r & 7);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      auto pk = [&](int j) {
        __half2 h2 = __floats2half2_rn(v[8 * q + j] - b, v[8 * q + j + 1] - b);
        return *reinterpret_cast<uint32_t*>(&h2);
      };
      dst[8 * q] = make_uint4(pk(0), pk(2), pk(4), pk(6));
    }
    // k-th block of this chunk (xk folds to a constant in the unrolled loop)
#pragma unroll
    for (int k = 0; k < BN / 64; ++k) xo[k] = xk == k ? b : xo[k];
    ++xk;
  }
  __device__ void finish(uint8_t*, int) {}
};

// Backward epilogue on the recomputed logits: forms dh in registers,
//   dh[v] = 2^((h_v + b_v) log2(e) + s)       s = alpha + beta - logZ - lse log2(e)
// for every column, then patches the two edge columns of the cell with the
// precomputed blank / label edge values (edge_kernel; reference
// src/loss.cpp:100-127). The hot loop is branch-free packed fp32x2 math +
// MUFU.EX2. Each warp stages its 32x32 block of dh in smem in the slab
// precision (the patches land there) and one lane TMA-stores it to the dh
// slab as full 32-column row segments. db_O is not summed here: the dW_O
// GEMM gets it from the tensor core (EpiAtomicDb).
template <int BN, int kFmt>
struct EpiBwdDh {
  static constexpr bool kTF32 = kFmt == 1;
  static constexpr bool kF16 = kFmt == 2;
  using E = OpElem<kFmt>;
  // per warp two staging tiles (fp32 128B rows / 16-bit 64B rows), used in
  // turn: a block's smem writes need not wait for the previous block's TMA
  // store to finish reading its tile (16-bit: the second tile costs no
  // mainloop stage)
  static constexpr int kWarpBytes = kTF32 ? 4096 : 2048;
  static constexpr int kTiles = kTF32 ? 1 : 2;
  static constexpr int kSmemBytes = 8 * kTiles * kWarpBytes;
  BwdDhArgs a;  // a.bias_out padded to a multiple of 32 floats
  // active tiles only: z read at the real tile, dh written at the compacted row
  static constexpr int kRowMap = 1;
  RowMap map;
  float so;     // s (log2 units)
  float d_b, d_y;
  int y;
  uint8_t* wsm;
  const CUtensorMap* tm;
  int bad;
  int nblk;  // blocks this thread has staged

  // the next unit's row scalars, loaded one unit ahead (prefetch): begin()
  // then finds them in registers instead of waiting on a chain of dependent
  // global loads (tile -> sample -> lattice index -> scalars)
  float n_so, n_db, n_dy;
  int n_y;
  bool have_next, n_valid;

  __device__ void setup(uint8_t* smem, int tid, const CUtensorMap* tmC) {
    wsm = smem + (tid >> 5) * kTiles * kWarpBytes;
    tm = tmC;
    bad = 0;
    nblk = 0;
    have_next = false;
  }
  __device__ bool load_row(const GemmUnit& g, int row, float& o_so, float& o_db,
                           float& o_dy, int& o_y) {
    SampleDesc sd;
    const CellInfo c = cell_of(a.tiles, a.samples, g.m0, row, sd);
    o_y = -1;
    o_so = -INFINITY;
    o_db = o_dy = 0.f;
    if (!c.valid) return false;
    // per-cell scalars precomputed by edge_kernel (overlapped on the lattice
    // stream): no f64 work in the GEMM's epilogue
    const long long i = skew(sd.lat, sd.U1, c.t, c.u);
    o_so = a.so[i];
    o_db = a.eb[i];
    if (c.u < sd.U1 - 1) {
      o_y = a.labels[sd.lab + c.u];
      o_dy = a.ey[i];
    }
    return true;
  }
  __device__ void prefetch(const GemmUnit& gn, int row) {
    n_valid = load_row(gn, row, n_so, n_db, n_dy, n_y);
    have_next = true;
  }
  __device__ void begin(const GemmUnit& g, int row) {
    bool valid;
    if (have_next) {
      so = n_so;
      d_b = n_db;
      d_y = n_dy;
      y = n_y;
      valid = n_valid;
      have_next = false;
    } else {
      valid = load_row(g, row, so, d_b, d_y, y);
    }
    // non-finite dh (reference loss.cpp:129-131) can only come from these
    if (valid) bad |= !(isfinite(so) && isfinite(d_b) && isfinite(d_y));
  }
  static constexpr bool kEarlyRelease = true;
  template <class Rel>
  __device__ void chunk(const GemmUnit& g, int n0, int row, int half,
                        uint32_t taddr, Rel&& rel) {
    constexpr float kL2E = 1.4426950408889634f;
    const float2 so2 = make_float2(so, so), l2e2 = make_float2(kL2E, kL2E);
    const int lane = threadIdx.x & 31;
    const int r = lane;
    const int row0 = g.m0c + (row & ~31);  // the dh slab row (compacted order)
    // bias of the next block is loaded while the current one is processed
    float4 bnx[8];
    auto bload = [&](int base) {
      const float4* b4 = reinterpret_cast<const float4*>(a.bias_out + base);
#pragma unroll
      for (int q = 0; q < 8; ++q) bnx[q] = __ldg(b4 + q);
    };
    if (32 * half < a.V - n0) bload(n0 + 32 * half);
    tmem_blocks<BN>(taddr, half, a.V - n0, [&](int c, float (&v)[32]) {
      const int base = n0 + c;
      float4 bc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) bc[q] = bnx[q];
      if (c + 64 < BN && base + 64 < a.V) bload(base + 64);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = bc[q];
        const float2 x0 = fma2(add2(make_float2(v[4 * q], v[4 * q + 1]), make_float2(b.x, b.y)), l2e2, so2);
        const float2 x1 = fma2(add2(make_float2(v[4 * q + 2], v[4 * q + 3]), make_float2(b.z, b.w)), l2e2, so2);
        v[4 * q] = ex2(x0.x);
        v[4 * q + 1] = ex2(x0.y);
        v[4 * q + 2] = ex2(x1.x);
        v[4 * q + 3] = ex2(x1.y);
      }
      // the store issued kTiles blocks ago has read the tile this block uses
      if (lane == 0) bulk_wait_read<kTiles - 1>();
      __syncwarp();
      uint8_t* tile = wsm + (nblk % kTiles) * kWarpBytes;
      ++nblk;
      const int yc = y - base;  // label column inside this block?
      const uint32_t ws = smem_u32(tile);
      if constexpr (kTF32) {  // 128-B rows, 128B swizzle
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts_v4(ws + r * 128 + ((q ^ (r & 7)) << 4), E::cvt(v[4 * q]), E::cvt(v[4 * q + 1]),
                 E::cvt(v[4 * q + 2]), E::cvt(v[4 * q + 3]));
        if (base == 0) sts_f32(ws + r * 128 + ((0 ^ (r & 7)) << 4), E::cvt(d_b));
        if ((unsigned)yc < 32u)
          sts_f32(ws + r * 128 + (((yc >> 2) ^ (r & 7)) << 4) + (yc & 3) * 4, E::cvt(d_y));
      } else {  // 32 rows x 64 B, 64B swizzle (bf16 or fp16)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          sts_v4u(ws + r * 64 + ((q ^ ((r >> 1) & 3)) << 4), E::pack2(v[8 * q], v[8 * q + 1]),
                  E::pack2(v[8 * q + 2], v[8 * q + 3]), E::pack2(v[8 * q + 4], v[8 * q + 5]),
                  E::pack2(v[8 * q + 6], v[8 * q + 7]));
        if (base == 0) sts_u16(ws + r * 64 + ((((r >> 1) & 3)) << 4), E::bits(d_b));
        if ((unsigned)yc < 32u)
          sts_u16(ws + r * 64 + ((((yc >> 3) ^ ((r >> 1) & 3))) << 4) + (yc & 7) * 2, E::bits(d_y));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tm, tile, base, row0);
        bulk_commit();
      }
    }, rel);
  }
  __device__ void end(const GemmUnit&, int) {}
  __device__ void finish(uint8_t*, int) {
    if ((threadIdx.x & 31) == 0) bulk_wait<0>();
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.bad, 1);
  }
};

// dz epilogue: tanh gate g = dz (1 - z^2) (reference src/compute.cpp:141-157)
// and both lattice-axis reductions of g. Each warp stages its 32x32 block of
// g in a swizzled smem tile; lane j then reads column j and forms, from the
// same 32 values (rows r = 8*tt + uu), the 4 per-frame sums over label rows
// (-> ga partials) and the 8 per-label-row sums over its 4 frames; the 4
// warps of a column half combine their label-row sums in smem, giving per
// tile part_a[tile][tt][h] (16 rows) and part_l[tile][uu][h] (8 rows).
template <int BN, int kFmt, bool kF32Stage = (kFmt == 1)>
struct EpiDzGate {
  static constexpr bool kTF32 = kFmt == 1;
  static constexpr bool kF16 = kFmt == 2;
  // the bf16 staging tile is a plain-bf16 trade-off; fp16 keeps fp32 staging
  static_assert(kF32Stage || kFmt == 0, "16-bit staging is bf16 only");
  using E = OpElem<kFmt>;
  static constexpr int kGBytes = 4 * kTileU * 32 * 4;  // one half, one buffer
  // z of each warp's 32x32 block arrives by TMA (one 2D box per block, issued
  // a block ahead) into a 2-slot per-warp ring: one coalesced bulk request
  // instead of 32 scattered row segments per load instruction
  static constexpr int kZBlk = 32 * 32 * (kTF32 ? 4 : 2);
  // two slots: block k+1 is issued into the slot block k-1 used, whose z
  // values the gate math of block k-1 has consumed (a single slot would
  // need the in-flight LDS results consumed before the TMA overwrites it)
  static constexpr int kZSlots = 2;
  // per-warp staging tile of the gated block for the transposed column
  // reads: fp32 (128-B rows) in the tf32 / bf16x modes, bf16 (64-B rows) in
  // plain bf16 — 16 KB less shared memory, which buys the mainloop a fifth
  // stage (the gate sums then see bf16-rounded terms: within the bf16 bound)
  static constexpr int kFBytes = kF32Stage ? 4096 : 2048;
  static constexpr int kGOff = 8 * kFBytes;
  static constexpr int kZOff = kGOff + 2 * 2 * kGBytes;
  static constexpr int kBarOff = kZOff + 8 * kZSlots * kZBlk;
  static constexpr int kSmemBytes = kBarOff + 8 * 2 * 8;
  // active tiles only: dh (A) rows compacted, z and partials at the real tile
  static constexpr int kRowMap = 2;
  RowMap map;
  GateArgs a;
  bool valid;
  long long zrow;
  int tile;
  uint32_t F;   // this warp's staging tile (shared address)
  uint32_t G;   // [half][parity][4 quarters][8 uu][32] fp32 (shared address)
  int blk;
  uint8_t* zs;     // this warp's 2 z slots (TMA destination)
  uint32_t zs32;   // same, shared address
  uint64_t* zbar;  // their mbarriers
  const CUtensorMap* tmz;
  int m0w;          // first slab row of this warp's 32 rows in the unit
  uint32_t zk;      // z blocks consumed by this warp so far

  __device__ void setup(uint8_t* smem, int tid, const CUtensorMap* tm) {
    F = smem_u32(smem + (tid >> 5) * kFBytes);
    G = smem_u32(smem + kGOff);
    zs = smem + kZOff + (tid >> 5) * kZSlots * kZBlk;
    zs32 = smem_u32(zs);
    zbar = reinterpret_cast<uint64_t*>(smem + kBarOff) + (tid >> 5) * 2;
    tmz = tm;
    blk = 0;
    zk = 0;
    if ((tid & 31) == 0) {
      mbar_init(&zbar[0], 1);
      mbar_init(&zbar[1], 1);
      fence_mbar_init();
    }
  }
  __device__ void prefetch(const GemmUnit&, int) {}
  // lane 0: bring z block (cols col0..+32, this warp's rows) into its slot
  __device__ void zissue(uint32_t k, int col0) {
    uint64_t* b = &zbar[k % kZSlots];
    mbar_arrive_expect_tx(b, kZBlk);
    tma_load_2d(zs + (k % kZSlots) * kZBlk, tmz, b, col0, m0w);
  }
  __device__ void begin(const GemmUnit& g, int row) {
    SampleDesc sd;
    const CellInfo c = cell_of(a.tiles, a.samples, g.m0, row, sd);
    valid = c.valid;
    zrow = g.m0 + row;
    tile = g.m0 / kGemmBM;
    m0w = g.m0 + (row & ~31);
    // the unit's first block of this warp (chunk 0, column 32 * half)
    const int half = ((threadIdx.x >> 5) - 2) >> 2;
    __syncwarp();
    if ((threadIdx.x & 31) == 0 && 32 * half < a.H) zissue(zk, 32 * half);
  }
  static constexpr bool kEarlyRelease = true;
  template <class Rel>
  __device__ void chunk(const GemmUnit&, int n0, int row, int half,
                        uint32_t taddr, Rel&& rel) {
    const int lane = threadIdx.x & 31;
    const int quarter = row >> 5;
    const float vmask = valid ? 1.f : 0.f;
    tmem_blocks<BN>(taddr, half, a.H - n0, [&](int c, float (&v)[32]) {
      const int base = n0 + c;
      // issue the warp's next z block (same chunk, else the next chunk of the
      // unit; the next unit's first block is issued by begin())
      int nxt = -1;
      if (c + 64 < BN && base + 64 < a.H)
        nxt = base + 64;
      else if (n0 + BN + 32 * half < a.H)
        nxt = n0 + BN + 32 * half;
      if (lane == 0 && nxt >= 0) zissue(zk + 1, nxt);
      mbar_wait(&zbar[zk % kZSlots], (zk / kZSlots) & 1);
      const uint32_t zsl = zs32 + (zk % kZSlots) * kZBlk;
      const int r = lane;
      float z[32];
      if constexpr (kTF32) {  // 128-B rows, 128B swizzle
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 t = lds_v4u(zsl + r * 128 + ((q ^ (r & 7)) << 4));
          z[4 * q] = __uint_as_float(t.x); z[4 * q + 1] = __uint_as_float(t.y);
          z[4 * q + 2] = __uint_as_float(t.z); z[4 * q + 3] = __uint_as_float(t.w);
        }
      } else {  // 64-B rows, 64B swizzle
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 t = lds_v4u(zsl + r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
          const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = E::unpack2(w[e]);
            z[8 * q + 2 * e] = f.x;
            z[8 * q + 2 * e + 1] = f.y;
          }
        }
      }
      __syncwarp();  // this slot is free again
      ++zk;
      // z beyond H is zero in the slab and dz beyond H is zero (OOB B rows)
      const float2 vm2 = make_float2(vmask, vmask);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 zz = make_float2(z[j], z[j + 1]);
        const float2 gate = fma2(make_float2(-zz.x, -zz.y), zz, make_float2(1.f, 1.f));
        const float2 g2 = mul2(mul2(make_float2(v[j], v[j + 1]), gate), vm2);
        v[j] = g2.x;
        v[j + 1] = g2.y;
      }
      float ga[4] = {0.f, 0.f, 0.f, 0.f};
      float gl[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if constexpr (kF32Stage) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts_v4(F + r * 128 + ((q ^ (r & 7)) << 4), v[4 * q], v[4 * q + 1], v[4 * q + 2],
                 v[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const float x = lds_f32(F + rr * 128 + ((((lane >> 2) ^ (rr & 7)) << 2) + (lane & 3)) * 4);
          ga[rr >> 3] += x;
          gl[rr & 7] += x;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) w[e] = E::pack2(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
          sts_v4u(F + r * 64 + ((q ^ ((r >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
        }
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const float x =
              lds_bf16(F + rr * 64 + (((lane >> 3) ^ ((rr >> 1) & 3)) << 4) + (lane & 7) * 2);
          ga[rr >> 3] += x;
          gl[rr & 7] += x;
        }
      }
      __syncwarp();  // F is rewritten by the next block
#pragma unroll
      for (int k = 0; k < 4; ++k)
        a.part_a[((long long)tile * kTileT + 4 * quarter + k) * a.ldp + base + lane] = ga[k];
      const uint32_t Gb = G + (half * 2 + (blk & 1)) * kGBytes;
#pragma unroll
      for (int uu = 0; uu < kTileU; ++uu) sts_f32(Gb + ((quarter * kTileU + uu) * 32 + lane) * 4, gl[uu]);
      half_bar(half);
      {
        // 128 threads of this half: 8 uu x 32 columns, 2 outputs each
        const int t = quarter * 32 + lane;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int o = t + 128 * k;
          const int uu = o >> 5, col = o & 31;
          auto gat = [&](int qq) { return lds_f32(Gb + ((qq * kTileU + uu) * 32 + col) * 4); };
          const float sum = (gat(0) + gat(1)) + (gat(2) + gat(3));
          a.part_l[((long long)tile * kTileU + uu) * a.ldp + base + col] = sum;
        }
      }
      ++blk;  // double-buffered G: the next block writes the other parity
    }, rel);
  }
  __device__ void end(const GemmUnit&, int) {}
  __device__ void finish(uint8_t*, int) {}
};

// ---------------------------------------------------------------------------
// Host-side GEMM plumbing

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D tensor map over a row-major buffer: `inner` contiguous elements per row
// (`ld` apart), `outer` rows; box {box_inner, box_outer}; 128-B swizzle.
enum class Swz { k128, k128Atom32, k64 };

CUtensorMap make_tmap(const void* ptr, bool tf32, long long inner,
                      long long outer, long long ld, int box_inner,
                      int box_outer, Swz swz = Swz::k128) {
  CUtensorMap m;
  const int esz = tf32 ? 4 : 2;
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld * esz)};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  if ((ld * esz) % 16 != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("TMA operand must be 16-byte aligned");
  CUresult r = get_encode()(
      &m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
      2, const_cast<void*>(ptr), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      swz == Swz::k128Atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
      : swz == Swz::k64      ? CU_TENSOR_MAP_SWIZZLE_64B
                             : CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" +
                             std::to_string(int(r)) + ")");
  return m;
}

// kernels launched by this thread (every launch site calls check_launch
// exactly once): the engine's per-step launch count
thread_local long long g_launches = 0;

void check_launch(const char* what) {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// SMs the persistent GEMMs leave free (for a concurrently running lattice
// launch on another stream); set by the engine around overlapped regions.
thread_local int g_gemm_sm_reserve = 0;
// deterministic split-K: partials go here, then an ordered reduction
thread_local float* g_split_ws = nullptr;
thread_local size_t g_split_ws_floats = 0;
// deterministic dW_O / db_O: per-split accumulator slices that persist over
// the step's dW launches ([S][V][H] then [S][V]), reduced once at the end
thread_local float* g_dw_acc = nullptr;
thread_local int g_dw_acc_slices = 0;

// CTA group of the big output-layer GEMMs: 2 = CTA pairs issuing 2-SM MMAs
// (gemm.cuh), 1 = single-SM; SWTB_CTA_GROUP overrides (read once).
int big_cs() {
  static const int cs = [] {
    const char* e = std::getenv("SWTB_CTA_GROUP");
    return (e && std::atoi(e) == 1) ? 1 : 2;
  }();
  return cs;
}
// Calls f(std::integral_constant<int, CG>) for the configured CTA group.
template <class F>
void with_big_cs(F&& f) {
  if (big_cs() == 1)
    f(std::integral_constant<int, 1>{});
  else
    f(std::integral_constant<int, 2>{});
}

// kCS: CTA group (1, or 2 = 2-SM pairs)
template <bool kTF32, bool kAMN, bool kBMN, int BN, class Epi, int kCS = 1>
void run_gemm(const Mat& A, const Mat& B, int M, int N, int K, int splits,
              const Epi& epi, const CUtensorMap* tmC, cudaStream_t st,
              const Mat* A2 = nullptr, const Mat* B2 = nullptr) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  auto go = [&](auto split_tag) {
    constexpr int kSplit = decltype(split_tag)::value;
    using S = GemmShape<kTF32, BN, Epi::kSmemBytes, kSplit, kCS, epi_ones_cols<Epi>()>;
    // operand A: M x K ; B: N x K (logical). 32-bit MN-major operands use
    // the 32-byte-atom 128B swizzle the tensor core expects for them.
    const Swz mn = kTF32 ? Swz::k128Atom32 : Swz::k128;
    auto map_a = [&](const Mat& X) {
      return kAMN ? make_tmap(X.ptr, kTF32, M, K, X.ld, S::MNB, S::BK, mn)
                  : make_tmap(X.ptr, kTF32, K, M, X.ld, S::BK, kGemmBM);
    };
    // row-mapped K (kRowMap 3): B's K rows are read at the real tiles, so its
    // view spans the operand's own rows, not the GEMM's (compacted) K
    const long long kb_ext =
        epi_row_map<Epi>() == 3 ? std::max<long long>(K, B.rows) : (long long)K;
    auto map_b = [&](const Mat& X) {
      return kBMN ? make_tmap(X.ptr, kTF32, N, kb_ext, X.ld, S::MNB, S::BK, mn)
                  : make_tmap(X.ptr, kTF32, kb_ext, N, X.ld, S::BK, S::kBRows);
    };
    const CUtensorMap ta = map_a(A), tb = map_b(B);
    const CUtensorMap ta2 = kSplit == 2 ? map_a(*A2) : ta;
    const CUtensorMap tb2 = kSplit >= 1 ? map_b(*B2) : tb;
    auto kern = gemm_kernel<kTF32, kAMN, kBMN, BN, Epi, kSplit, kCS>;
    const size_t smem = S::kFixedSmem;
    int dev = 0;
    cudaGetDevice(&dev);
    // the shared-memory opt-in is a per-device function attribute: set once
    // per (instantiation, device), thread-safe
    static std::atomic<uint64_t> configured{0};
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem));
      configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    const int num_m = (M + kGemmBM - 1) / kGemmBM;
    const int num_kb = (K + S::BK - 1) / S::BK;
    const int sp = std::max(1, std::min(splits, num_kb));
    const int num_n = (N + BN - 1) / BN;
    const int units = ((num_m + kCS - 1) / kCS) * sp *  // one per cluster
                      (epi_chunk_units<Epi>() ? num_n : 1);
    const int clusters =
        std::min(units, std::max(1, (num_sms(dev) - g_gemm_sm_reserve) / kCS));
    if constexpr (kCS == 1) {
      kern<<<clusters, kGemmThreads, smem, st>>>(ta, tb, tmC ? *tmC : tb, ta2, tb2,
                                                 M, N, K, sp, epi);
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(clusters * kCS);
      cfg.blockDim = dim3(kGemmThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kCS;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const CUtensorMap tc = tmC ? *tmC : tb;
      cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, ta2, tb2, M, N, K, sp, epi);
    }
  };
  if (A2 && !B2) throw std::runtime_error("split A requires split B");
  if (A2) {
    if constexpr (!kTF32 && Epi::kSmemBytes == 0 && !epi_f16<Epi>()) {  // joint GEMMs only
      go(std::integral_constant<int, 2>{});
      check_launch("gemm_kernel(split2)");
      return;
    }
    throw std::runtime_error("split-A GEMM not instantiated for this epilogue");
  }
  if (B2) {
    go(std::integral_constant<int, 1>{});
    check_launch("gemm_kernel(split1)");
    return;
  }
  go(std::integral_constant<int, 0>{});
  check_launch("gemm_kernel");
}

int splits_for(int M, int target_units, int cs = 1) {
  const int num_m = (M + kGemmBM * cs - 1) / (kGemmBM * cs);
  return std::max(1, target_units / std::max(1, num_m));
}

}  // namespace

void set_gemm_sm_reserve(int n) { g_gemm_sm_reserve = n < 0 ? 0 : n; }

long long launch_count() { return g_launches; }

// K splits a launch really runs (run_gemm clamps to the K blocks)
int eff_splits(int splits, long long K, bool tf32) {
  const long long bk = tf32 ? 32 : 64;
  return int(std::max<long long>(1, std::min<long long>(splits, (K + bk - 1) / bk)));
}

void set_split_workspace(float* ws, size_t floats) {
  g_split_ws = ws;
  g_split_ws_floats = ws ? floats : 0;
}

void set_dw_accumulator(float* acc, int slices) {
  g_dw_acc = acc;
  g_dw_acc_slices = acc ? slices : 0;
}

int dw_acc_slices(int device, int V, long long K_dw, bool tf32) {
  return eff_splits(splits_for(V, num_sms(device) / 2, 2), K_dw, tf32);
}


size_t split_workspace_floats(int device, int V, int H, int H_A, int H_L,
                              long long K_joint, long long K_dw, bool tf32) {
  const int sms = num_sms(device);
  (void)K_dw;
  (void)tf32;
  const size_t dw = 0;  // dW_O uses its own accumulator slices
  const size_t joint = size_t(eff_splits(splits_for(H, sms), K_joint, false)) *
                       size_t(H) * std::max(H_A, H_L);
  const size_t dbz = size_t(std::min<long long>(1024, (K_joint + 7) / 8)) * H;
  return std::max(std::max(dw, joint), dbz);
}

namespace {
// out[i] += sum_{s < S} part[s * stride + i] in a fixed order: thread row y
// of a (32 x R) block sums s = y, y + R, ... for one column i, then the R
// row sums are added in y order. Deterministic for a given (S, R).
template <int R>
__global__ void __launch_bounds__(32 * R)
    split_reduce_kernel(const float* __restrict__ part, int S, long long n,
                        long long stride, float* __restrict__ out) {
  __shared__ float red[R][33];
  const long long i = blockIdx.x * 32LL + threadIdx.x;
  float acc = 0.f;
  if (i < n) {
#pragma unroll 4
    for (int s = threadIdx.y; s < S; s += R) acc += part[s * stride + i];
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && i < n) {
    float t = red[0][threadIdx.x];
    for (int y = 1; y < R; ++y) t += red[y][threadIdx.x];
    out[i] += t;
  }
}
}  // namespace

void launch_split_reduce(const float* part, int S, long long n, long long stride,
                         float* out, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = int((n + 31) / 32);
  if (S >= 128)  // long sums over few columns (db_Z block rows): 32 rows
    split_reduce_kernel<32><<<blocks, dim3(32, 32), 0, st>>>(part, S, n, stride, out);
  else
    split_reduce_kernel<8><<<blocks, dim3(32, 8), 0, st>>>(part, S, n, stride, out);
  check_launch("split_reduce_kernel");
}

int num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cached[device]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    cached[device] = n > 0 ? n : 148;
  }
  return cached[device];
}

// ---------------------------------------------------------------------------
// GEMM entry points

#define SWTB_DISPATCH_MAJOR(TF, BNV, EPI, ...)                                 \
  do {                                                                         \
    if (a_mn && b_mn)                                                          \
      run_gemm<TF, true, true, BNV>(__VA_ARGS__);                              \
    else if (a_mn)                                                             \
      run_gemm<TF, true, false, BNV>(__VA_ARGS__);                             \
    else if (b_mn)                                                             \
      run_gemm<TF, false, true, BNV>(__VA_ARGS__);                             \
    else                                                                       \
      run_gemm<TF, false, false, BNV>(__VA_ARGS__);                            \
  } while (0)

#define SWTB_DISPATCH_MAJOR_CS(TF, BNV, EPI, ...)                              \
  with_big_cs([&](auto cs_tag) {                                               \
    constexpr int CS = decltype(cs_tag)::value;                                \
    if (a_mn && b_mn)                                                          \
      run_gemm<TF, true, true, BNV, decltype(EPI), CS>(__VA_ARGS__);           \
    else if (a_mn)                                                             \
      run_gemm<TF, true, false, BNV, decltype(EPI), CS>(__VA_ARGS__);          \
    else if (b_mn)                                                             \
      run_gemm<TF, false, true, BNV, decltype(EPI), CS>(__VA_ARGS__);          \
    else                                                                       \
      run_gemm<TF, false, false, BNV, decltype(EPI), CS>(__VA_ARGS__);         \
  })

void gemm_store(Prec prec, bool a_mn, bool b_mn, const Mat& A, const Mat& B,
                int M, int N, int K, float* out, long long ldo,
                const float* bias, const long long* row_map, cudaStream_t st,
                const Mat* A_lo, const Mat* B_lo) {
  auto body = [&](auto e) {
    e.out = out;
    e.ldo = ldo;
    e.M = M;
    e.N = N;
    e.bias = bias;
    e.row_map = row_map;
    if constexpr (decltype(e)::kF16) {  // fp16 operands (batched scores)
      SWTB_DISPATCH_MAJOR_CS(false, 256, e, A, B, M, N, K, 1, e, nullptr, st, nullptr, B_lo);
    } else if (A_lo) {  // split-operand joint GEMMs (bf16 pairs): small, no clusters
      SWTB_DISPATCH_MAJOR(false, 256, e, A, B, M, N, K, 1, e, nullptr, st, A_lo, B_lo);
    } else if (prec == Prec::kTF32) {
      SWTB_DISPATCH_MAJOR_CS(true, 256, e, A, B, M, N, K, 1, e, nullptr, st, nullptr, B_lo);
    } else {
      SWTB_DISPATCH_MAJOR_CS(false, 256, e, A, B, M, N, K, 1, e, nullptr, st, nullptr, B_lo);
    }
  };
  if (prec == Prec::kFP16) {
    if (A_lo) throw std::runtime_error("split-A fp16 GEMM not instantiated");
    body(EpiStore<256, true>{});
  } else {
    body(EpiStore<256>{});
  }
}

void gemm_atomic(Prec prec, bool a_mn, bool b_mn, const Mat& A, const Mat& B,
                 int M, int N, int K, float* out, long long ldo,
                 cudaStream_t st, const Mat* A_lo, const Mat* B_lo) {
  EpiAtomic<256> e;
  e.out = out;
  e.ldo = ldo;
  e.M = M;
  e.N = N;
  int dev = 0;
  cudaGetDevice(&dev);
  const bool split_bf16 = A_lo || B_lo;
  const int splits = eff_splits(
      split_bf16 ? splits_for(M, num_sms(dev) - g_gemm_sm_reserve)
                 : splits_for(M, (num_sms(dev) - g_gemm_sm_reserve) / big_cs(), big_cs()),
      K, prec == Prec::kTF32);
  // deterministic: per-split partials + ordered reduction (one split adds
  // exactly once per element: the atomic is already order-free)
  const long long part_n = (long long)M * ldo;
  const bool det = g_split_ws && splits > 1;
  if (det && (size_t(splits) * part_n > g_split_ws_floats || ldo != N))
    throw std::runtime_error("deterministic split workspace too small");
  if (det) {
    e.out = g_split_ws;
    e.split_stride = part_n;
  }
  if (split_bf16) {
    if (prec == Prec::kTF32)
      SWTB_DISPATCH_MAJOR(true, 256, e, A, B, M, N, K, splits, e, nullptr, st, A_lo, B_lo);
    else
      SWTB_DISPATCH_MAJOR(false, 256, e, A, B, M, N, K, splits, e, nullptr, st, A_lo, B_lo);
  } else {
    if (prec == Prec::kTF32)
      SWTB_DISPATCH_MAJOR_CS(true, 256, e, A, B, M, N, K, splits, e, nullptr, st);
    else
      SWTB_DISPATCH_MAJOR_CS(false, 256, e, A, B, M, N, K, splits, e, nullptr, st);
  }
  if (det) launch_split_reduce(g_split_ws, splits, part_n, part_n, out, st);
}

void gemm_dw_db(Prec prec, const Mat& dh, const Mat& z, int V, int H, int rows,
                float* dw_out, float* db_out, int* bad, cudaStream_t st,
                const RowMap& map) {
  // dW_O[v, h] += sum_cells dh[cell, v] z[cell, h] (both operands MN-major
  // views of the slabs, split-K over cells) and db_O[v] += sum_cells dh[cell, v]
  auto body = [&](auto e) {
    e.out = dw_out;
    e.ldo = H;
    e.M = V;
    e.N = H;
    e.db = db_out;
    e.bad = bad;
    e.map = map;
    int dev = 0;
    cudaGetDevice(&dev);
    // one wave: units (row-block pairs x N chunks x K splits) fit the CTA
    // pairs available
    const int chunks = (H + 255) / 256;
    const int splits = eff_splits(
        splits_for(V, (num_sms(dev) - g_gemm_sm_reserve) / 2 / chunks, 2), rows,
        prec == Prec::kTF32);
    const long long part_n = (long long)V * H;
    if (g_dw_acc) {  // deterministic: split s adds into accumulator slice s
      if (splits > g_dw_acc_slices)
        throw std::runtime_error("dW_O accumulator has too few slices");
      e.out = g_dw_acc;
      e.split_stride = part_n;
      e.split_accumulate = true;
      e.db = g_dw_acc + size_t(g_dw_acc_slices) * part_n;
      e.db_stride = V;
    }
    if (prec == Prec::kTF32)
      run_gemm<true, true, true, 256, decltype(e), 2>(dh, z, V, H, rows, splits, e, nullptr, st);
    else
      run_gemm<false, true, true, 256, decltype(e), 2>(dh, z, V, H, rows, splits, e, nullptr, st);
  };
  if (prec == Prec::kFP16)
    body(EpiAtomicDb<256, true>{});
  else
    body(EpiAtomicDb<256>{});
}

void gemm_fwd_lse(Prec prec, const Mat& z, const Mat& w_out, int rows, int V,
                  int H, const FwdLseArgs& a, cudaStream_t st,
                  const Mat* w_lo) {
  if (a.xs) {  // logits kept as the fp16 x slab (16-bit operand modes)
    if (prec == Prec::kTF32) throw std::runtime_error("x slab: 16-bit operand modes only");
    if (a.ld_x % 32 || a.ld_xoff % 8) throw std::runtime_error("x slab: ld_x % 32, ld_xoff % 8");
    auto go = [&](auto e) {
      e.a = a;
      with_big_cs([&](auto cs) { run_gemm<false, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, nullptr, st, nullptr, w_lo); });
    };
    if (prec == Prec::kFP16)
      go(EpiFwdLse<256, true, true>{});
    else
      go(EpiFwdLse<256, false, true>{});
    return;
  }
  if (prec == Prec::kTF32) {
    EpiFwdLse<256> e;
    e.a = a;
    with_big_cs([&](auto cs) { run_gemm<true, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, nullptr, st, nullptr, w_lo); });
  } else if (prec == Prec::kFP16) {
    EpiFwdLse<256, true> e;
    e.a = a;
    with_big_cs([&](auto cs) { run_gemm<false, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, nullptr, st, nullptr, w_lo); });
  } else {
    EpiFwdLse<256> e;
    e.a = a;
    with_big_cs([&](auto cs) { run_gemm<false, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, nullptr, st, nullptr, w_lo); });
  }
}

void gemm_bwd_dh(Prec prec, const Mat& z, const Mat& w_out, int rows, int V,
                 int H, const BwdDhArgs& a, cudaStream_t st,
                 const Mat* w_lo) {
  // TMA-store map of the dh slab: 32x32 blocks, swizzle matching the
  // epilogue's staging tiles (fp32: 128B rows, bf16: 64B rows).
  const bool tf = prec == Prec::kTF32;
  // row-mapped: `rows` are z's (the real tiles'), the dh slab holds a.dh_rows
  // compacted rows
  const CUtensorMap tm_dh = make_tmap(a.dh, tf, V, a.dh_rows > 0 ? a.dh_rows : rows, a.ld_dh,
                                      32, 32, tf ? Swz::k128 : Swz::k64);
  if (a.map.list && tf) throw std::runtime_error("row maps: 16-bit operand modes only");
  if (tf) {
    EpiBwdDh<256, 1> e;
    e.a = a;
    e.map = a.map;
    with_big_cs([&](auto cs) { run_gemm<true, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, &tm_dh, st, nullptr, w_lo); });
  } else if (prec == Prec::kFP16) {
    EpiBwdDh<256, 2> e;
    e.a = a;
    e.map = a.map;
    with_big_cs([&](auto cs) { run_gemm<false, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, &tm_dh, st, nullptr, w_lo); });
  } else {
    EpiBwdDh<256, 0> e;
    e.a = a;
    e.map = a.map;
    with_big_cs([&](auto cs) { run_gemm<false, false, false, 256, decltype(e), decltype(cs)::value>(z, w_out, rows, V, H, 1, e, &tm_dh, st, nullptr, w_lo); });
  }
}

void gemm_dz_gate(Prec prec, const Mat& dh, const Mat& w_out, int rows, int V,
                  int H, const GateArgs& a, cudaStream_t st, const Mat* w_lo) {
  // dz[cell, h] = sum_v dh[cell, v] W_O[v, h]: A = dh (K-major over V),
  // B = W_O viewed N(=H)-major, K = V rows. The epilogue reads z by TMA:
  // 32x32 boxes of the z slab, swizzled like its staging reads expect.
  const bool tf = prec == Prec::kTF32;
  // row-mapped: `rows` are the compacted dh rows; z (read at the real tiles)
  // spans a.z_rows
  const CUtensorMap tm_z = make_tmap(a.z, tf, a.ld_z, a.z_rows > 0 ? a.z_rows : rows, a.ld_z,
                                     32, 32, tf ? Swz::k128 : Swz::k64);
  if (a.map.list && tf) throw std::runtime_error("row maps: 16-bit operand modes only");
  if (tf) {
    EpiDzGate<256, 1> e;  // pairs only: with the z ring, 1-SM stages would not fit
    e.a = a;
    e.map = a.map;
    run_gemm<true, false, true, 256, decltype(e), 2>(dh, w_out, rows, H, V, 1, e, &tm_z, st, nullptr, w_lo);
  } else if (prec == Prec::kFP16) {  // fp32 staging: gate sums at fp16 grade
    EpiDzGate<256, 2, true> e;
    e.a = a;
    e.map = a.map;
    run_gemm<false, false, true, 256, decltype(e), 2>(dh, w_out, rows, H, V, 1, e, &tm_z, st, nullptr, w_lo);
  } else if (w_lo) {  // bf16x: fp32 staging keeps the gate sums at its bound
    EpiDzGate<256, 0, true> e;
    e.a = a;
    e.map = a.map;
    run_gemm<false, false, true, 256, decltype(e), 2>(dh, w_out, rows, H, V, 1, e, &tm_z, st, nullptr, w_lo);
  } else {
    EpiDzGate<256, 0> e;
    e.a = a;
    e.map = a.map;
    run_gemm<false, false, true, 256, decltype(e), 2>(dh, w_out, rows, H, V, 1, e, &tm_z, st, nullptr, w_lo);
  }
}

// ---------------------------------------------------------------------------
// Elementwise kernels

namespace {

// dst = round(src) in the operand precision; with dst_lo also the residual
// round(src - dst), so dst + dst_lo carries the weights at ~2x the precision.
__global__ void convert_pad_kernel(const float* __restrict__ src,
                                   long long rows, long long cols,
                                   long long src_ld, void* dst,
                                   long long dst_ld, int fmt, void* dst_lo) {
  const long long total = rows * dst_ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / dst_ld, c = i % dst_ld;
    const float x = c < cols ? src[r * src_ld + c] : 0.f;
    if (fmt == int(Prec::kTF32)) {
      const float h = round_tf32(x);
      reinterpret_cast<float*>(dst)[i] = h;
      if (dst_lo) reinterpret_cast<float*>(dst_lo)[i] = round_tf32(x - h);
    } else if (fmt == int(Prec::kFP16)) {
      const __half h = __float2half_rn(x);
      reinterpret_cast<__half*>(dst)[i] = h;
      if (dst_lo) reinterpret_cast<__half*>(dst_lo)[i] = __float2half_rn(x - __half2float(h));
    } else {
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      reinterpret_cast<__nv_bfloat16*>(dst)[i] = h;
      if (dst_lo)
        reinterpret_cast<__nv_bfloat16*>(dst_lo)[i] =
            __float2bfloat16_rn(x - __bfloat162float(h));
    }
  }
}

// zbar[r, h] = mean over n sampled frames t_i = floor(i T_b / n) of
// tanh(P_A[a0 + t_i, h] + P_L[r, h]) for the R label rows of a joint batch,
// row r's sample given by info[2r] = a0 (its first P_A row), info[2r+1] = T_b.
// The per-label-row mean of z, from which the fp16 forward's logit
// correction zbar_u . (W_O - fp16(W_O))^T is formed: the part of the W_O
// rounding error that every frame of label row u repeats (and that the
// dh^L sums over t would accumulate coherently). The tanh is the z slab's.
__global__ void __launch_bounds__(256)
    zmean_kernel(const float* __restrict__ pa, const float* __restrict__ pl,
                 long long ldp, int H, const int* __restrict__ info, int R, int nsamp,
                 __half* __restrict__ zbar, long long ldz) {
  const int h = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (h >= ldz) return;
  for (int r = blockIdx.y * blockDim.y + threadIdx.y; r < R; r += gridDim.y * blockDim.y) {
    const int a0 = info[2 * r], T = info[2 * r + 1];
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int n = T < nsamp ? T : nsamp;
    if (h < H) {
      const float4 l = __ldg(reinterpret_cast<const float4*>(pl + (long long)r * ldp + h));
#pragma unroll 4
      for (int i = 0; i < n; ++i) {
        const int t = int((long long)i * T / n);
        const float4 x = __ldg(reinterpret_cast<const float4*>(pa + (long long)(a0 + t) * ldp + h));
        acc[0] += fast_tanh(x.x + l.x);
        acc[1] += fast_tanh(x.y + l.y);
        acc[2] += fast_tanh(x.z + l.z);
        acc[3] += fast_tanh(x.w + l.w);
      }
    }
    const float inv = n > 0 ? 1.f / float(n) : 0.f;
    __half o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = __float2half_rn(h + j < H ? acc[j] * inv : 0.f);
    *reinterpret_cast<uint2*>(zbar + (long long)r * ldz + h) = *reinterpret_cast<uint2*>(o);
  }
}

// x ~= hi + lo with hi = bf16(x), lo = bf16(x - hi): |x - hi - lo| <=
// 2^-18 |x|, so hi*hi + hi*lo + lo*hi reproduces float32 products to ~2^-16.
__global__ void split_rows_kernel(const float* __restrict__ src, long long cols,
                                  long long src_ld,
                                  const long long* __restrict__ row_src,
                                  __nv_bfloat16* __restrict__ hi,
                                  __nv_bfloat16* __restrict__ lo,
                                  long long dst_ld, long long rows) {
  const long long total = rows * dst_ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / dst_ld, c = i % dst_ld;
    const long long sr = row_src ? row_src[r] : r;
    const float x = c < cols ? src[sr * src_ld + c] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[i] = h;
    lo[i] = __float2bfloat16_rn(x - __bfloat162float(h));
  }
}

// z slab, one block per 128-cell tile (grid-stride over tiles). Thread
// (x, y): 8-wide h group x (a warp covers 32 groups = 512 contiguous output
// bytes per cell) and frame quad y (4 of the tile's 16 frames). Each thread
// keeps the 8 label rows' P_L slice in registers and streams its 4 frames'
// P_A slices past them: 32 cells x 8 h per 12 loads of 32 B, so L1 traffic
// stays below the bytes written (the HBM write is the bound).
template <int kFmt>
__global__ void __launch_bounds__(256)
    zslab_kernel(const float* __restrict__ pa, const float* __restrict__ pl,
                 long long ldp, int H, const TileDesc* __restrict__ tiles,
                 const SampleDesc* __restrict__ samples, int n_tiles, void* z,
                 long long ldz) {
  constexpr bool kTF32 = kFmt == 1;
  using E = OpElem<kFmt>;
  static_assert(kTileU == 8 && kTileT == 16, "tile shape");
  const int groups = int(ldz / 8);
  auto th = [](float x) { return kTF32 ? tanhf(x) : fast_tanh(x); };
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const TileDesc td = tiles[tile];
    const SampleDesc sd = samples[td.s];
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
      const int h0 = g * 8;
      const bool full = h0 + 8 <= H;
      float l[kTileU][8];
#pragma unroll
      for (int uu = 0; uu < kTileU; ++uu) {
        const int u = td.u0 + uu;
        const float* src = pl + (long long)(sd.l_row0 + u) * ldp + h0;
        if (u < sd.U1 && full) {
          const float4 x0 = __ldg(reinterpret_cast<const float4*>(src));
          const float4 x1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
          l[uu][0] = x0.x; l[uu][1] = x0.y; l[uu][2] = x0.z; l[uu][3] = x0.w;
          l[uu][4] = x1.x; l[uu][5] = x1.y; l[uu][6] = x1.z; l[uu][7] = x1.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) l[uu][j] = (u < sd.U1 && h0 + j < H) ? src[j] : 0.f;
        }
      }
#pragma unroll 1
      for (int tt = threadIdx.y * 4; tt < threadIdx.y * 4 + 4; ++tt) {
        const int t = td.t0 + tt;
        const bool tv = t < sd.T;
        float a[8];
        const float* src = pa + (long long)(sd.a_row0 + t) * ldp + h0;
        if (tv && full) {
          const float4 x0 = __ldg(reinterpret_cast<const float4*>(src));
          const float4 x1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
          a[0] = x0.x; a[1] = x0.y; a[2] = x0.z; a[3] = x0.w;
          a[4] = x1.x; a[5] = x1.y; a[6] = x1.z; a[7] = x1.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = (tv && h0 + j < H) ? src[j] : 0.f;
        }
#pragma unroll
        for (int uu = 0; uu < kTileU; ++uu) {
          const bool ok = tv && td.u0 + uu < sd.U1;
          float zz[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) zz[j] = ok ? th(a[j] + l[uu][j]) : 0.f;
          if (!full) {  // h beyond H is zero in the slab (tanh(0) is 0 anyway)
#pragma unroll
            for (int j = 0; j < 8; ++j) zz[j] = h0 + j < H ? zz[j] : 0.f;
          }
          const long long cell = (long long)tile * kGemmBM + tt * kTileU + uu;
          typename E::T* dst = reinterpret_cast<typename E::T*>(z) + cell * ldz + h0;
          if constexpr (kTF32) {
            reinterpret_cast<float4*>(dst)[0] =
                make_float4(E::cvt(zz[0]), E::cvt(zz[1]), E::cvt(zz[2]), E::cvt(zz[3]));
            reinterpret_cast<float4*>(dst)[1] =
                make_float4(E::cvt(zz[4]), E::cvt(zz[5]), E::cvt(zz[6]), E::cvt(zz[7]));
          } else {
            *reinterpret_cast<uint4*>(dst) =
                make_uint4(E::pack2(zz[0], zz[1]), E::pack2(zz[2], zz[3]),
                           E::pack2(zz[4], zz[5]), E::pack2(zz[6], zz[7]));
          }
        }
      }
    }
  }
}

// log2(2^a + 2^b) with -inf as identity (reference include/swt/loss.hpp:
// 56-64, in log2 units): f64 accumulation, the bounded correction from two
// MUFU ops (|abs err| of a few 1e-7 per step).
__device__ __forceinline__ double lae_fast(double a, double b) {  // log2 units
  if (a == kNegInfD) return b;
  if (b == kNegInfD) return a;
  const double hi = fmax(a, b), lo = fmin(a, b);
  return hi + double(__log2f(1.f + ex2(float(lo - hi))));
}

// The wavefronts' log-add-exp, log2(2^a + 2^b) in log2 units (which saves
// the scalings of e^x / ln x per step): f64 accumulation, the bounded
// correction log2(1 + 2^-|a-b|) in f32 from MUFU ex2/lg2; -inf safe without
// branches (one -inf gives |a-b| = inf, both give NaN; either way the
// clamped exponent flushes the correction to 0 and max(a, b) is returned).
// va[i] = log2(2^va[i] + 2^vb[i]) for R independent rows, written phase by
// phase so the chains interleave.
template <int R>
__device__ __forceinline__ void lae_rows(double (&va)[R], const double (&vb)[R]) {
  double diff[R];
  float x[R];
#pragma unroll
  for (int i = 0; i < R; ++i) diff[i] = va[i] - vb[i];
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = fmaxf(-fabsf(float(diff[i])), -200.f);
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = ex2(x[i]);
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = __log2f(1.f + x[i]);
#pragma unroll
  for (int i = 0; i < R; ++i) va[i] = (diff[i] > 0.0 ? va[i] : vb[i]) + double(x[i]);
}

// One warp per (sample, direction): lane l owns the R consecutive label rows
// u = l*R .. l*R+R-1, so a diagonal step is R independent log-add-exps per
// lane (ILP R) plus ONE shuffle for the row crossing a lane boundary — no
// block barrier on the T+U dependent steps. lp_blank / lp_label arrive in
// kLatChunk-diagonal chunks by bulk copy (cp.async.bulk, mbarrier completion)
// into a double-buffered shared-memory ring, one chunk ahead of use.
// Requires the group's lattice arrays to hold finite values (zero) at every
// off-lattice position and lat_slack() of slack around the samples.
template <int R>
__global__ void __launch_bounds__(128)
    lattice_warp_kernel(const SampleDesc* __restrict__ samples, int n_samples,
                        const double* __restrict__ lpb,
                        const double* __restrict__ lpy,
                        double* __restrict__ alpha, double* __restrict__ beta,
                        double* __restrict__ logz, float* __restrict__ loss_out,
                        int C, int ring_elems) {
  // several (sample, direction) warps share a CTA, so a whole launch group
  // can sit on one SM beside a persistent GEMM running on the others
  extern __shared__ __align__(128) double lsm[];  // per warp: [2 buf][2 arr][C][P]
  __shared__ __align__(8) uint64_t bars[4][2];
  const int warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  if (gw >= 2 * n_samples) return;
  const int s = gw >> 1;
  const bool bwd = gw & 1;
  double* lring = lsm + (size_t)warp * ring_elems;
  uint64_t* bar = bars[warp];
  const SampleDesc sd = samples[s];
  const int T = sd.T, U1 = sd.U1, D = T + U1 - 1, P = lat_pitch(U1);
  const long long L = sd.lat;
  const int lane = threadIdx.x & 31;
  const int u0 = lane * R;
  const int CP = C * P;
  double* out = bwd ? beta : alpha;
  const int nchunks = (D + C - 1) / C;

  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // chunk kc holds the diagonals of steps [kc*C, kc*C + C) in step order:
  // alpha step k reads diagonal k-1, beta step k reads diagonal D-1-k.
  auto issue = [&](int kc) {
    const int buf = kc & 1;
    const long long first = bwd ? (long long)D - (long long)kc * C - C : (long long)kc * C - 1;
    double* dst = lring + buf * 2 * CP;
    mbar_arrive_expect_tx(&bar[buf], uint32_t(2 * CP * 8));
    bulk_g2s(dst, lpb + L + first * P, uint32_t(CP * 8), &bar[buf]);
    bulk_g2s(dst + CP, lpy + L + first * P, uint32_t(CP * 8), &bar[buf]);
  };
  if (lane == 0) issue(0);

  double prev[R];
#pragma unroll
  for (int i = 0; i < R; ++i) prev[i] = kNegInfD;

  for (int kc = 0; kc < nchunks; ++kc) {
    mbar_wait(&bar[kc & 1], (kc >> 1) & 1);
    __syncwarp();
    // the refilled buffer was read (generic proxy) in the previous chunk:
    // order those reads before the bulk copy (async proxy) overwrites it
    if (lane == 0 && kc + 1 < nchunks) {
      fence_proxy_async_smem();
      issue(kc + 1);
    }
    const double* sb = lring + (kc & 1) * 2 * CP;
    const double* sy = sb + CP;
    const int kend = min(C, D - kc * C);
    for (int j = 0; j < kend; ++j) {
      const int k = kc * C + j;
      // ring row of this step: alpha diag k-1 sits at j, beta diag D-1-k at C-1-j
      const int rr = bwd ? (C - 1 - j) * P : j * P;
      // Phase-ordered over the R rows (each phase an unrolled loop) so that
      // the R independent log-add-exp chains interleave in the schedule.
      double va[R], vb[R];
      if (!bwd) {
        const int d = k;
        double left = __shfl_up_sync(0xffffffffu, prev[R - 1], 1);
        if (lane == 0) left = kNegInfD;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          va[i] = prev[i] + sb[rr + u];  // (t-1, u) --blank-->
          vb[i] = (i == 0 ? left : prev[i - 1]) +
                  ((i > 0 || lane > 0) ? sy[rr + u - 1] : 0.0);  // (t, u-1) --label-->
        }
        lae_rows<R>(va, vb);
        double* po = out + L + (long long)d * P + u0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          const double v = (d == 0 && u == 0) ? 0.0 : va[i];
          const bool ok = u < U1 && (unsigned)(d - u) < (unsigned)T;
          prev[i] = ok ? v : kNegInfD;
          if (ok) po[i] = v;
        }
      } else {
        const int d = D - 1 - k;
        double right = __shfl_down_sync(0xffffffffu, prev[0], 1);
        if (lane == 31) right = kNegInfD;
        double cbt[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          cbt[i] = sb[rr + u];
          va[i] = cbt[i] + prev[i];                                        // --blank--> (t+1, u)
          vb[i] = sy[rr + u] + (i == R - 1 ? right : prev[i + 1]);         // --label--> (t, u+1)
        }
        lae_rows<R>(va, vb);
        double* po = out + L + (long long)d * P + u0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          const int t = d - u;
          const double v = (t == T - 1 && u == U1 - 1) ? cbt[i] : va[i];
          const bool ok = u < U1 && (unsigned)t < (unsigned)T;
          prev[i] = ok ? v : kNegInfD;
          if (ok) po[i] = v;
        }
        if (d == 0 && lane == 0) {  // beta[0,0] = log2 Z
          logz[s] = prev[0];
          loss_out[sd.b] = float(-prev[0] * 0.6931471805599453);
        }
      }
    }
  }
}

// Multi-warp wavefront: one CTA of W warps per (sample, direction); lane
// (w, l) owns the R consecutive label rows u = (32 w + l) R + i, so each warp
// carries 1/W of a diagonal step. The row crossing a warp boundary is handed
// over through a double-buffered shared slot with one named barrier per
// step; within a warp it moves by shuffle as in lattice_warp_kernel. Trades
// more SMs for a W-times shorter dependent chain per step: the wavefront
// then fits under the forward GEMMs it overlaps with.
// kPair: one CTA per sample runs both directions (warps [0, W) alpha,
// [W, 2W) beta, each half with its own ring, barriers and named barrier):
// half the SMs held for the same latency.
template <int R, bool kPair = false>
__global__ void __launch_bounds__(512)
    lattice_group_kernel(const SampleDesc* __restrict__ samples,
                         const double* __restrict__ lpb,
                         const double* __restrict__ lpy,
                         double* __restrict__ alpha, double* __restrict__ beta,
                         double* __restrict__ logz, float* __restrict__ loss_out,
                         int C, int ring_doubles) {
  extern __shared__ __align__(128) double lring_all[];  // per half: [2 buf][2 arr][C][P]
  __shared__ __align__(8) uint64_t bars[2][2];
  __shared__ double slots[2][2][16];
  const int W = (blockDim.x >> 5) / (kPair ? 2 : 1);
  const int gwarp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = kPair ? gwarp / W : 0;
  const int warp = gwarp - half * W;
  const int s = kPair ? int(blockIdx.x) : int(blockIdx.x >> 1);
  const bool bwd = kPair ? half == 1 : (blockIdx.x & 1);
  double* lring = lring_all + (size_t)half * ring_doubles;
  uint64_t* bar = bars[half];
  const SampleDesc sd = samples[s];
  const int T = sd.T, U1 = sd.U1, D = T + U1 - 1, P = lat_pitch(U1);
  const long long L = sd.lat;
  const int u0 = (warp * 32 + lane) * R;
  const int CP = C * P;
  double* out = bwd ? beta : alpha;
  const int nchunks = (D + C - 1) / C;
  const bool leader = warp == 0 && lane == 0;

  if (leader) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int kc) {
    const int buf = kc & 1;
    const long long first = bwd ? (long long)D - (long long)kc * C - C : (long long)kc * C - 1;
    double* dst = lring + buf * 2 * CP;
    mbar_arrive_expect_tx(&bar[buf], uint32_t(2 * CP * 8));
    bulk_g2s(dst, lpb + L + first * P, uint32_t(CP * 8), &bar[buf]);
    bulk_g2s(dst + CP, lpy + L + first * P, uint32_t(CP * 8), &bar[buf]);
  };
  if (leader) issue(0);

  double prev[R];
#pragma unroll
  for (int i = 0; i < R; ++i) prev[i] = kNegInfD;

  for (int kc = 0; kc < nchunks; ++kc) {
    mbar_wait(&bar[kc & 1], (kc >> 1) & 1);
    // every warp passed the last step barrier of chunk kc-1: its buffer is
    // free (generic-proxy reads ordered before the async-proxy refill)
    if (leader && kc + 1 < nchunks) {
      fence_proxy_async_smem();
      issue(kc + 1);
    }
    const double* sb = lring + (kc & 1) * 2 * CP;
    const double* sy = sb + CP;
    const int kend = min(C, D - kc * C);
    for (int j = 0; j < kend; ++j) {
      const int k = kc * C + j;
      const int rr = bwd ? (C - 1 - j) * P : j * P;
      double va[R], vb[R];
      if (!bwd) {
        const int d = k;
        double left = __shfl_up_sync(0xffffffffu, prev[R - 1], 1);
        if (lane == 0) left = (warp > 0 && k > 0) ? slots[half][(k - 1) & 1][warp - 1] : kNegInfD;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          va[i] = prev[i] + sb[rr + u];
          vb[i] = (i == 0 ? left : prev[i - 1]) + ((u > 0) ? sy[rr + u - 1] : 0.0);
        }
        lae_rows<R>(va, vb);
        double* po = out + L + (long long)d * P + u0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          const double v = (d == 0 && u == 0) ? 0.0 : va[i];
          const bool ok = u < U1 && (unsigned)(d - u) < (unsigned)T;
          prev[i] = ok ? v : kNegInfD;
          if (ok) po[i] = v;
        }
        if (lane == 31) slots[half][k & 1][warp] = prev[R - 1];
      } else {
        const int d = D - 1 - k;
        double right = __shfl_down_sync(0xffffffffu, prev[0], 1);
        if (lane == 31) right = (warp < W - 1 && k > 0) ? slots[half][(k - 1) & 1][warp + 1] : kNegInfD;
        double cbt[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          cbt[i] = sb[rr + u];
          va[i] = cbt[i] + prev[i];
          vb[i] = sy[rr + u] + (i == R - 1 ? right : prev[i + 1]);
        }
        lae_rows<R>(va, vb);
        double* po = out + L + (long long)d * P + u0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int u = u0 + i;
          const int t = d - u;
          const double v = (t == T - 1 && u == U1 - 1) ? cbt[i] : va[i];
          const bool ok = u < U1 && (unsigned)t < (unsigned)T;
          prev[i] = ok ? v : kNegInfD;
          if (ok) po[i] = v;
        }
        if (lane == 0) slots[half][k & 1][warp] = prev[0];
        if (d == 0 && leader) {  // beta[0,0] = log2 Z
          logz[s] = prev[0];
          loss_out[sd.b] = float(-prev[0] * 0.6931471805599453);
        }
      }
      named_bar_sync(1 + half, W * 32);
    }
  }
}

// Generic wavefront for U1 > 1024 label rows (several rows per thread; the
// previous diagonal lives in shared memory).
__global__ void lattice_kernel_wide(const SampleDesc* __restrict__ samples,
                                    const double* __restrict__ lpb,
                                    const double* __restrict__ lpy,
                                    double* __restrict__ alpha,
                                    double* __restrict__ beta,
                                    double* __restrict__ logz,
                                    float* __restrict__ loss_out) {
  extern __shared__ double lat_smem[];
  const int s = blockIdx.x >> 1;
  const bool bwd = blockIdx.x & 1;
  const SampleDesc sd = samples[s];
  const int T = sd.T, U1 = sd.U1;
  const int D = T + U1 - 1;
  double* prev = lat_smem;
  double* cur = lat_smem + U1;
  const long long L = sd.lat;
  const int P = lat_pitch(U1);
  for (int step = 0; step < D; ++step) {
    const int d = bwd ? D - 1 - step : step;
    for (int u = threadIdx.x; u < U1; u += blockDim.x) {
      const int t = d - u;
      if (t < 0 || t >= T) continue;
      const long long i = L + (long long)d * P + u;
      double v;
      if (!bwd) {
        if (d == 0) {
          v = 0.0;
        } else {
          const double fb = t > 0 ? prev[u] + lpb[i - P] : kNegInfD;
          const double fl = u > 0 ? prev[u - 1] + lpy[i - P - 1] : kNegInfD;
          v = lae_fast(fb, fl);
        }
        alpha[i] = v;
      } else {
        if (t == T - 1 && u == U1 - 1) {
          v = lpb[i];
        } else {
          const double vb = t < T - 1 ? lpb[i] + prev[u] : kNegInfD;
          const double vl = u < U1 - 1 ? lpy[i] + prev[u + 1] : kNegInfD;
          v = lae_fast(vb, vl);
        }
        beta[i] = v;
        if (d == 0) {
          logz[s] = v;
          loss_out[sd.b] = float(-v * 0.6931471805599453);
        }
      }
      cur[u] = v;
    }
    __syncthreads();
    double* tmp = prev;
    prev = cur;
    cur = tmp;
  }
}

// Per-cell scalars of the logit gradient (reference src/loss.cpp:100-127),
// from the lattice (log2 units) once alpha and beta are known:
//   so  = alpha + beta - logZ - lse*log2(e)        (log2 scale of the node)
//   eb  = dh[blank]  = 2^(occ + lp_b) (1 - 2^(beta_dest - beta))
//   ey  = dh[label]  = 2^(occ + lp_y) (1 - 2^(beta[t,u+1] - beta))
// with occ = alpha + beta - logZ; beta_dest = beta[t+1,u], 0 past the
// terminal node, -inf in the last frame otherwise. One block per (sample,
// 32-diagonal slab); threads walk the slab's cells in skewed order, so every
// access is coalesced. Written in place of lse (so), and into eb / ey.
__global__ void __launch_bounds__(256)
    edge_kernel(const SampleDesc* __restrict__ samples,
                const double* __restrict__ lpb, const double* __restrict__ lpy,
                const double* __restrict__ alpha, const double* __restrict__ beta,
                const double* __restrict__ logz, float* __restrict__ lse_so,
                float* __restrict__ eb, float* __restrict__ ey,
                const float* __restrict__ weights, uint8_t* __restrict__ tile_flags,
                float thr, const float* __restrict__ lmp) {
  const int s = blockIdx.y;
  const SampleDesc sd = samples[s];
  const int T = sd.T, U1 = sd.U1, D = T + U1 - 1, P = lat_pitch(U1);
  const int d0 = blockIdx.x * 32;
  if (d0 >= D) return;
  const int nd = min(32, D - d0);
  // per-sample loss weight w_b >= 0: every dh term of the sample scales by
  // w_b, i.e. log2 w_b joins the occupancy exponent (w_b = 0: a finite
  // exponent that flushes every term to 0)
  const double lz = logz[s] - (weights ? (weights[sd.b] > 0.f ? double(log2f(weights[sd.b])) : -1e30)
                                       : 0.0);
  for (int k = threadIdx.x; k < nd * P; k += blockDim.x) {
    const int d = d0 + k / P, u = k % P, t = d - u;
    if (u >= U1 || t < 0 || t >= T) continue;
    const long long i = sd.lat + (long long)d * P + u;
    const double be = beta[i];
    const float occ = float(alpha[i] + be - lz);
    lse_so[i] = occ - lse_so[i] * 1.4426950408889634f;
    // every dh term of the cell is at most occupancy x largest softmax
    // probability (both edge terms too): its tile stays in the backward if
    // any cell's bound reaches the threshold
    if (tile_flags) {
      const float bound = occ + (lmp ? lmp[i] : 0.f);
      if (!(bound <= thr))  // (a non-finite bound keeps its tile)
        tile_flags[sd.tile0 + (t / kTileT) * sd.n_ub + u / kTileU] = 1;
    }
    double bd = kNegInfD;
    if (t < T - 1) bd = beta[i + P];
    else if (u == U1 - 1) bd = 0.0;
    eb[i] = ex2(occ + float(lpb[i])) * (1.f - ex2(float(bd - be)));
    if (u < U1 - 1)
      ey[i] = ex2(occ + float(lpy[i])) * (1.f - ex2(float(beta[i + P + 1] - be)));
  }
}

// ga[r, h] = sum over the sample's u-tiles of part_a; gl[r, h] = sum over its
// t-tiles of part_l. Optionally db += column sums. Each thread owns 4
// consecutive columns (float4 loads: a warp reads 512 contiguous bytes) and
// keeps 4 tile loads in flight (independent partial sums, added in a fixed
// order): the kernel streams the partials at HBM rate instead of waiting on
// one dependent load per tile.
__global__ void __launch_bounds__(256)
    reduce_partials_kernel(const float* __restrict__ part,
                           const SampleDesc* __restrict__ samples,
                           const int* __restrict__ row_sample,
                           int r0, int R, int H, long long ldp, int is_label,
                           __nv_bfloat16* __restrict__ out_hi,
                           __nv_bfloat16* __restrict__ out_lo,
                           float* __restrict__ dbias,
                           float* __restrict__ dbias_part,
                           const uint8_t* __restrict__ active) {
  const int h = (blockIdx.x * 32 + threadIdx.x) * 4;
  __shared__ float4 red[8][33];
  float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
  auto add4 = [](float4& a, const float4 b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  };
  for (int rr = blockIdx.y * blockDim.y + threadIdx.y; rr < R;
       rr += gridDim.y * blockDim.y) {
    if (h >= H) continue;
    const int r = r0 + rr;  // row of the joint batch
    const SampleDesc sd = samples[row_sample[rr]];
    // tiles k = 0..n-1 at part + (base + k * step) * ldp + h; tile index
    // tile0 + k * tstep; inactive tiles (zero dh: the dz GEMM skipped them)
    // contribute 0 and their partials are not read
    long long base, step;
    int n, tfirst, tstep;
    if (!is_label) {
      const int t = r - sd.a_row0;
      const int tb = t / kTileT, tt = t % kTileT;
      base = (sd.tile0 + (long long)tb * sd.n_ub) * kTileT + tt;
      step = kTileT;
      n = sd.n_ub;
      tfirst = sd.tile0 + tb * sd.n_ub;
      tstep = 1;
    } else {
      const int u = r - sd.l_row0;
      const int ub = u / kTileU, uu = u % kTileU;
      base = (sd.tile0 + (long long)ub) * kTileU + uu;
      step = (long long)sd.n_ub * kTileU;
      n = sd.n_tb;
      tfirst = sd.tile0 + ub;
      tstep = sd.n_ub;
    }
    const float* p = part + base * ldp + h;
    const long long st = step * ldp;
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    auto ld = [&](int k) {
      if (active && !active[tfirst + k * tstep]) return zero4;
      return __ldcs(reinterpret_cast<const float4*>(p + k * st));
    };
    float4 a0 = zero4, a1 = a0, a2 = a0, a3 = a0;
    int k = 0;
    for (; k + 4 <= n; k += 4) {
      const float4 x0 = ld(k), x1 = ld(k + 1), x2 = ld(k + 2), x3 = ld(k + 3);
      add4(a0, x0); add4(a1, x1); add4(a2, x2); add4(a3, x3);
    }
    for (; k < n; ++k) add4(a0, ld(k));
    add4(a0, a1);
    add4(a2, a3);
    add4(a0, a2);
    float v[4] = {a0.x, a0.y, a0.z, a0.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h + j >= H) v[j] = 0.f;
    add4(col, make_float4(v[0], v[1], v[2], v[3]));
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      hi[j] = __float2bfloat16_rn(v[j]);
      lo[j] = __float2bfloat16_rn(v[j] - __bfloat162float(hi[j]));
    }
    *reinterpret_cast<uint2*>(out_hi + (long long)r * ldp + h) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(out_lo + (long long)r * ldp + h) = *reinterpret_cast<const uint2*>(lo);
  }
  if (dbias) {
    red[threadIdx.y][threadIdx.x] = col;
    __syncthreads();
    if (threadIdx.y == 0 && h < H) {
      float4 s = red[0][threadIdx.x];
      for (int y = 1; y < 8; ++y) add4(s, red[y][threadIdx.x]);
      const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (h + j >= H) break;
        if (dbias_part)  // deterministic: one row per block, ordered reduction
          dbias_part[(long long)blockIdx.y * H + h + j] = sv[j];
        else
          atomicAdd(&dbias[h + j], sv[j]);
      }
    }
  }
}

// --- f^W on explicit (f64) scores -------------------------------------------

__global__ void scores_lse_kernel(const double* __restrict__ scores, int T,
                                  int U1, int V, const int* __restrict__ y,
                                  const SampleDesc* sdp, float* lse,
                                  double* lpb, double* lpy) {
  const SampleDesc sd = *sdp;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < T * U1;
       c += gridDim.x * blockDim.x) {
    const int t = c / U1, u = c % U1;
    const double* row = scores + (long long)c * V;
    double m = -__builtin_huge_val();
    for (int v = 0; v < V; ++v) m = fmax(m, row[v]);
    double s = 0.0;
    for (int v = 0; v < V; ++v) s += exp(row[v] - m);
    const double l = m + log(s);
    const long long i = skew(sd.lat, U1, t, u);
    lse[i] = float(l);
    lpb[i] = (row[0] - l) * kL2Ed;  // log2 units (lattice convention)
    if (u < U1 - 1) lpy[i] = (row[y[u]] - l) * kL2Ed;
  }
}

__global__ void scores_grad_kernel(const double* __restrict__ scores, int T,
                                   int U1, int V, const int* __restrict__ y,
                                   const SampleDesc* sdp,
                                   const float* __restrict__ lse,
                                   const double* __restrict__ alpha,
                                   const double* __restrict__ beta,
                                   const double* __restrict__ logz,
                                   double* __restrict__ dscores) {
  const SampleDesc sd = *sdp;
  const long long total = (long long)T * U1 * V;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       k < total; k += (long long)gridDim.x * blockDim.x) {
    const int v = int(k % V);
    const long long c = k / V;
    const int t = int(c / U1), u = int(c % U1);
    const long long i = skew(sd.lat, U1, t, u);
    // alpha / beta / logZ are in log2 units
    const double base = (alpha[i] - logz[0]) * kLn2d - double(lse[i]);
    const double h = scores[k];
    double d = exp(h + base + beta[i] * kLn2d);
    if (v == 0) {
      const double bdest = t < T - 1 ? beta[skew(sd.lat, U1, t + 1, u)]
                           : (u == U1 - 1 ? 0.0 : kNegInfD);
      d -= exp(h + base + bdest * kLn2d);
    } else if (u < U1 - 1 && v == y[u]) {
      d -= exp(h + base + beta[skew(sd.lat, U1, t, u + 1)] * kLn2d);
    }
    dscores[k] = d;
  }
}

// --- batched comparator: materialized fp32 scores in tile order ------------
// (reference run_batched, engine.cpp:245-323: log_denominator_kernel and
// loss_gradient_kernel as separate passes over the stored scores). One warp
// per cell row, float4 column blocks; padded cells (outside the sample's
// (T_b, U_b+1) sub-lattice) are skipped by the lse pass and get dh = 0.

__global__ void __launch_bounds__(256)
    tile_scores_lse_kernel(const float* __restrict__ scores, long long ld,
                           long long rows, const TileDesc* __restrict__ tiles,
                           const SampleDesc* __restrict__ samples,
                           const int* __restrict__ labels, int V, float* lse,
                           double* lpb, double* lpy) {
  constexpr float kL2E = 1.4426950408889634f;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
       r < rows; r += nw) {
    SampleDesc sd;
    const CellInfo c = cell_of(tiles, samples, int(r - r % kGemmBM), int(r % kGemmBM), sd);
    if (!c.valid) continue;
    const float* row = scores + r * ld;
    float m = -INFINITY, s = 0.f;
    for (int v0 = 4 * lane; v0 < V; v0 += 128) {
      float x[4];
      if (v0 + 4 <= V) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(row + v0));
        x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
      } else {
        for (int j = 0; j < 4; ++j) x[j] = v0 + j < V ? row[v0 + j] : -INFINITY;
      }
      const float bm = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
      const float nm = fmaxf(m, bm);
      float acc = m == -INFINITY ? 0.f : s * ex2((m - nm) * kL2E);
      for (int j = 0; j < 4; ++j) acc += ex2((x[j] - nm) * kL2E);
      s = acc;
      m = nm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const float os = __shfl_xor_sync(0xffffffffu, s, o);
      const float nm = fmaxf(m, om);
      s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) +
          (om == -INFINITY ? 0.f : os * __expf(om - nm));
      m = nm;
    }
    if (lane == 0) {
      const float l = m + logf(s);
      const long long i = skew(sd.lat, sd.U1, c.t, c.u);
      lse[i] = l;
      lpb[i] = double(row[0] - l) * kL2Ed;
      if (c.u < sd.U1 - 1) lpy[i] = double(row[labels[sd.lab + c.u]] - l) * kL2Ed;
    }
  }
}

template <int kFmt>
__global__ void __launch_bounds__(256)
    tile_dscores_kernel(const float* __restrict__ scores, long long ld,
                        long long rows, const TileDesc* __restrict__ tiles,
                        const SampleDesc* __restrict__ samples,
                        const int* __restrict__ labels, int V, long long V_pad,
                        const float* __restrict__ so_v, const float* __restrict__ eb,
                        const float* __restrict__ ey, void* dh, long long ld_dh,
                        int* bad) {
  constexpr bool kTF32 = kFmt == 1;
  using E = OpElem<kFmt>;
  using T = typename E::T;
  constexpr float kL2E = 1.4426950408889634f;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  int nonfinite = 0;
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
       r < rows; r += nw) {
    SampleDesc sd;
    const CellInfo c = cell_of(tiles, samples, int(r - r % kGemmBM), int(r % kGemmBM), sd);
    float so = -INFINITY, d_b = 0.f, d_y = 0.f;
    int y = -1;
    if (c.valid) {
      const long long i = skew(sd.lat, sd.U1, c.t, c.u);
      so = so_v[i];
      d_b = eb[i];
      if (c.u < sd.U1 - 1) {
        y = labels[sd.lab + c.u];
        d_y = ey[i];
      }
      nonfinite |= !(isfinite(so) && isfinite(d_b) && isfinite(d_y));
    }
    const float* row = scores + r * ld;
    T* out = static_cast<T*>(dh) + r * ld_dh;
    for (long long v0 = 4 * lane; v0 < V_pad; v0 += 128) {
      float x[4] = {0.f, 0.f, 0.f, 0.f};
      if (c.valid) {
        if (v0 + 4 <= V) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(row + v0));
          x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
        } else {
          for (int j = 0; j < 4; ++j) x[j] = v0 + j < V ? row[v0 + j] : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          x[j] = ex2(fmaf(x[j], kL2E, so));
          if (v0 + j == 0) x[j] = d_b;
          if (v0 + j == y) x[j] = d_y;
        }
      }
      if constexpr (kTF32) {
        *reinterpret_cast<float4*>(out + v0) =
            make_float4(E::cvt(x[0]), E::cvt(x[1]), E::cvt(x[2]), E::cvt(x[3]));
      } else {
        *reinterpret_cast<uint2*>(out + v0) = make_uint2(E::pack2(x[0], x[1]), E::pack2(x[2], x[3]));
      }
    }
  }
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(bad, 1);
}

// dh from the forward's x slab, in place (the logit recompute's epilogue
// math on stored logits: reference src/loss.cpp:83-132). A CTA walks 8-row
// strips (grid-stride); each strip's x (8 ld_x fp16, strip-interleaved) and
// its block maxima (8 rows of ld_xoff floats) arrive by 1-D bulk copy into a
// double-buffered shared-memory ring, one strip ahead; every thread then
// forms dh for its 16-B pieces and writes them in the row-major slab layout
// (the GEMM operand) over the strip's own bytes — the strip is entirely in
// shared memory by then. Per warp store instruction: 8 rows x 64 contiguous
// bytes. Thread t always owns row t % 8 of a strip; its row scalars (so,
// edge values, label) are loaded one strip ahead. HBM-bound: 2 B read and
// 2 B written per element, plus 4 B per 32-column block maximum.
template <int kFmt>
__global__ void __launch_bounds__(256)
    x_to_dh_kernel(char* __restrict__ xs, long long ld_x, const float* __restrict__ xoff,
                   long long ld_xoff, long long rows, const TileDesc* __restrict__ tiles,
                   const SampleDesc* __restrict__ samples, const int* __restrict__ labels,
                   int V, const float* __restrict__ so_v, const float* __restrict__ eb,
                   const float* __restrict__ ey, int* bad) {
  using E = OpElem<kFmt>;
  constexpr float kL2E = 1.4426950408889634f;
  extern __shared__ __align__(128) uint8_t xsm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int t = threadIdx.x;
  const int pieces = int(ld_x);              // 16-B pieces per strip (8 rows x ld_x / 8)
  const uint32_t xbytes = uint32_t(16 * ld_x);
  const uint32_t obytes = uint32_t(32 * ld_xoff);  // 8 rows of maxima
  const uint32_t buf_bytes = xbytes + obytes;
  const long long strips = rows / 8;
  if (blockIdx.x >= strips) return;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long long sp, int buf) {
    uint8_t* dst = xsm + buf * buf_bytes;
    mbar_arrive_expect_tx(&bar[buf], buf_bytes);
    bulk_g2s(dst, xs + sp * xbytes, xbytes, &bar[buf]);
    bulk_g2s(dst + xbytes, xoff + sp * 8 * ld_xoff, obytes, &bar[buf]);
  };
  if (t == 0) {
    issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < strips) issue(blockIdx.x + gridDim.x, 1);
  }
  struct RowS {
    float so, d_b, d_y;
    int y;
    bool valid;
  };
  auto row_scalars = [&](long long sp) {
    RowS q{-INFINITY, 0.f, 0.f, -1, false};
    const long long r = sp * 8 + (t & 7);
    SampleDesc sd;
    const CellInfo c = cell_of(tiles, samples, int(r - r % kGemmBM), int(r % kGemmBM), sd);
    if (c.valid) {
      const long long i = skew(sd.lat, sd.U1, c.t, c.u);
      q.valid = true;
      q.so = so_v[i];
      q.d_b = eb[i];
      if (c.u < sd.U1 - 1) {
        q.y = labels[sd.lab + c.u];
        q.d_y = ey[i];
      }
    }
    return q;
  };
  int nonfinite = 0;
  RowS cur = row_scalars(blockIdx.x);
  int k = 0;
  for (long long sp = blockIdx.x; sp < strips; sp += gridDim.x, ++k) {
    const long long nxt = sp + gridDim.x;
    RowS nrs{};
    if (nxt < strips) nrs = row_scalars(nxt);  // in flight during this strip
    const int buf = k & 1;
    mbar_wait(&bar[buf], (k >> 1) & 1);
    const uint4* xin = reinterpret_cast<const uint4*>(xsm + buf * buf_bytes);
    const float* om = reinterpret_cast<const float*>(xsm + buf * buf_bytes + xbytes) +
                      (t & 7) * ld_xoff;
    if (cur.valid)
      nonfinite |= !(isfinite(cur.so) && isfinite(cur.d_b) && isfinite(cur.d_y));
    char* out = xs + sp * xbytes + (t & 7) * 2 * ld_x;  // row t % 8, row-major
    for (int p = t; p < pieces; p += 256) {
      const int v0 = (p >> 3) * 8;  // = 32 (p / 32) + 8 ((p / 8) % 4)
      float d[8];
      if (cur.valid) {
        // block b = p / 32; maxima slot 8 (b / 8) + 4 (b % 2) + (b % 8) / 2
        const int b = p >> 5;
        const float cst = fmaf(om[(b & ~7) + 4 * (b & 1) + ((b & 7) >> 1)], kL2E, cur.so);
        const uint4 q = xin[p];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
          d[2 * j] = ex2(fmaf(x.x, kL2E, cst));
          d[2 * j + 1] = ex2(fmaf(x.y, kL2E, cst));
        }
        if (v0 == 0) d[0] = cur.d_b;
        if ((unsigned)(cur.y - v0) < 8u) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (v0 + j == cur.y) d[j] = cur.d_y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = 0.f;
      }
      if (v0 + 8 > V) {  // vocabulary tail (and the padded columns): 0
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v0 + j >= V) d[j] = 0.f;
      }
      *reinterpret_cast<uint4*>(out + 2 * v0) =
          make_uint4(E::pack2(d[0], d[1]), E::pack2(d[2], d[3]), E::pack2(d[4], d[5]),
                     E::pack2(d[6], d[7]));
    }
    // every thread is done reading this buffer: refill it with strip k + 2
    __syncthreads();
    if (t == 0 && sp + 2 * (long long)gridDim.x < strips) {
      fence_proxy_async_smem();
      issue(sp + 2 * (long long)gridDim.x, buf);
    }
    cur = nrs;
  }
  if (__any_sync(0xffffffffu, nonfinite) && (t & 31) == 0) atomicOr(bad, 1);
}

int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g > 148 * 32) g = 148 * 32;
  return int(std::max<long long>(g, 1));
}

}  // namespace

void launch_x_to_dh(void* xs, long long ld_x, const float* xoff, long long ld_xoff,
                    long long rows, const TileDesc* tiles, const SampleDesc* samples,
                    const int* labels, int V, const float* so, const float* eb,
                    const float* ey, Prec prec, int* bad, cudaStream_t st) {
  if (rows <= 0) return;
  if (ld_x % 32 || rows % 8) throw std::runtime_error("x slab: ld_x % 32, rows % 8");
  if (ld_x > kXMaxLd) throw std::runtime_error("x slab: vocabulary too large");
  int dev = 0;
  cudaGetDevice(&dev);
  // strips are independent, grid-stride; shared memory (two strip buffers
  // per CTA) sets the CTAs per SM
  const size_t smem = 2 * size_t(16 * ld_x + 32 * ld_xoff);
  const int per_sm = int(std::max<size_t>(1, std::min<size_t>(8, (200u << 10) / smem)));
  const int grid = int(std::min<long long>(rows / 8, (long long)num_sms(dev) * per_sm));
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, 256, smem, st>>>(static_cast<char*>(xs), ld_x, xoff, ld_xoff, rows, tiles,
                                  samples, labels, V, so, eb, ey, bad);
  };
  if (prec == Prec::kFP16)
    go(x_to_dh_kernel<2>);
  else if (prec == Prec::kBF16)
    go(x_to_dh_kernel<0>);
  else
    throw std::runtime_error("x slab: 16-bit operand modes only");
  check_launch("x_to_dh_kernel");
}

void launch_tile_scores_lse(const float* scores, long long ld, long long rows,
                            const TileDesc* tiles, const SampleDesc* samples,
                            const int* labels, int V, float* lse, double* lpb,
                            double* lpy, cudaStream_t st) {
  tile_scores_lse_kernel<<<grid_for(rows * 32, 256), 256, 0, st>>>(
      scores, ld, rows, tiles, samples, labels, V, lse, lpb, lpy);
  check_launch("tile_scores_lse_kernel");
}

void launch_tile_dscores(const float* scores, long long ld, long long rows,
                         const TileDesc* tiles, const SampleDesc* samples,
                         const int* labels, int V, long long V_pad,
                         const float* so, const float* eb, const float* ey,
                         void* dh, long long ld_dh, Prec prec, int* bad,
                         cudaStream_t st) {
  if (prec == Prec::kTF32)
    tile_dscores_kernel<1><<<grid_for(rows * 32, 256), 256, 0, st>>>(
        scores, ld, rows, tiles, samples, labels, V, V_pad, so, eb, ey, dh, ld_dh, bad);
  else if (prec == Prec::kFP16)
    tile_dscores_kernel<2><<<grid_for(rows * 32, 256), 256, 0, st>>>(
        scores, ld, rows, tiles, samples, labels, V, V_pad, so, eb, ey, dh, ld_dh, bad);
  else
    tile_dscores_kernel<0><<<grid_for(rows * 32, 256), 256, 0, st>>>(
        scores, ld, rows, tiles, samples, labels, V, V_pad, so, eb, ey, dh, ld_dh, bad);
  check_launch("tile_dscores_kernel");
}

void launch_convert_pad(const float* src, long long rows, long long cols,
                        long long src_ld, void* dst, long long dst_ld,
                        Prec prec, cudaStream_t st, void* dst_lo) {
  if (rows <= 0) return;
  convert_pad_kernel<<<grid_for(rows * dst_ld, 256), 256, 0, st>>>(
      src, rows, cols, src_ld, dst, dst_ld, int(prec), dst_lo);
  check_launch("convert_pad_kernel");
}

void launch_zslab(const float* pa, const float* pl, long long ldp, int H,
                  const TileDesc* tiles, const SampleDesc* samples,
                  int n_tiles, void* z, long long ldz, Prec prec,
                  cudaStream_t st) {
  if (n_tiles <= 0) return;
  const dim3 block(64, kTileT / 4);
  const int grid = std::min(n_tiles, 148 * 8);
  if (prec == Prec::kTF32)
    zslab_kernel<1><<<grid, block, 0, st>>>(pa, pl, ldp, H, tiles, samples, n_tiles, z, ldz);
  else if (prec == Prec::kFP16)
    zslab_kernel<2><<<grid, block, 0, st>>>(pa, pl, ldp, H, tiles, samples, n_tiles, z, ldz);
  else
    zslab_kernel<0><<<grid, block, 0, st>>>(pa, pl, ldp, H, tiles, samples, n_tiles, z, ldz);
  check_launch("zslab_kernel");
}

namespace {

struct LatticeWarpPlan {
  int C, ring, per_cta, grid;
};
LatticeWarpPlan lattice_warp_plan(int n_samples, int max_U1) {
  const int R = (max_U1 + 31) / 32;
  const int units = 2 * n_samples;
  const int P = lat_pitch(max_U1);
  // at most 4 warps (one per SMSP) per CTA: the wavefront warps are
  // issue-bound, sharing a scheduler slows each of them down
  const int wpb = std::min(4, units);
  constexpr size_t kBudget = 200 * 1024;
  LatticeWarpPlan p;
  p.C = kLatChunk;
  while (p.C > 2 && size_t(wpb) * (4 * p.C * P + 32 * R) * 8 > kBudget) p.C >>= 1;
  p.ring = 4 * p.C * P + 32 * R;  // doubles per warp (+ lane overhang)
  p.per_cta = int(std::max<size_t>(1, std::min<size_t>(wpb, kBudget / (size_t(p.ring) * 8))));
  p.grid = (units + p.per_cta - 1) / p.per_cta;
  return p;
}

template <int R>
void launch_lattice_warp(const SampleDesc* samples, int n_samples,
                         const double* lpb, const double* lpy, double* alpha,
                         double* beta, double* logz, float* loss_out, int max_U1,
                         cudaStream_t st) {
  // all (sample, direction) warps of the launch in as few CTAs as shared
  // memory allows; ring depth C (diagonals per bulk copy) shrinks to fit
  const LatticeWarpPlan p = lattice_warp_plan(n_samples, max_U1);
  const size_t smem = size_t(p.per_cta) * p.ring * 8;
  // per-device function attribute: set on every launch (a host-side call of
  // ~1 us; the lattice launches a few times per group)
  cudaFuncSetAttribute(lattice_warp_kernel<R>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  lattice_warp_kernel<R><<<p.grid, 32 * p.per_cta, smem, st>>>(
      samples, n_samples, lpb, lpy, alpha, beta, logz, loss_out, p.C, p.ring);
}

}  // namespace

// Warps per (sample, direction) of the group wavefront: <= 2 label rows per
// lane, up to 16 warps (U1 <= 1024); 1 = the single-warp kernel. SWTB_LAT_W
// caps it (1 forces the single-warp kernel).
int lattice_group_warps(int max_U1) {
  static const int cap = [] {
    const char* e = std::getenv("SWTB_LAT_W");
    const int v = e ? std::atoi(e) : 16;
    return std::max(1, std::min(16, v));
  }();
  // target label rows per lane (SWTB_LAT_R, experiments): fewer rows per lane
  // shorten each step's work, more warps lengthen its barrier
  static const int rows = [] {
    const char* e = std::getenv("SWTB_LAT_R");
    const int v = e ? std::atoi(e) : 2;
    return std::max(1, std::min(8, v));
  }();
  if (max_U1 > 1024) return 1;
  const int w = std::min(cap, (max_U1 + 32 * rows - 1) / (32 * rows));
  // rows per lane must fit the largest instantiation (8)
  return (max_U1 + 32 * w - 1) / (32 * w) <= 8 ? w : 1;
}

// both directions of a sample in one CTA (when 2 W warps fit 512 threads).
// Off by default: A/B at c4 gave the GEMMs -10 ms (fewer reserved SMs) but
// the two directions sharing an SM run 20 % longer and the engine stream
// then waits on them (+8 ms). SWTB_LAT_PAIR=1 turns it on.
bool lattice_pair(int gw) {
  static const bool on = [] {
    const char* e = std::getenv("SWTB_LAT_PAIR");
    return e && std::atoi(e) != 0;
  }();
  return on && 2 * gw * 32 <= 512;
}

int lattice_launch_ctas(int n_samples, int max_U1) {
  if (n_samples <= 0) return 0;
  const int gw = lattice_group_warps(max_U1);
  if (gw > 1) return (lattice_pair(gw) ? 1 : 2) * n_samples;  // one CTA (= SM) each
  if (max_U1 <= 1024) return lattice_warp_plan(n_samples, max_U1).grid;
  return 2 * n_samples;
}

void launch_lattice(const SampleDesc* samples, int n_samples, const int*,
                    const double* lpb, const double* lpy, double* alpha,
                    double* beta, double* logz, float* loss_out, int max_U1,
                    cudaStream_t st) {
  if (n_samples <= 0) return;
  const int gw = lattice_group_warps(max_U1);
  if (gw > 1) {  // several warps per (sample, direction)
    const int P = lat_pitch(max_U1);
    const int C = kLatChunk;
    const int need = (max_U1 + 32 * gw - 1) / (32 * gw);  // rows per lane
    // ring + the lanes' overhang past the last pitch row (per direction)
    const int ring = 4 * C * P + 32 * gw * 8;
    const bool pair = lattice_pair(gw);
    const size_t smem = size_t(ring) * 8 * (pair ? 2 : 1);
    auto go = [&](auto rtag) {
      constexpr int R = decltype(rtag)::value;
      auto launch = [&](auto kern, int grid, int threads) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<grid, threads, smem, st>>>(samples, lpb, lpy, alpha, beta, logz, loss_out, C,
                                          ring);
      };
      if (pair)
        launch(lattice_group_kernel<R, true>, n_samples, 64 * gw);
      else
        launch(lattice_group_kernel<R, false>, 2 * n_samples, 32 * gw);
    };
    if (need <= 1) go(std::integral_constant<int, 1>{});
    else if (need <= 2) go(std::integral_constant<int, 2>{});
    else if (need <= 4) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 8>{});
    check_launch("lattice_group_kernel");
    return;
  }
  const int r = (max_U1 + 31) / 32;  // label rows per lane
  if (r <= 32) {
#define SWTB_LAT(R)                                                             \
  if (r <= R) {                                                                \
    launch_lattice_warp<R>(samples, n_samples, lpb, lpy, alpha, beta, logz,    \
                           loss_out, max_U1, st);                              \
    check_launch("lattice_warp_kernel");                                       \
    return;                                                                    \
  }
    SWTB_LAT(1) SWTB_LAT(2) SWTB_LAT(3) SWTB_LAT(4) SWTB_LAT(5) SWTB_LAT(6)
    SWTB_LAT(7) SWTB_LAT(8) SWTB_LAT(12) SWTB_LAT(16) SWTB_LAT(24) SWTB_LAT(32)
#undef SWTB_LAT
  }
  const size_t smem = size_t(2) * max_U1 * sizeof(double);
  cudaFuncSetAttribute(lattice_kernel_wide,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  lattice_kernel_wide<<<2 * n_samples, 1024, smem, st>>>(
      samples, lpb, lpy, alpha, beta, logz, loss_out);
  check_launch("lattice_kernel");
}

void launch_edge(const SampleDesc* samples, int n_samples, int max_D,
                 const double* lpb, const double* lpy, const double* alpha,
                 const double* beta, const double* logz, float* lse_so,
                 float* eb, float* ey, cudaStream_t st, const float* weights,
                 uint8_t* tile_flags, float thr, const float* lmp) {
  if (n_samples <= 0) return;
  const dim3 grid((max_D + 31) / 32, n_samples);
  edge_kernel<<<grid, 256, 0, st>>>(samples, lpb, lpy, alpha, beta, logz, lse_so,
                                    eb, ey, weights, tile_flags, thr, lmp);
  check_launch("edge_kernel");
}

namespace {
// Active-tile list of one part: list[0, n) = the indices i in [0, n_flags)
// with flags[i] != 0, ascending (deterministic); *count = n, and n is added
// to *total (step statistics). One CTA: a block-wide scan per 1024 flags.
__global__ void __launch_bounds__(1024)
    compact_tiles_kernel(const uint8_t* __restrict__ flags, int n_flags, int* __restrict__ list,
                         int* __restrict__ count, unsigned long long* __restrict__ total) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n_flags; c0 += 1024) {
    const int i = c0 + tid;
    const bool f = i < n_flags && flags[i] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 warp counts
      const int v = wsum[lane];
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      wsum[lane] = x - v;
    }
    __syncthreads();
    if (f) list[base + wsum[warp] + __popc(m & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (tid == 1023) base += wsum[31] + __popc(m);  // the last warp's prefix + count
    __syncthreads();
  }
  if (tid == 0) {
    *count = base;
    if (total) atomicAdd(total, (unsigned long long)base);
  }
}
}  // namespace

void launch_compact_tiles(const uint8_t* flags, int n_flags, int* list, int* count,
                          unsigned long long* total, cudaStream_t st) {
  compact_tiles_kernel<<<1, 1024, 0, st>>>(flags, n_flags, list, count, total);
  check_launch("compact_tiles_kernel");
}

void launch_reduce_partials(const float* part_a, const float* part_l,
                            const SampleDesc* samples, int,
                            const int* row_sample_a, const int* row_sample_l,
                            int ra0, int rl0, int R_A, int R_L, int H, long long ldp,
                            __nv_bfloat16* ga_hi, __nv_bfloat16* ga_lo,
                            __nv_bfloat16* gl_hi, __nv_bfloat16* gl_lo,
                            float* dbias, cudaStream_t st, const uint8_t* active) {
  dim3 block(32, 8);
  const int gx = ((H + 3) / 4 + 31) / 32;  // 4 columns per thread
  if (ldp % 4 != 0) throw std::runtime_error("reduce_partials: ldp must be a multiple of 4");
  if (R_A > 0) {
    dim3 grid(gx, std::min(1024, (R_A + 7) / 8));
    float* dpart = dbias && g_split_ws ? g_split_ws : nullptr;
    if (dpart && size_t(grid.y) * H > g_split_ws_floats)
      throw std::runtime_error("deterministic split workspace too small");
    reduce_partials_kernel<<<grid, block, 0, st>>>(part_a, samples, row_sample_a,
                                                   ra0, R_A, H, ldp, 0, ga_hi,
                                                   ga_lo, dbias, dpart, active);
    check_launch("reduce_partials_kernel(a)");
    if (dpart) launch_split_reduce(dpart, int(grid.y), H, H, dbias, st);
  }
  if (R_L > 0) {
    dim3 grid(gx, std::min(1024, (R_L + 7) / 8));
    reduce_partials_kernel<<<grid, block, 0, st>>>(part_l, samples, row_sample_l,
                                                   rl0, R_L, H, ldp, 1, gl_hi,
                                                   gl_lo, nullptr, nullptr, active);
    check_launch("reduce_partials_kernel(l)");
  }
}

void launch_zmean(const float* pa, const float* pl, long long ldp, int H,
                  const int* row_info, int R, int nsamp, __half* zbar, long long ldz,
                  cudaStream_t st) {
  if (R <= 0) return;
  const dim3 block(32, 8);
  const dim3 grid(unsigned((ldz / 4 + 31) / 32), unsigned(std::min(8192, (R + 7) / 8)));
  zmean_kernel<<<grid, block, 0, st>>>(pa, pl, ldp, H, row_info, R, nsamp, zbar, ldz);
  check_launch("zmean_kernel");
}

void launch_split_rows(const float* src, long long rows, long long cols,
                       long long src_ld, const long long* row_src,
                       __nv_bfloat16* hi, __nv_bfloat16* lo, long long dst_ld,
                       cudaStream_t st) {
  if (rows <= 0) return;
  split_rows_kernel<<<grid_for(rows * dst_ld, 256), 256, 0, st>>>(
      src, cols, src_ld, row_src, hi, lo, dst_ld, rows);
  check_launch("split_rows_kernel");
}

void launch_scores_lse(const double* scores, int T, int U1, int V,
                       const int* y, const SampleDesc* sd, float* lse,
                       double* lpb, double* lpy, cudaStream_t st) {
  scores_lse_kernel<<<grid_for((long long)T * U1, 128), 128, 0, st>>>(
      scores, T, U1, V, y, sd, lse, lpb, lpy);
  check_launch("scores_lse_kernel");
}

void launch_scores_grad(const double* scores, int T, int U1, int V,
                        const int* y, const SampleDesc* sd, const float* lse,
                        const double* alpha, const double* beta,
                        const double* logz, double* dscores, cudaStream_t st) {
  scores_grad_kernel<<<grid_for((long long)T * U1 * V, 256), 256, 0, st>>>(
      scores, T, U1, V, y, sd, lse, alpha, beta, logz, dscores);
  check_launch("scores_grad_kernel");
}

}  // namespace swtb
