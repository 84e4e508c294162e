// SPDX-License-Identifier: Apache-2.0
//
// Persistent, warp-specialized tcgen05 GEMM for sm_100a.
//
//   D[m, n] = sum_k A[m, k] * B[n, k]        (fp32 accumulate in TMEM)
//
// A and B are read by TMA into 128-byte-swizzled shared-memory stages; each
// operand is either K-major (K contiguous in global memory) or MN-major (M/N
// contiguous), selected at compile time, so no transposed copies of the
// lattice slabs or weights are ever made. Element type is bf16 or fp16
// (tcgen05.mma kind::f16) or fp32 read as tf32 (kind::tf32).
//
// Work unit = (128-row block, K split). Inside a unit the kernel walks every
// BN-wide column chunk, so one CTA sees complete rows of D — this is what lets
// the log-softmax epilogue reduce over the whole vocabulary without writing
// logits to HBM.
//
// Roles (320 threads):
//   warp 0      TMA producer (the warp runs the loop converged, one
//               elect.sync lane issues: addresses stay warp-uniform)
//   warp 1      TMEM allocator + MMA issuer (same; the elected lane issues
//               the tcgen05.mma / commit, descriptors in uniform registers)
//   warps 2..9  epilogue: TMEM -> registers -> Epi functor. Warp w reads TMEM
//               lane quarter w%4 (one accumulator row per thread); warps 2-5
//               take the even 32-column blocks of a chunk, 6-9 the odd ones.
// Pipelines: smem stages full/empty (TMA <-> MMA) and two TMEM accumulators
// full/empty (MMA <-> epilogue), so the epilogue of chunk i overlaps the MMAs
// of chunk i+1.
//
// CTA pairs (kCG = 2, a 2-CTA cluster): one 2-SM tcgen05.mma
// (cta_group::2, M = 256) covers two consecutive 128-row blocks. Each CTA
// stages its own 128 rows of A and one half (128 rows along N) of the B tile,
// so per SM the shared-memory traffic per k block is A + B/2 written by TMA
// plus A + B/2 read by the tensor core (the 1-SM form moves A + B each way,
// 1.5x more: that bound, not the MMA rate, capped the 1-SM mainloop). The
// leader CTA (rank 0) owns the smem-stage "full" barriers (both CTAs' TMA
// bytes land there) and issues the MMAs; its commits release the stage in
// both CTAs and signal both CTAs' accumulator-full barriers; both CTAs'
// epilogue warps release the accumulator on the leader's "empty" barrier.

#pragma once

#include <cuda.h>

#include "sm100.cuh"

namespace swtb {

constexpr int kGemmBM = 128;
constexpr int kGemmThreads = 320;
constexpr int kEpiThreads = 256;  // warps 2..9

template <bool kTF32, int BN, int kEpiSmem = 0, int kSplit = 0, int kCG = 1,
          int kOnes = 0>
struct GemmShape {
  static constexpr int kElem = kTF32 ? 4 : 2;
  static constexpr int BK = 128 / kElem;   // one 128-B swizzle row of K
  static constexpr int UK = 32 / kElem;    // K per tcgen05.mma
  static constexpr int MNB = 128 / kElem;  // MN elements per 128-B row
  // MN-major operands: 16-bit types use the plain 128B swizzle (8-k atoms,
  // 1024 B); 32-bit types need the 32-byte-atom variant (4-k atoms, 512 B).
  static constexpr uint32_t kMNLayout = kTF32 ? 1u : 2u;
  static constexpr uint32_t kMNSbo = kTF32 ? 512u : 1024u;
  // Split operands, x ~= hi + lo with lo = round(x - hi):
  //   kSplit 1: B only (the weights): every k-step issues A*Bhi + A*Blo,
  //             removing B's rounding error (it is systematic, W_O is reused
  //             by every cell);
  //   kSplit 2: both: Ahi*Bhi + Ahi*Blo + Alo*Bhi (float32-grade products).
  static constexpr int kPartsA = kSplit == 2 ? 2 : 1;
  static constexpr int kPartsB = kSplit >= 1 ? 2 : 1;
  static constexpr int kABytes = kGemmBM * 128;
  static constexpr int kBRows = BN / kCG;  // B rows (along N) this CTA stages
  static constexpr int kBBytes = kBRows * 128;
  static constexpr int kStageBytes = kPartsA * kABytes + kPartsB * kBBytes;
  static constexpr int kBarBytes = 256;
  // kOnes > 0: an extra all-ones B operand (kOnes rows, K-major) whose MMA
  // yields the row sums of A (sum over K) in kOnes extra TMEM columns
  static constexpr int kOnesBytes = kOnes ? 2048 : 0;
  static constexpr int kEpiBytes = (kEpiSmem + 1023) / 1024 * 1024;
  // stages fill what the epilogue's shared memory leaves of 227 KB
  static constexpr int kBudget = 227 * 1024 - 1024 - kBarBytes - kEpiBytes - kOnesBytes;
  static constexpr int kStages =
      (kBudget / kStageBytes) > 8 ? 8 : (kBudget / kStageBytes);
  static_assert(kStages >= 2, "not enough shared memory for 2 stages");
  // with the ones accumulator the chunk accumulator is single-buffered
  static constexpr int kAccBufs = kOnes ? 1 : 2;
  static constexpr int kTmemUsed = kAccBufs * BN + kOnes;
  static constexpr int kTmemCols = kTmemUsed <= 32 ? 32 : kTmemUsed <= 64 ? 64
                                   : kTmemUsed <= 128 ? 128 : kTmemUsed <= 256 ? 256 : 512;
  static constexpr int kFixedSmem = 1024 /*align slack*/ +
                                    kStages * kStageBytes + kOnesBytes +
                                    kEpiBytes + kBarBytes;
  static_assert(BN == 64 || BN == 128 || BN == 256, "BN in {64,128,256}");
};

struct GemmUnit {
  int m0;       // first row of the 128-row block (mapped GEMMs: the real tile's)
  int m0c;      // its row in the compacted order (= m0 unless the rows are mapped)
  bool live;    // the block exists (a cluster's last row group may be short)
  int split;    // K-split index
  int k_begin;  // K range of this split, in BK blocks
  int k_end;
  int nc_begin;  // N chunks the unit walks: all of them, or one (kChunkUnits)
  int nc_end;
};

// Epilogue contract (all methods run on the 256 epilogue threads; `row` in
// [0,128) is the thread's accumulator row, `half` in {0,1} selects the even
// or odd 32-column blocks, tid in [0,256) is the epilogue-thread index):
//   static constexpr int kSmemBytes;                   1024-aligned region
//   void setup(uint8_t* smem, int tid, const CUtensorMap* tmC);
//                                                      once, then bar among epi
//   void begin(const GemmUnit&, int row);
//   void chunk(const GemmUnit&, int n0, int row, int half, uint32_t taddr);
//        tmem_ld32(taddr + c, v) yields columns [n0+c, n0+c+32) of the row
//        for c = 32*half, 32*half + 64, ...; warp-collective, so every lane
//        of a warp calls chunk() together.
//   void end(const GemmUnit&, int row);
//   void finish(uint8_t* extra_smem, int tid);         after bar among epi

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, 256;" ::: "memory");
}
// barrier among the 4 epilogue warps of one column half
__device__ __forceinline__ void half_bar(int half) {
  asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
}

template <class Epi>
constexpr int epi_ones_cols() {
  if constexpr (requires { Epi::kOnesCols; })
    return Epi::kOnesCols;
  else
    return 0;
}

// Epilogues of GEMMs whose 16-bit operands are fp16 (not bf16) say so with
// `static constexpr bool kF16 = true`: only the instruction descriptor's
// operand format (and the all-ones operand) change.
template <class Epi>
constexpr bool epi_f16() {
  if constexpr (requires { Epi::kF16; })
    return Epi::kF16;
  else
    return false;
}

// Epilogues with `kChunkUnits = true` get one N chunk per work unit instead
// of whole rows: unit u = (row group, chunk, split) with the row group
// fastest, so the units of one K split run side by side and read the same A
// rows (both chunks) and B rows (all row groups) from L2 at the same time —
// each operand byte comes from DRAM about once (the dW_O GEMM, whose A and B
// are both multi-GB slabs).
// Row maps (active-tile lists). An epilogue with `kRowMap` > 0 carries a
// `RowMap map`: the GEMM then walks only the 128-row tiles listed in
// map.list[0, n), n = clamp(*map.count - map.offset, 0, map.max) read from
// device memory at kernel start (the list is built on the device; the host
// never learns n):
//   kRowMap 1: M row blocks are the listed tiles; A rows are read at the real
//              tile (m0), the epilogue may write at the compacted row (m0c)
//   kRowMap 2: the same, but A rows are read at the compacted row (A is a
//              compacted slab); the epilogue's metadata use the real tile
//   kRowMap 3: K is the listed tiles' rows (128 / BK K blocks per tile): A's
//              K rows compacted, B's K rows at the real tile
// A null map.list means every tile, in order (the dense path). (RowMap:
// swtb_kernels.h.)
template <class Epi>
constexpr int epi_row_map() {
  if constexpr (requires { Epi::kRowMap; })
    return Epi::kRowMap;
  else
    return 0;
}

// Epilogues with `kEarlyRelease = true` take a release functor as chunk()'s
// last argument and pass it to tmem_blocks: the accumulator goes back to
// the MMA warp once its last TMEM load landed, not after the chunk's math.
template <class Epi>
constexpr bool epi_early_release() {
  if constexpr (requires { Epi::kEarlyRelease; })
    return Epi::kEarlyRelease;
  else
    return false;
}

template <class Epi>
constexpr bool epi_chunk_units() {
  if constexpr (requires { Epi::kChunkUnits; })
    return Epi::kChunkUnits;
  else
    return false;
}

template <bool kTF32, bool kAMN, bool kBMN, int BN, class Epi,
          int kSplit = 0, int kCG = 1>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC,
                const __grid_constant__ CUtensorMap tmA2,
                const __grid_constant__ CUtensorMap tmB2, int M, int N, int K,
                int splits, const Epi epi) {
  constexpr int kOnes = epi_ones_cols<Epi>();
  using S = GemmShape<kTF32, BN, Epi::kSmemBytes, kSplit, kCG, kOnes>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ones_smem = smem + S::kStages * S::kStageBytes;  // 1024-aligned
  uint8_t* epi_smem = ones_smem + S::kOnesBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + S::kEpiBytes);
  uint64_t* empty = full + S::kStages;
  uint64_t* tfull = empty + S::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  static_assert(kCG == 1 || kCG == 2, "CTA group");
  const int crank = kCG > 1 ? int(cluster_ctarank()) : 0;
  const bool leader = crank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if constexpr (kSplit >= 1) tma_prefetch_desc(&tmB2);
    if constexpr (kSplit == 2) tma_prefetch_desc(&tmA2);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      // 1-SM: every epilogue thread; pair: one arrive per epilogue warp of
      // both CTAs (only the leader's copy is used)
      mbar_init(&tempty[a], kCG == 1 ? kEpiThreads : 2 * kEpiThreads / 32);
    }
    fence_mbar_init();
  }
  // pair: both CTAs are resident before the 2-SM allocation, which writes
  // the TMEM address into the slot of both CTAs
  if constexpr (kCG > 1) cluster_sync();
  if (warp == 1) tmem_alloc<S::kTmemCols, kCG>(tmem_slot);
  if constexpr (kOnes > 0) {  // the all-ones operand (any swizzle of ones is ones)
    for (int i = threadIdx.x; i < S::kOnesBytes / 4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(ones_smem)[i] =
          kTF32 ? 0x3F800000u : epi_f16<Epi>() ? 0x3C003C00u : 0x3F803F80u;
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCG > 1) cluster_sync();  // the pair's barriers exist before use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  constexpr int kMap = epi_row_map<Epi>();
  constexpr int kKbPerTile = kGemmBM / S::BK;
  int nmap = 0;  // listed tiles
  const int* mlist = nullptr;
  if constexpr (kMap > 0) {
    mlist = epi.map.list;
    nmap = mlist ? min(epi.map.max, max(0, *epi.map.count - epi.map.offset))
                 : (kMap == 3 ? K : M) / kGemmBM;
  }
  const int num_m = (kMap == 1 || kMap == 2) ? nmap : (M + kGemmBM - 1) / kGemmBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_kb = kMap == 3 ? kKbPerTile * nmap : (K + S::BK - 1) / S::BK;
  const int num_mg = (num_m + kCG - 1) / kCG;  // row-block groups (one per pair)
  constexpr bool kChunks = epi_chunk_units<Epi>();
  const int units = num_mg * splits * (kChunks ? num_n : 1);
  const int cid = int(blockIdx.x) / kCG, ncl = int(gridDim.x) / kCG;

  auto unit_of = [&](int u) {
    GemmUnit g;
    const int rb = (u % num_mg) * kCG + crank;  // may be past the end in the last pair
    g.m0c = rb * kGemmBM;
    if constexpr (kMap == 1 || kMap == 2) {
      g.live = rb < nmap;
      g.m0 = (g.live && mlist) ? mlist[rb] * kGemmBM : g.m0c;
    } else {
      g.m0 = g.m0c;
      g.live = g.m0 < M;
    }
    if constexpr (kChunks) {
      g.nc_begin = (u / num_mg) % num_n;
      g.nc_end = g.nc_begin + 1;
      g.split = u / (num_mg * num_n);
    } else {
      g.nc_begin = 0;
      g.nc_end = num_n;
      g.split = u / num_mg;
    }
    g.k_begin = int((long long)num_kb * g.split / splits);
    g.k_end = int((long long)num_kb * (g.split + 1) / splits);
    return g;
  };

  if (warp == 0) {
    {
      // ---------------- TMA producer ----------------
      // the whole warp runs the loop; one elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < units; u += ncl) {
        const GemmUnit g = unit_of(u);
        if (g.k_end <= g.k_begin) continue;  // an empty K split (row-mapped K)
        // A's rows: the real tile, or its compacted row (kRowMap 2)
        const int am0 = kMap == 2 ? g.m0c : g.m0;
        for (int nc = g.nc_begin; nc < g.nc_end; ++nc) {
          const int n0 = nc * BN;
          for (int kb = g.k_begin; kb < g.k_end; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * S::kStageBytes;
            uint8_t* sb = sa + S::kPartsA * S::kABytes;
            if (elect_one()) {
            // pair: both CTAs' bytes complete on the leader's barrier
            if (leader) mbar_arrive_expect_tx(&full[stage], kCG * S::kStageBytes);
            const int k0 = kb * S::BK;
            // kRowMap 3: B's K rows at the real tile (A's stay compacted)
            int k0b = k0;
            if constexpr (kMap == 3) {
              if (mlist) k0b = mlist[kb / kKbPerTile] * kGemmBM + (kb % kKbPerTile) * S::BK;
            }
            auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
              if constexpr (kCG == 1)
                tma_load_2d(dst, m, &full[stage], c0, c1);
              else
                tma_load_2d_pair(dst, m, &full[stage], c0, c1);
            };
#pragma unroll
            for (int part = 0; part < S::kPartsA; ++part) {
              const CUtensorMap* ta = part ? &tmA2 : &tmA;
              uint8_t* pa = sa + part * S::kABytes;
              if constexpr (kAMN) {
#pragma unroll
                for (int j = 0; j < kGemmBM / S::MNB; ++j)
                  load(pa + j * S::BK * 128, ta, am0 + j * S::MNB, k0);
              } else {
                load(pa, ta, k0, am0);
              }
            }
#pragma unroll
            for (int part = 0; part < S::kPartsB; ++part) {
              const CUtensorMap* tb = part ? &tmB2 : &tmB;
              uint8_t* pb = sb + part * S::kBBytes;
              // this CTA's rows [crank*kBRows, +kBRows) of the N chunk
              const int nb = n0 + crank * S::kBRows;
              if constexpr (kBMN) {
#pragma unroll
                for (int j = 0; j < S::kBRows / S::MNB; ++j)
                  load(pb + j * S::BK * 128, tb, nb + j * S::MNB, k0b);
              } else {
                load(pb, tb, k0b, nb);
              }
            }
            }  // elected lane
            __syncwarp();
            if (++stage == S::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // CTA-uniform; the whole warp runs, one elected lane issues
      // ---------------- MMA issuer (pair: leader only) ----------------
      constexpr bool kF16 = epi_f16<Epi>();
      constexpr uint32_t idesc = make_idesc<kTF32>(kGemmBM * kCG, BN, kAMN, kBMN, kF16);
      constexpr uint32_t idesc_ones =
          make_idesc<kTF32>(kGemmBM * kCG, kOnes ? kOnes : 16, kAMN, false, kF16);
      const uint32_t ones_base = smem_u32(ones_smem);
      const uint32_t d_ones = tmem_base + uint32_t(S::kAccBufs * BN);
      constexpr uint16_t kPairMask = 0x3;
      auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc_in) {
        if constexpr (kCG == 1)
          mma_ss<kTF32>(d, a, b, idesc, acc_in);
        else
          mma_ss_pair<kTF32>(d, a, b, idesc, acc_in);
      };
      auto commit = [&](uint64_t* bar) {
        if constexpr (kCG == 1)
          mma_commit(bar);
        else
          mma_commit_pair_mc(bar, kPairMask);
      };
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cid; u < units; u += ncl) {
        const GemmUnit g = unit_of(u);
        if (g.k_end <= g.k_begin) continue;
        for (int nc = g.nc_begin; nc < g.nc_end; ++nc) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
          for (int kb = g.k_begin; kb < g.k_end; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
            const uint32_t sb = sa + S::kPartsA * S::kABytes;
            auto desc_a = [&](uint32_t base, int k) {
              if constexpr (kAMN)
                return smem_desc_sw128(base + k * S::UK * 128, S::BK * 128,
                                       S::kMNSbo, S::kMNLayout);
              else
                return smem_desc_sw128(base + k * 32, 16, 1024);
            };
            auto desc_b = [&](uint32_t base, int k) {
              if constexpr (kBMN)
                return smem_desc_sw128(base + k * S::UK * 128, S::BK * 128,
                                       S::kMNSbo, S::kMNLayout);
              else
                return smem_desc_sw128(base + k * 32, 16, 1024);
            };
            const bool issuer = elect_one();
            if (issuer) {
#pragma unroll
            for (int k = 0; k < S::BK / S::UK; ++k) {
              const uint32_t acc_in = (kb > g.k_begin || k > 0) ? 1u : 0u;
              mma(d_tmem, desc_a(sa, k), desc_b(sb, k), acc_in);
              if constexpr (kSplit >= 1)
                mma(d_tmem, desc_a(sa, k), desc_b(sb + S::kBBytes, k), 1u);
              if constexpr (kSplit == 2)
                mma(d_tmem, desc_a(sa + S::kABytes, k), desc_b(sb, k), 1u);
              if constexpr (kOnes > 0) {  // row sums of A, once per unit (chunk 0)
                if (nc == 0) {
                  const uint64_t od = smem_desc_sw128(ones_base + k * 32, 16, 1024);
                  if constexpr (kCG == 1)
                    mma_ss<kTF32>(d_ones, desc_a(sa, k), od, idesc_ones, acc_in);
                  else
                    mma_ss_pair<kTF32>(d_ones, desc_a(sa, k), od, idesc_ones, acc_in);
                }
              }
            }
            commit(&empty[stage]);
            }  // issuer
            __syncwarp();
            if (++stage == S::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (elect_one()) commit(&tfull[acc]);
          __syncwarp();
          if (++acc == S::kAccBufs) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9) ----------------
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int half = (warp - 2) >> 2;
    const int tid = (warp - 2) * 32 + lane;
    Epi e = epi;
    e.setup(epi_smem, tid, &tmC);
    epi_bar();
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cid; u < units; u += ncl) {
      const GemmUnit g = unit_of(u);
      if (g.k_end <= g.k_begin) continue;
      const bool live = g.live;  // a cluster's last row group may be short
      if (live) e.begin(g, row);
      // optional hook: the epilogue may start loads for its next unit
      if (u + ncl < units) {
        const GemmUnit gn = unit_of(u + ncl);
        if (gn.live && gn.k_end > gn.k_begin) e.prefetch(gn, row);
      }
      for (int nc = g.nc_begin; nc < g.nc_end; ++nc) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
        auto release = [&] {
          tc_fence_before();
          if constexpr (kCG == 1) {
            mbar_arrive(&tempty[acc]);
          } else {  // one arrive per warp on the leader's barrier
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
          }
        };
        if constexpr (epi_early_release<Epi>()) {
          if (live)
            e.chunk(g, nc * BN, row, half, taddr, release);
          else
            release();
        } else {
          if (live) e.chunk(g, nc * BN, row, half, taddr);
          if constexpr (kOnes > 0) {  // the unit's A row sums, after its chunk 0
            if (live && nc == 0)
              e.ones(g, row, half, tmem_base + (uint32_t(quarter * 32) << 16) +
                                       uint32_t(S::kAccBufs * BN));
          }
          release();
        }
        if (++acc == S::kAccBufs) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (live) e.end(g, row);
    }
    epi_bar();
    e.finish(epi_smem, tid);
  }

  __syncthreads();
  // no CTA may leave while its peer can still signal its barriers / TMEM
  if constexpr (kCG > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<S::kTmemCols, kCG>(tmem_base);
  }
}

}  // namespace swtb
