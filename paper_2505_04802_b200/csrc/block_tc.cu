// block_tc.cu -- the second half of a pre-norm Reslim block on tcgen05 for
// D = 256 (the 9.5M-class Reslim), fused into one persistent kernel:
//     z'  = z + W_o . o + b_o                         (attention output o, R9)
//     z'' = z' + W_2 . GELU(W_1 . LN2(z') + b_1) + b_2  (tanh-form GELU, reading R28; LN eps 1e-5)
//     xn  = LN1_{l+1}(z'')  (bf16, the next block's QKV input; not for the last block)
// Per 128-token row block the residual row z' never leaves the SM: the
// O-projection accumulates in TMEM, the epilogue warps add b_o and z (streamed
// in by TMA) and write z' BACK into the TMEM accumulator that the MLP's second
// GEMM then accumulates on top of, take the LayerNorm statistics from TMEM
// (two-pass), and write LN2(z') as the bf16 A operand of the first MLP GEMM
// straight into shared memory.  HBM traffic per token: o (512 B) + z read
// (1 KB) + z'' write (1 KB), against 3 KB (O-projection + LN2 kernel) + 2.5 KB
// (MLP kernel with a residual reduce-add) for the unfused pair.
//
// TMEM (512 columns): S region [0, 256) = O-projection accumulator, then the
// two 128-column S/H buffers of the MLP; O region [256, 512) = z' + MLP output.
// Shared memory: X tile (64 KB: o, then LN2(z')), a 3-slot 32 KB ring carrying
// W_o slices, z slices and W_1 / W_2 slices in consumption order, store staging.
//
// Persistent, one CTA per SM, warp-specialised (384 threads):
//   warp 0 lane 0 : TMA producer
//   warp 1 lane 0 : MMA issuer: O-projection (SS, N = 256), then per hidden
//                   chunk h: GEMM1(h) S_h = X W_1[h]^T (SS, N = 128), GEMM2(h-1)
//                   O += H W_2[:,h]^T (TS, N = 256; H in TMEM over S)
//   warp 2        : TMEM allocator
//   warps 4-11    : epilogue, 2 warpgroups (thread = token row = TMEM lane;
//                   warpgroup wg owns features [128 wg, 128 wg + 128) of the
//                   residual and hidden columns [64 wg, 64 wg + 64) of a chunk)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include <atomic>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);
bool make_tmap_f32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols, CUtensorMapSwizzle swz);

extern long long* g_mlp_timeline;   // debug timeline buffer (orbit2_debug_mlp_timeline)

namespace {

// debug timeline (-DORBIT2_BLOCK_TIMELINE): tl[(role * 64 + block) * 8 + event], CTA 0
#ifdef ORBIT2_BLOCK_TIMELINE
#define BTL(role, b, ev)                                                                              \
  do {                                                                                                \
    if (tl != nullptr && blockIdx.x == 0 && (b) < 64) tl[((role) * 64 + (b)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define BTL(role, b, ev) \
  do {                   \
  } while (0)
#endif

constexpr int BM = 128;
constexpr int DM = 256;           // model width D
constexpr int FH = 1024;          // hidden width 4D
constexpr int HC = 128;           // hidden chunk
constexpr int NCH = FH / HC;      // 8 chunks
constexpr int RS = 3;             // ring slots
constexpr int SLOT = 32768;
constexpr int RI_WO = 4;          // ring items per block: W_o K-slices (256 rows x 64 K)
constexpr int RI_Z = 4;           //   z slices (128 rows x 64 features fp32, two 32-column boxes)
constexpr int RI_BLOCK = RI_WO + RI_Z + 4 * NCH;   // + W_1 / W_2 slices
constexpr int X_BYTES = BM * DM * 2;               // 64 KB
constexpr int ZC = 32;                              // features per fp32 staging box (128-byte rows, SW128)
constexpr int ZBOX = BM * ZC * 4;                   // 16 KB
constexpr int STG_BYTES = 2 * ZBOX;                 // per warpgroup: double-buffered store staging
constexpr int EW = 2;
constexpr int CW = HC / EW;                         // hidden columns per warpgroup and chunk
constexpr int ET = 128 * EW;                        // epilogue threads
constexpr int THREADS = 128 + ET;
constexpr int STATS_BYTES = EW * BM * 4;            // per-row partials of the two warpgroups
constexpr int SMEM = X_BYTES + RS * SLOT + EW * STG_BYTES + STATS_BYTES + 1024 + 256;
static_assert(SMEM <= 227 * 1024, "shared memory");

#ifndef ORBIT2_BLOCK_PREFETCH
#define ORBIT2_BLOCK_PREFETCH 0   // L2 prefetch of the next block: faults at large M (unexplained), off
#endif
#ifndef ORBIT2_GELU_TANH
#define ORBIT2_GELU_TANH 1
#endif
// tanh-form GELU on the MUFU (R28): the erf form is FMA-pipe bound here
__device__ __forceinline__ float2 gelu2(float2 x) {
  if (ORBIT2_GELU_TANH) return tc::gelu2_tanh_fast(x);
  return tc::gelu2_erf_fast(x);
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Row statistics over D = 256 features held by two warpgroups (128 each):
// per warpgroup n = 128, mean_w = shift + sum / n, M2_w = sq - sum^2 / n
// (about the warpgroup mean); mean = (mean_0 + mean_1) / 2 and
// M2 = sum_w M2_w + n (mean_w - mean)^2 (Chan's pairwise combination), one
// float per row and warpgroup exchanged at a time (named barrier 3).
__device__ __forceinline__ void combine_stats(float* sStat, int wg, int r, float shift, float sum, float sq,
                                              float& mean, float& rstd) {
  const float mw = shift + sum * (1.f / 128);
  const float m2 = fmaf(-sum, sum * (1.f / 128), sq);
  sStat[wg * BM + r] = mw;
  named_bar(3, ET);
  mean = 0.5f * (mw + sStat[(wg ^ 1) * BM + r]);
  const float dm = mw - mean;
  const float m2g = fmaf(dm * dm, 128.f, m2);   // M2 of this warpgroup's values about the row mean
  named_bar(3, ET);                             // both means read before the slots are reused
  sStat[wg * BM + r] = m2g;
  named_bar(3, ET);
  const float var = (m2g + sStat[(wg ^ 1) * BM + r]) * (1.f / DM);
  rstd = rsqrtf(fmaxf(var, 0.f) + 1e-5f);
  named_bar(3, ET);                             // both read before the next exchange writes
}

__global__ void __launch_bounds__(THREADS, 1)
    block_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmWo,
                    const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
                    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmXn,
                    const float* __restrict__ bo, const float* __restrict__ g2, const float* __restrict__ be2,
                    const float* __restrict__ b1, const float* __restrict__ b2, const float* __restrict__ g1n,
                    const float* __restrict__ be1n, int64_t M, const int32_t* __restrict__ rblk,
                    int32_t nrblk, long long* __restrict__ tl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;                      // o tile, then LN2(z') (SW128 K-major, 4 atoms of 64 columns)
  uint8_t* sW = sX + X_BYTES;              // [RS][SLOT]
  uint8_t* sZ = sW + RS * SLOT;            // [EW][STG_BYTES] store staging
  float* sStat = reinterpret_cast<float*>(sZ + EW * STG_BYTES);   // [EW][BM] exchange slots
  uint64_t* bar = reinterpret_cast<uint64_t*>(sStat + EW * BM);
  uint64_t* x_full = bar;                  // o tile landed
  uint64_t* x_free = x_full + 1;           // GEMM1(7) done: X may take the next block's o
  uint64_t* w_full = x_free + 1;           // [RS]
  uint64_t* w_empty = w_full + RS;         // [RS]
  uint64_t* s_full = w_empty + RS;         // [2] S_h in TMEM
  uint64_t* h_full = s_full + 2;           // [2] H_h written over S_h
  uint64_t* h_free = h_full + 2;           // [2] GEMM2(h) done
  uint64_t* o_full = h_free + 2;           // last GEMM2 of the block done
  uint64_t* op_full = o_full + 1;          // O-projection done
  uint64_t* xn_full = op_full + 1;         // z' in TMEM, LN2(z') in X
  uint64_t* zready = xn_full + 1;          // [RI_Z] z slice p of this block landed (relayed by the MMA thread)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zready + RI_Z);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work list: every 128-row block, or (last block of the model) the listed ones
  const int64_t num_tiles = rblk != nullptr ? (int64_t)nrblk : (M + BM - 1) / BM;
  auto row_block = [&](int64_t k) -> int64_t { return rblk != nullptr ? (int64_t)__ldg(rblk + k) : k; };

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmWo);
    tc::prefetch_tmap(&tmW1);
    tc::prefetch_tmap(&tmW2);
    tc::prefetch_tmap(&tmZ);
    if (g1n != nullptr) tc::prefetch_tmap(&tmXn);
    tc::mbar_init(x_full, 1);
    tc::mbar_init(x_free, 1);
    for (int s = 0; s < RS; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);      // one arrival: an MMA commit or one epilogue thread
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&h_full[s], ET);
      tc::mbar_init(&h_free[s], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(op_full, 1);
    tc::mbar_init(xn_full, ET);
    for (int z = 0; z < RI_Z; ++z) tc::mbar_init(&zready[z], 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t it = 0, tl_ = 0;
      auto slot_begin = [&]() -> uint8_t* {
        const uint32_t s = it % RS, ph = (it / RS) & 1;
        tc::mbar_wait(&w_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&w_full[s], SLOT);
        return sW + s * SLOT;
      };
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
        const int32_t m0 = (int32_t)(row_block(tile) * BM);
        tc::mbar_wait(x_free, (tl_ & 1) ^ 1);
        tc::mbar_arrive_expect_tx(x_full, X_BYTES);
        for (int a = 0; a < DM / 64; ++a) tc::tma_load_2d(&tmA, sX + a * 16384, x_full, a * 64, m0);
        for (int ks = 0; ks < RI_WO; ++ks, ++it) {   // W_o: all 256 output rows, K slice 64 ks
          uint8_t* dst = slot_begin();
          uint64_t* fb = &w_full[it % RS];
          tc::tma_load_2d(&tmWo, dst, fb, ks * 64, 0);
          tc::tma_load_2d(&tmWo, dst + 16384, fb, ks * 64, 128);
        }
        if (ORBIT2_BLOCK_PREFETCH && tile + gridDim.x < num_tiles) {   // warm the L2 with the next block's o, z
          const int32_t mn = (int32_t)((tile + gridDim.x) * BM);
          for (int a = 0; a < DM / 64; ++a) tc::tma_prefetch_2d(&tmA, a * 64, mn);
          for (int c = 0; c < DM / ZC; ++c) tc::tma_prefetch_2d(&tmZ, c * ZC, mn);
        }
        for (int p = 0; p < RI_Z; ++p, ++it) {      // z rows m0.., features 64 zs .. 64 zs + 63,
          const int zs = 2 * (p & 1) + (p >> 1);    // warpgroups interleaved: zs 0, 2, 1, 3
          uint8_t* dst = slot_begin();
          uint64_t* fb = &w_full[it % RS];
          tc::tma_load_2d(&tmZ, dst, fb, zs * 64, m0);
          tc::tma_load_2d(&tmZ, dst + ZBOX, fb, zs * 64 + ZC, m0);
        }
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            for (int pr = 0; pr < 2; ++pr, ++it) {   // W1 rows s*128.., K slices 2pr, 2pr+1
              uint8_t* dst = slot_begin();
              uint64_t* fb = &w_full[it % RS];
              tc::tma_load_2d(&tmW1, dst, fb, (2 * pr) * 64, s * HC);
              tc::tma_load_2d(&tmW1, dst + 16384, fb, (2 * pr + 1) * 64, s * HC);
            }
          }
          if (s >= 1) {
            const int h = s - 1;
            for (int k2 = 0; k2 < 2; ++k2, ++it) {    // W2 all 256 rows, K slice h*128 + 64*k2
              uint8_t* dst = slot_begin();
              uint64_t* fb = &w_full[it % RS];
              tc::tma_load_2d(&tmW2, dst, fb, h * HC + k2 * 64, 0);
              tc::tma_load_2d(&tmW2, dst + 16384, fb, h * HC + k2 * 64, 128);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id1 = tc::idesc_bf16(BM, HC, 0, 0);   // S = X W1^T: 128 tokens x 128 hidden
      constexpr uint32_t id2 = tc::idesc_bf16(BM, DM, 0, 0);   // 128 tokens x 256 features
      const uint32_t x_addr = tc::smem_u32(sX), w_addr = tc::smem_u32(sW);
      uint32_t it = 0, tl_ = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
        // O-projection into the S region: both S/H buffers consumed by the
        // previous block's last two GEMM2s
        tc::mbar_wait(x_full, tl_ & 1);
        BTL(0, tl_, 0);
        if (tl_ >= 1) {
          tc::mbar_wait(&h_free[0], 1);   // completion (8 tl_ - 2) / 2 = 4 tl_ - 1 of each: odd
          tc::mbar_wait(&h_free[1], 1);
        }
        tc::tc_fence_after();
        for (int ks = 0; ks < RI_WO; ++ks, ++it) {
          const uint32_t sl = it % RS;
          tc::mbar_wait(&w_full[sl], (it / RS) & 1);
          tc::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = tc::sdesc(x_addr + ks * 16384 + kk * 32, 16, 1024, tc::SW_128B);
            const uint64_t bd = tc::sdesc(w_addr + sl * SLOT + kk * 32, 16, 1024, tc::SW_128B);
            tc::mma_bf16_ss(tmem, ad, bd, id2, (ks | kk) != 0);
          }
          tc::mma_commit(&w_empty[sl]);
        }
        tc::mma_commit(op_full);
        BTL(0, tl_, 1);
        // z slices: consumed by the epilogue.  The ring's full barriers are waited
        // on by this thread only, in ring order (a parity wait is only safe when the
        // slot's previous load is known to be complete), and relayed per slice.
        for (int zp = 0; zp < RI_Z; ++zp, ++it) {
          tc::mbar_wait(&w_full[it % RS], (it / RS) & 1);
          tc::mbar_arrive(&zready[zp]);
        }
        tc::mbar_wait(xn_full, tl_ & 1);     // z' in the O region, LN2(z') in X
        BTL(0, tl_, 2);
        tc::tc_fence_after();
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            const uint32_t gc = tl_ * NCH + s, buf = gc & 1, use = gc >> 1;
            if (use >= 1) tc::mbar_wait(&h_free[buf], (use - 1) & 1);   // GEMM2(gc - 2) read H
            tc::tc_fence_after();
            for (int pr = 0; pr < 2; ++pr, ++it) {
              const uint32_t sl = it % RS;
              tc::mbar_wait(&w_full[sl], (it / RS) & 1);
              tc::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {     // two 64-wide K slices per slot
                const int ks = 2 * pr + (kk >> 2);
                const uint64_t ad = tc::sdesc(x_addr + ks * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                const uint64_t bd =
                    tc::sdesc(w_addr + sl * SLOT + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ss(tmem + buf * HC, ad, bd, id1, (pr | kk) != 0);
              }
              tc::mma_commit(&w_empty[sl]);
            }
            tc::mma_commit(&s_full[buf]);
            if (s == NCH - 1) tc::mma_commit(x_free);
          }
          if (s >= 1) {
            const int h = s - 1;
            const uint32_t gc = tl_ * NCH + h, hb = gc & 1;
            tc::mbar_wait(&h_full[hb], (gc >> 1) & 1);
            tc::tc_fence_after();
            for (int k2 = 0; k2 < 2; ++k2, ++it) {
              const uint32_t sl = it % RS;
              tc::mbar_wait(&w_full[sl], (it / RS) & 1);
              tc::tc_fence_after();
              const uint32_t a_tm = tmem + hb * HC + 64 * k2;   // warpgroup k2's H (bf16 pairs)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {     // O[t, f] += H[t, hidden] W2[f, hidden] on top of z'
                const uint64_t bd = tc::sdesc(w_addr + sl * SLOT + kk * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ts(tmem + 256, a_tm + kk * 8, bd, id2, 1u);
              }
              tc::mma_commit(&w_empty[sl]);
            }
            tc::mma_commit(&h_free[hb]);
            if (h == NCH - 1) {
              tc::mma_commit(o_full);
              BTL(0, tl_, 3);
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 2 warpgroups ----------------
    const int q = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int r = q * 32 + lane;                 // row within the block = TMEM lane
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t nb = 1 + wg;                  // named barrier of this warpgroup (128 threads)
    const bool issuer = q == 0 && lane == 0;     // per warpgroup: ring releases, TMA stores
    const int f0 = wg * 128;                     // this warpgroup's residual features
    uint8_t* stg = sZ + wg * STG_BYTES;
    const int sw = r & 7;                        // SW128 16-byte unit swizzle of row r
    uint32_t tl_ = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
      const uint32_t ring0 = tl_ * RI_BLOCK + RI_WO;   // ring index of this block's first z slice
      // ---- z' = z + acc + b_o -> O region (TMEM); LN2 statistics (two-pass) ----
      const bool stp = warp == 4 && lane == 0;
      tc::mbar_wait(op_full, tl_ & 1);
      if (stp) BTL(1, tl_, 0);
      tc::tc_fence_after();
      // single-pass statistics about a per-thread shift (the row's first value of
      // this warpgroup: |mean - shift| ~ std, no cancellation), combined across
      // the two warpgroups with Chan's pairwise formula
      float sum = 0.f, sq = 0.f, shift = 0.f;
#pragma unroll 1
      for (int zi = 0; zi < 2; ++zi) {
        const uint32_t gi = ring0 + 2 * zi + wg, sl = gi % RS;
        tc::mbar_wait(&zready[2 * zi + wg], tl_ & 1);   // relayed by the MMA thread
        const uint8_t* zs = sW + sl * SLOT;
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const int c0 = f0 + zi * 64 + hb * ZC;     // first feature of this 32-column box
          uint32_t a[32];
          tc::tmem_ld32(lane_addr + c0, a);
          const float4* b4 = reinterpret_cast<const float4*>(bo + c0);
          const uint8_t* zrow = zs + hb * ZBOX + r * 128;
          tc::tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 zv = *reinterpret_cast<const float4*>(zrow + ((u ^ sw) << 4));
            const float4 bq = __ldg(b4 + u);
            const float y0 = __uint_as_float(a[4 * u]) + bq.x + zv.x;
            const float y1 = __uint_as_float(a[4 * u + 1]) + bq.y + zv.y;
            const float y2 = __uint_as_float(a[4 * u + 2]) + bq.z + zv.z;
            const float y3 = __uint_as_float(a[4 * u + 3]) + bq.w + zv.w;
            if (zi == 0 && hb == 0 && u == 0) shift = y0;
            const float d0 = y0 - shift, d1 = y1 - shift, d2 = y2 - shift, d3 = y3 - shift;
            sum += (d0 + d1) + (d2 + d3);
            // (d0^2 + d1^2) + (d2^2 + d3^2): one dependent add per 4 values, not 4 FMAs
            sq += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
            a[4 * u] = __float_as_uint(y0);
            a[4 * u + 1] = __float_as_uint(y1);
            a[4 * u + 2] = __float_as_uint(y2);
            a[4 * u + 3] = __float_as_uint(y3);
          }
          tc::tmem_st32(lane_addr + 256 + c0, a);
        }
        named_bar(nb, 128);                      // the warpgroup has read the z slice
        if (issuer) tc::mbar_arrive(&w_empty[sl]);
      }
      tc::tmem_st_wait();
      if (stp) BTL(1, tl_, 1);
      float mean, rstd;
      combine_stats(sStat, wg, r, shift, sum, sq, mean, rstd);
      if (stp) BTL(1, tl_, 2);
      // ---- LN2(z') -> bf16 X (the o tile was consumed by the O-projection) ----
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t a[32];
        tc::tmem_ld32(lane_addr + 256 + f0 + c0, a);
        tc::tmem_ld_wait();
        const int k0 = f0 + c0;                  // global feature of a[0]
        uint8_t* xrow = sX + (k0 >> 6) * 16384 + r * 128;
        const float4* g4 = reinterpret_cast<const float4*>(g2 + k0);
        const float4* e4 = reinterpret_cast<const float4*>(be2 + k0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {            // 8 features = one 16-byte unit
          const float4 ga = __ldg(g4 + 2 * u), gb = __ldg(g4 + 2 * u + 1);
          const float4 ea = __ldg(e4 + 2 * u), eb = __ldg(e4 + 2 * u + 1);
          const float* x8 = reinterpret_cast<const float*>(a + 8 * u);
          const uint4 pk = make_uint4(
              tc::pack_bf16((x8[0] - mean) * rstd * ga.x + ea.x, (x8[1] - mean) * rstd * ga.y + ea.y),
              tc::pack_bf16((x8[2] - mean) * rstd * ga.z + ea.z, (x8[3] - mean) * rstd * ga.w + ea.w),
              tc::pack_bf16((x8[4] - mean) * rstd * gb.x + eb.x, (x8[5] - mean) * rstd * gb.y + eb.y),
              tc::pack_bf16((x8[6] - mean) * rstd * gb.z + eb.z, (x8[7] - mean) * rstd * gb.w + eb.w));
          const int unit = ((k0 & 63) >> 3) + u;
          *reinterpret_cast<uint4*>(xrow + ((unit ^ sw) << 4)) = pk;
        }
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(xn_full);
      if (stp) BTL(1, tl_, 3);
      // ---- MLP hidden chunks: bias + GELU, bf16 H over S ----
      for (int h = 0; h < NCH; ++h) {
        const uint32_t gc = tl_ * NCH + h, buf = gc & 1, use = gc >> 1;
        tc::mbar_wait(&s_full[buf], use & 1);
        if (stp && h == 0) BTL(1, tl_, 4);
        if (stp) BTL(2 + (h >> 3), tl_, h & 7);
        tc::tc_fence_after();
        const uint32_t scol = lane_addr + buf * HC + wg * CW;   // this warpgroup's S (and H) columns
        float v[CW];
#pragma unroll
        for (int c = 0; c < CW; c += 32) tc::tmem_ld32(scol + c, *reinterpret_cast<uint32_t(*)[32]>(v + c));
        tc::tmem_ld_wait();
        const float4* bb = reinterpret_cast<const float4*>(b1 + h * HC + wg * CW);
        uint32_t hv[CW / 2];
#pragma unroll
        for (int c8 = 0; c8 < CW / 8; ++c8) {
          const float4 ba = __ldg(bb + 2 * c8), bc = __ldg(bb + 2 * c8 + 1);
          const float* x8 = v + 8 * c8;
          const float2 q0 = gelu2(tc::add2(make_float2(x8[0], x8[1]), make_float2(ba.x, ba.y)));
          const float2 q1 = gelu2(tc::add2(make_float2(x8[2], x8[3]), make_float2(ba.z, ba.w)));
          const float2 q2 = gelu2(tc::add2(make_float2(x8[4], x8[5]), make_float2(bc.x, bc.y)));
          const float2 q3 = gelu2(tc::add2(make_float2(x8[6], x8[7]), make_float2(bc.z, bc.w)));
          hv[4 * c8 + 0] = tc::pack_bf16(q0.x, q0.y);
          hv[4 * c8 + 1] = tc::pack_bf16(q1.x, q1.y);
          hv[4 * c8 + 2] = tc::pack_bf16(q2.x, q2.y);
          hv[4 * c8 + 3] = tc::pack_bf16(q3.x, q3.y);
        }
        tc::tmem_st32(scol, *reinterpret_cast<const uint32_t(*)[32]>(hv));
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&h_full[buf]);
      }
      // ---- z'' = O + b_2 -> z (TMA tensor stores from swizzled staging) ----
      tc::mbar_wait(o_full, tl_ & 1);
      if (stp) BTL(1, tl_, 5);
      tc::tc_fence_after();
      const int32_t m0 = (int32_t)(row_block(tile) * BM);
      float sum2 = 0.f, sq2 = 0.f, shift2 = 0.f;
#pragma unroll 1
      for (int k = 0; k < 128 / ZC; ++k) {
        uint32_t o[ZC];
        tc::tmem_ld32(lane_addr + 256 + f0 + k * ZC, o);
        tc::tmem_ld_wait();
        uint8_t* sb = stg + (k & 1) * ZBOX;
        if (issuer) tc::bulk_wait_read<1>();   // this buffer's previous store has read it
        named_bar(nb, 128);
        const float4* b4 = reinterpret_cast<const float4*>(b2 + f0 + k * ZC);
        uint8_t* srow = sb + r * (ZC * 4);
#pragma unroll
        for (int u = 0; u < ZC / 4; ++u) {
          const float4 bq = __ldg(b4 + u);
          const float4 y = make_float4(__uint_as_float(o[4 * u]) + bq.x, __uint_as_float(o[4 * u + 1]) + bq.y,
                                       __uint_as_float(o[4 * u + 2]) + bq.z, __uint_as_float(o[4 * u + 3]) + bq.w);
          if (k == 0 && u == 0) shift2 = y.x;
          const float d0 = y.x - shift2, d1 = y.y - shift2, d2 = y.z - shift2, d3 = y.w - shift2;
          sum2 += (d0 + d1) + (d2 + d3);
          sq2 += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
          *reinterpret_cast<float4*>(srow + ((u ^ sw) << 4)) = y;
        }
        tc::fence_proxy_async_smem();
        named_bar(nb, 128);
        if (issuer) {
          tc::tma_store_2d(&tmZ, sb, f0 + k * ZC, m0);
          tc::bulk_commit();
        }
      }
      if (stp) BTL(1, tl_, 6);
      if (g1n != nullptr) {
        // ---- LN1 of the next block: xn = LN1(z'') (bf16) -> HBM, the QKV GEMM's input ----
        float mean1, rstd1;
        combine_stats(sStat, wg, r, shift2, sum2, sq2, mean1, rstd1);
        // two bf16 boxes of 128 rows x 64 features per warpgroup, one per staging buffer
#pragma unroll 1
        for (int xb = 0; xb < 2; ++xb) {
          uint8_t* sb = stg + xb * ZBOX;
          if (issuer) tc::bulk_wait_read<1>();
          named_bar(nb, 128);
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 32) {
            const int k0 = f0 + xb * 64 + c0;
            uint32_t a[32];
            tc::tmem_ld32(lane_addr + 256 + k0, a);
            tc::tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int kk = k0 + 8 * u;
              const float4 ba = __ldg(reinterpret_cast<const float4*>(b2 + kk)), bb = __ldg(reinterpret_cast<const float4*>(b2 + kk + 4));
              const float4 ga = __ldg(reinterpret_cast<const float4*>(g1n + kk)), gb = __ldg(reinterpret_cast<const float4*>(g1n + kk + 4));
              const float4 ea = __ldg(reinterpret_cast<const float4*>(be1n + kk)), eb = __ldg(reinterpret_cast<const float4*>(be1n + kk + 4));
              const float* x8 = reinterpret_cast<const float*>(a + 8 * u);
              const uint4 pk = make_uint4(
                  tc::pack_bf16((x8[0] + ba.x - mean1) * rstd1 * ga.x + ea.x, (x8[1] + ba.y - mean1) * rstd1 * ga.y + ea.y),
                  tc::pack_bf16((x8[2] + ba.z - mean1) * rstd1 * ga.z + ea.z, (x8[3] + ba.w - mean1) * rstd1 * ga.w + ea.w),
                  tc::pack_bf16((x8[4] + bb.x - mean1) * rstd1 * gb.x + eb.x, (x8[5] + bb.y - mean1) * rstd1 * gb.y + eb.y),
                  tc::pack_bf16((x8[6] + bb.z - mean1) * rstd1 * gb.z + eb.z, (x8[7] + bb.w - mean1) * rstd1 * gb.w + eb.w));
              const int unit = (c0 >> 3) + u;
              *reinterpret_cast<uint4*>(sb + r * 128 + ((unit ^ sw) << 4)) = pk;
            }
          }
          tc::fence_proxy_async_smem();
          named_bar(nb, 128);
          if (issuer) {
            tc::tma_store_2d(&tmXn, sb, f0 + xb * 64, m0);
            tc::bulk_commit();
          }
        }
      }
      if (stp) BTL(1, tl_, 7);
      tc::tc_fence_before();                   // O region read: the next block's z' may overwrite it
    }
    if (issuer) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool launch_block_tail(const void* ao, int64_t rows_alloc, const void* wo, const float* bo, const float* ln2_g,
                       const float* ln2_b, const void* w1, const float* b1, const void* w2, const float* b2,
                       float* z, int64_t M, int D, const float* ln1n_g, const float* ln1n_b, void* xn_next,
                       const int32_t* row_blocks, int32_t n_row_blocks, cudaStream_t st) {
  if (D != DM || M <= 0) return false;
  CUtensorMap ta, two, t1, t2, tz, txn;
  std::memset(&txn, 0, sizeof(txn));
  if (ln1n_g != nullptr && !make_tmap_bf16(&txn, xn_next, M, DM, DM, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  if (!make_tmap_bf16(&ta, ao, rows_alloc, DM, DM, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&two, wo, DM, DM, DM, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t1, w1, FH, DM, DM, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t2, w2, DM, FH, FH, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  // residual stream z fp32 [M][256]: 128 x 32 boxes (loads zero-fill and stores clip past M)
  if (!make_tmap_f32(&tz, z, M, DM, DM, BM, ZC, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(block_tc_kernel), SMEM, &attr_done)) return false;
  const int sms = num_sms();
  const int64_t tiles = row_blocks != nullptr ? (int64_t)n_row_blocks : (M + BM - 1) / BM;
  if (tiles == 0) return true;
#ifndef ORBIT2_BLOCK_GRID_DIV   // A/B experiments only: fewer persistent CTAs than SMs
#define ORBIT2_BLOCK_GRID_DIV 1
#endif
  const int grid = (int)std::min<int64_t>(tiles, sms / ORBIT2_BLOCK_GRID_DIV);
  block_tc_kernel<<<grid, THREADS, SMEM, st>>>(ta, two, t1, t2, tz, txn, bo, ln2_g, ln2_b, b1, b2, ln1n_g, ln1n_b,
                                               M, row_blocks, n_row_blocks, g_mlp_timeline);
  return true;
}

}  // namespace orbit2
