// attn_bwd_tc.cu -- backward of the per-tile attention on tcgen05 (training step,
// SURVEY.md §8(f) row 3; oracle/train.py _attn_bwd).
//
// For one (tile, head, sample) with S = Q K^T c (c = 1/sqrt(d)), P = softmax_rows(S),
// O = P V and the incoming dO:
//     dV = P^T dO;   dP = dO V^T;   dS = P (dP - Delta),  Delta_q = sum_d dO_q O_q;
//     dQ = c dS K;   dK = c dS^T Q
// P is recomputed from the forward's per-row log-sum-exp (log2 units:
// P = 2^(S log2(e) c - lse2)).  Attention stays inside the tile.
//
// Work item = (key block of 128 keys of a tile, head, sample); the CTA walks
// every 128-query block of the tile (persistent, one CTA per SM):
//   warp 0 lane 0 : TMA producer (K, V of the item into a 2-slot ring; Q_j, dO_j
//                   into a 2-slot ring)
//   warp 1        : tcgen05.mma issuer, per query half h (64 queries) of block j:
//       S^T_h  = K Q_h^T        (SS, both K-major, N = 64)    -> TMEM [128 h, 128 h + 64)
//       dP^T_h = V dO_h^T       (SS, both K-major, N = 64)    -> TMEM [128 h + 64, 128 h + 128)
//       dV  += P^T_h dO_h       (TS: P^T_h bf16 in TMEM, dO_h MN-major) -> [320,384)
//       dK  += dS^T_h Q_h       (SS: dS^T_h K-major in smem, Q_h MN-major) -> [384,448)
//     and after half B: dQ_j = dS K (SS: dS MN-major = the same smem, K MN-major) -> [448,512);
//     the softmax warps of one half overlap the other half's MMAs
//   warp 2        : TMEM allocator (512 columns)
//   warps 4..11   : thread = key row r (TMEM lane r), warps 4-7 query half A, 8-11 half B
//                   (two warps per SM sub-partition): P^T_h, dS^T_h of block j,
//                   P^T_h -> TMEM (bf16 pairs), dS^T_h -> smem (SW128, double-buffered);
//   warps 12..15  : thread = query row of block j: dQ_j c -> smem -> TMA reduce-add into dq_acc (fp32);
//                   at the item's end (thread = key row) dV and dK c -> dqkv (bf16)
// The same TMA tile [128 rows][64 bf16] (one SW128 atom) is a K-major operand when
// the contraction runs over head dim and an MN-major one when it runs over tokens.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);
bool make_tmap_f32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols, CUtensorMapSwizzle swz);

namespace {

#ifndef ORBIT2_BWD_NODQ
#define ORBIT2_BWD_NODQ 0   // experiment: skip the dQ atomics (wrong dQ; timing only)
#endif
#ifndef ORBIT2_BWD_PF
#define ORBIT2_BWD_PF 1     // prefetch the next block's lse2 / Delta into registers (off the critical path)
#endif
#ifndef ORBIT2_BWD_NOSM
#define ORBIT2_BWD_NOSM 0   // experiment: skip the exponentials (wrong P; timing only)
#endif

constexpr int DH = 64;
constexpr int TILE = 128 * DH * 2;          // 16 KB: one SW128 atom of 128 rows
constexpr int QST = 2;                      // Q_j / dO_j ring
constexpr int KVST = 2;                     // K / V ring (next item prefetched)
constexpr int IRING = 4;
constexpr int THREADS = 512;
// TMEM columns: per query half h (64 queries): S^T_h at 128 h, dP^T_h at 128 h + 64;
// P^T_h (bf16 pairs) at 256 + 32 h; the dV, dK accumulators; dQ of the block
constexpr uint32_t C_S = 0, C_DP = 64, C_P = 256, C_DV = 320, C_DK = 384, C_DQ = 448;
constexpr int DQ_STG = 4 * 32 * 32 * 4;       // dQ staging: 4 warps x one box [32 rows][32 fp32] (SW128)
constexpr int DS_BYTES = 2 * TILE;            // dS^T [128 keys][128 q] as 2 atoms; double-buffered
constexpr int SMEM = KVST * 2 * TILE + QST * 2 * TILE + 2 * DS_BYTES + DQ_STG + 2 * 2 * 2 * 64 * 4 + 1024 + 512;

struct __align__(16) BItem {
  int64_t base;     // first row of the tile's tokens
  int n, k0, nq, h;
};

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ BItem bitem(const ChunkDev& ch, int heads, int id) {
  const int per_b = ch.nqb * heads;        // item = (key block fastest, head, sample)
  BItem it;
  const int b = id / per_b;
  const int r = id - b * per_b;
  it.h = r / ch.nqb;
  const int g = ch.qb0 + (r - it.h * ch.nqb);
  const DevTile t = ch.tiles[ch.qblk_tile[g]];
  it.k0 = (g - t.qb_off) * 128;
  it.n = t.n_tokens;
  it.nq = (it.n + 127) / 128;
  it.base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  return it;
}

__device__ __forceinline__ BItem take(const BItem* sItem, uint64_t* full, uint64_t* empty, uint32_t li) {
  const uint32_t s = li % IRING;
  tc::mbar_wait(&full[s], (li / IRING) & 1);
  const BItem it = sItem[s];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) tc::mbar_arrive(&empty[s]);
  return it;
}

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                    const __grid_constant__ CUtensorMap tdq,
                    const float* __restrict__ lse, const float* __restrict__ delta, int64_t ld_stat,
                    float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, ChunkDev ch, int D, int heads,
                    int n_items) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;                               // [KVST][TILE]
  uint8_t* sV = sK + KVST * TILE;                   // [KVST][TILE]
  uint8_t* sQ = sV + KVST * TILE;                   // [QST][TILE]
  uint8_t* sDO = sQ + QST * TILE;                   // [QST][TILE]
  uint8_t* sDS = sDO + QST * TILE;                  // [2 (block parity)][DS_BYTES]
  uint8_t* sDQ = sDS + 2 * DS_BYTES;                // [4 warps][32 rows][128 B]
  float* sL = reinterpret_cast<float*>(sDQ + DQ_STG);   // [2 halves][2 parity][64] lse2 of the half's queries
  float* sDl = sL + 2 * 2 * 64;                     // [2 halves][2 parity][64] Delta
  BItem* sItem = reinterpret_cast<BItem*>(sDl + 2 * 2 * 64);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sItem + IRING);
  uint64_t* kv_full = bar;                          // [KVST]
  uint64_t* kv_empty = kv_full + KVST;              // [KVST]
  uint64_t* q_full = kv_empty + KVST;               // [QST]
  uint64_t* q_empty = q_full + QST;                 // [QST]
  uint64_t* s_full = q_empty + QST;                 // [2 halves] S^T_h, dP^T_h in TMEM
  uint64_t* p_full = s_full + 2;                    // [2 halves] P^T_h (TMEM) and dS^T_h (smem) written
  uint64_t* dq_full = p_full + 2;
  uint64_t* dq_free = dq_full + 1;
  uint64_t* dkv_full = dq_free + 1;
  uint64_t* dkv_free = dkv_full + 1;
  uint64_t* it_full = dkv_free + 1;                 // [IRING]
  uint64_t* it_empty = it_full + IRING;             // [IRING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(it_empty + IRING);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tqkv);
    tc::prefetch_tmap(&tdo);
    tc::prefetch_tmap(&tdq);
    for (int s = 0; s < KVST; ++s) {
      tc::mbar_init(&kv_full[s], 1);
      tc::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < QST; ++s) {
      tc::mbar_init(&q_full[s], 1);
      tc::mbar_init(&q_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      tc::mbar_init(&s_full[h], 1);
      tc::mbar_init(&p_full[h], 128);
    }
    tc::mbar_init(dq_full, 1);
    tc::mbar_init(dq_free, 128);
    tc::mbar_init(dkv_full, 1);
    tc::mbar_init(dkv_free, 128);
    for (int s = 0; s < IRING; ++s) {
      tc::mbar_init(&it_full[s], 1);
      tc::mbar_init(&it_empty[s], 13);   // MMA warp + 8 softmax warps + 4 dQ warps
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    __syncwarp();
    tc::tmem_alloc(tmem_slot, 512);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float cs = rsqrtf((float)DH);                    // c = 1/sqrt(d)
  const float sl = 1.4426950408889634f * cs;             // log2(e) c

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t li = 0, gq = 0;
      for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const BItem it = bitem(ch, heads, id);
        {
          const uint32_t s = li % IRING;
          tc::mbar_wait(&it_empty[s], ((li / IRING) & 1) ^ 1);
          sItem[s] = it;
          tc::mbar_arrive(&it_full[s]);
        }
        const int32_t y0 = (int32_t)it.base;
        const uint32_t kv = li % KVST;
        tc::mbar_wait(&kv_empty[kv], ((li / KVST) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&kv_full[kv], 2 * TILE);
        tc::tma_load_2d(&tqkv, sK + kv * TILE, &kv_full[kv], D + it.h * DH, y0 + it.k0);
        tc::tma_load_2d(&tqkv, sV + kv * TILE, &kv_full[kv], 2 * D + it.h * DH, y0 + it.k0);
        for (int j = 0; j < it.nq; ++j, ++gq) {
          const uint32_t s = gq % QST;
          tc::mbar_wait(&q_empty[s], ((gq / QST) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&q_full[s], 2 * TILE);
          tc::tma_load_2d(&tqkv, sQ + s * TILE, &q_full[s], it.h * DH, y0 + j * 128);
          tc::tma_load_2d(&tdo, sDO + s * TILE, &q_full[s], it.h * DH, y0 + j * 128);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp walks the loop; one lane issues) ----------------
    // Per query block j, in halves h = A (queries 0-63), B (64-127):
    //   SP_h(j) : S^T_h = K Q_h^T, dP^T_h = V dO_h^T                  (needs Q_j / dO_j)
    //   G_A(j)  : dV += P^T_A dO_A, dK += dS^T_A Q_A                    (needs p_full A)
    //   G_B(j)  : dV += P^T_B dO_B, dK += dS^T_B Q_B, dQ_j = dS_j K       (needs p_full B)
    // issued SP_A(j) SP_B(j) | G_A(j) SP_A(j+1) | G_B(j) SP_B(j+1) | ...: the softmax warps
    // work on one half while the tensor core runs the other half's MMAs.  dS^T is
    // double-buffered by block parity (G_B(j) reads both halves of block j's).
    constexpr uint32_t id_sp = tc::idesc_bf16(128, 64, 0, 0);    // S^T_h, dP^T_h: K-major x K-major, N = 64
    constexpr uint32_t id_kb = tc::idesc_bf16(128, DH, 0, 1);    // dV, dK: A K-major, B MN-major
    constexpr uint32_t id_mm = tc::idesc_bf16(128, DH, 1, 1);    // dQ: A (dS) MN-major, B (K) MN-major
    const uint32_t k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV), q_addr = tc::smem_u32(sQ);
    const uint32_t do_addr = tc::smem_u32(sDO), ds_addr = tc::smem_u32(sDS);
    uint32_t li = 0, gq = 0;
    // live = the half holds a valid query (a last block of <= 64 queries skips half B's MMAs;
    // its commits still arrive so every barrier phase advances)
    auto issue_sp = [&](uint32_t kv, uint32_t s, int h, bool live) {   // elected lane
      const uint64_t kd = tc::sdesc(k_addr + kv * TILE, 16, 1024, tc::SW_128B);
      const uint64_t vd = tc::sdesc(v_addr + kv * TILE, 16, 1024, tc::SW_128B);
      const uint64_t qd = tc::sdesc(q_addr + s * TILE + h * (TILE / 2), 16, 1024, tc::SW_128B);
      const uint64_t dod = tc::sdesc(do_addr + s * TILE + h * (TILE / 2), 16, 1024, tc::SW_128B);
      if (live) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16_ss(tmem + h * 128 + C_S, kd + kk * 2, qd + kk * 2, id_sp, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc::mma_bf16_ss(tmem + h * 128 + C_DP, vd + kk * 2, dod + kk * 2, id_sp, kk > 0);
      }
      tc::mma_commit(&s_full[h]);
    };
    auto issue_g = [&](uint32_t kv, uint32_t s, uint32_t dsb, int h, bool first, bool live) {   // elected lane
      const uint64_t q_mn = tc::sdesc(q_addr + s * TILE + h * (TILE / 2), TILE, 1024, tc::SW_128B);
      const uint64_t do_mn = tc::sdesc(do_addr + s * TILE + h * (TILE / 2), TILE, 1024, tc::SW_128B);
      const uint64_t ds_k = tc::sdesc(ds_addr + dsb * DS_BYTES + h * TILE, 16, 1024, tc::SW_128B);
#pragma unroll
      for (int kk = 0; kk < 4 && live; ++kk) {          // K = 64 queries of the half, 16 per MMA
        const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
        const uint32_t mn_adv = (uint32_t)(kk * 2048) >> 4;
        tc::mma_bf16_ts(tmem + C_DV, tmem + C_P + h * 32 + kk * 8, do_mn + mn_adv, id_kb, acc);
        tc::mma_bf16_ss(tmem + C_DK, ds_k + ((uint32_t)(kk * 32) >> 4), q_mn + mn_adv, id_kb, acc);
      }
      if (h == 1) {                                      // dQ_j = dS_j K: K = 128 keys
        const uint64_t k_mn = tc::sdesc(k_addr + kv * TILE, TILE, 1024, tc::SW_128B);
        const uint64_t ds_mn = tc::sdesc(ds_addr + dsb * DS_BYTES, TILE, 1024, tc::SW_128B);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t mn_adv = (uint32_t)(kk * 2048) >> 4;
          tc::mma_bf16_ss(tmem + C_DQ, ds_mn + mn_adv, k_mn + mn_adv, id_mm, kk > 0);
        }
      }
    };
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      const BItem it = take(sItem, it_full, it_empty, li);
      const uint32_t kv = li % KVST;
      tc::mbar_wait(&kv_full[kv], (li / KVST) & 1);
      for (int j = 0; j < it.nq; ++j, ++gq) {
        const uint32_t s = gq % QST;
        const uint32_t dsb = gq & 1;
        if (j == 0) {                                    // the item's first block: both halves' S, dP
          tc::mbar_wait(&q_full[s], (gq / QST) & 1);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            issue_sp(kv, s, 0, true);
            issue_sp(kv, s, 1, j * 128 + 64 < it.n);
          }
          __syncwarp();
        }
        const bool more = j + 1 < it.nq;
        const uint32_t s1 = (gq + 1) % QST;
        // half A of block j done by the softmax warps
        tc::mbar_wait(&p_full[0], gq & 1);
        if (j == 0 && li > 0) tc::mbar_wait(dkv_free, (li - 1) & 1);   // dK / dV of the last item read
        if (more) tc::mbar_wait(&q_full[s1], ((gq + 1) / QST) & 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          issue_g(kv, s, dsb, 0, j == 0, true);
          if (more) issue_sp(kv, s1, 0, true);
        }
        __syncwarp();
        // half B of block j
        tc::mbar_wait(&p_full[1], gq & 1);
        if (gq > 0) tc::mbar_wait(dq_free, (gq - 1) & 1);              // dQ of the last block read
        tc::tc_fence_after();
        if (tc::elect_one()) {
          issue_g(kv, s, dsb, 1, false, j * 128 + 64 < it.n);
          tc::mma_commit(dq_full);
          tc::mma_commit(&q_empty[s]);
          if (!more) {
            tc::mma_commit(dkv_full);
            tc::mma_commit(&kv_empty[kv]);
          } else {
            issue_sp(kv, s1, 1, (j + 1) * 128 + 64 < it.n);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------- P^T_h / dS^T_h (thread = key row; warps 4-7 half A, 8-11 half B) ----------------
    // Two warps per SM sub-partition (one per half) run concurrently.
    const int h = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(q4 * 32) << 16);
    const int sw = r & 7;
    float* hL = sL + h * 2 * 64;
    float* hDl = sDl + h * 2 * 64;
    uint32_t li = 0, gq = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      const BItem it = take(sItem, it_full, it_empty, li);
      const bool kval = it.k0 + r < it.n;
      // lse2 / Delta of query j*128 + 64 h + r (threads r < 64), block j + 1's loaded while
      // block j computes (a global load's latency is off the softmax critical path)
      auto ld_stats = [&](int j, float& l, float& dl) {
        const int q = j * 128 + h * 64 + r;
        const int64_t o = (int64_t)it.h * ld_stat + it.base + q;
        const bool ok = r < 64 && j < it.nq && q < it.n;
        l = ok ? -__ldg(lse + o) : 0.f;      // staged negated: the inner loop is FFMA2 / FADD2
        dl = ok ? -__ldg(delta + o) : 0.f;
      };
      float nl, nd;
      ld_stats(0, nl, nd);
      for (int j = 0; j < it.nq; ++j, ++gq) {
        const int buf = gq & 1;
        if (!ORBIT2_BWD_PF) ld_stats(j, nl, nd);
        if (r < 64) {   // stage this half's lse2 / Delta
          hL[buf * 64 + r] = nl;
          hDl[buf * 64 + r] = nd;
        }
        if (ORBIT2_BWD_PF) ld_stats(j + 1, nl, nd);
        asm volatile("bar.sync %0, 128;" ::"r"(1 + h) : "memory");
        const float* nL = hL + buf * 64;                  // -lse2 of the half's queries
        const float* nD = hDl + buf * 64;                 // -Delta
        const int qv = it.n - j * 128 - h * 64;            // valid queries in this half
        // no masking unless this key block or this query half runs past the tile end
        // (block-uniform): invalid keys / queries get P = dS = 0
        const bool fast = it.k0 + 128 <= it.n && qv >= 64;
        uint8_t* atom = sDS + (gq & 1) * DS_BYTES + h * TILE + r * 128;   // half h = atom h of dS^T
        tc::mbar_wait(&s_full[h], gq & 1);
        tc::tc_fence_after();
        const uint32_t sb = lb + h * 128;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          if (qv <= 0) break;                              // a half without queries: nothing to do
          uint32_t sr[16], dr[16];
          tc::tmem_ld16(sb + C_S + c0, sr);
          tc::tmem_ld16(sb + C_DP + c0, dr);
          tc::tmem_ld_wait();
          uint32_t pk[8], dk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 4) {
            const float4 nl = *reinterpret_cast<const float4*>(nL + c0 + e);
            const float4 nd = *reinterpret_cast<const float4*>(nD + c0 + e);
            const float2 x0 = tc::fma2(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])),
                                       tc::splat2(sl), make_float2(nl.x, nl.y));
            const float2 x1 = tc::fma2(make_float2(__uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3])),
                                       tc::splat2(sl), make_float2(nl.z, nl.w));
            float2 p0, p1;
            if (ORBIT2_BWD_NOSM) {
              p0 = x0;
              p1 = x1;
            } else {
              p0 = make_float2(ex2f(x0.x), ex2f(x0.y));
              p1 = make_float2(ex2f(x1.x), ex2f(x1.y));
            }
            if (!fast) {
              const int lim = kval ? qv : 0;
              p0.x = c0 + e < lim ? p0.x : 0.f;
              p0.y = c0 + e + 1 < lim ? p0.y : 0.f;
              p1.x = c0 + e + 2 < lim ? p1.x : 0.f;
              p1.y = c0 + e + 3 < lim ? p1.y : 0.f;
            }
            const float2 d0 = tc::mul2(p0, tc::add2(make_float2(__uint_as_float(dr[e]), __uint_as_float(dr[e + 1])),
                                                    make_float2(nd.x, nd.y)));
            const float2 d1 = tc::mul2(p1, tc::add2(make_float2(__uint_as_float(dr[e + 2]),
                                                                __uint_as_float(dr[e + 3])),
                                                    make_float2(nd.z, nd.w)));
            pk[e / 2] = tc::pack_bf16(p0.x, p0.y);
            pk[e / 2 + 1] = tc::pack_bf16(p1.x, p1.y);
            dk[e / 2] = tc::pack_bf16(d0.x, d0.y);
            dk[e / 2 + 1] = tc::pack_bf16(d1.x, d1.y);
          }
          tc::tmem_st8(lb + C_P + h * 32 + c0 / 2, pk);
          const int cb = c0 >> 3;
          *reinterpret_cast<uint4*>(atom + ((cb ^ sw) << 4)) = make_uint4(dk[0], dk[1], dk[2], dk[3]);
          *reinterpret_cast<uint4*>(atom + (((cb + 1) ^ sw) << 4)) = make_uint4(dk[4], dk[5], dk[6], dk[7]);
        }
        tc::tmem_st_wait();
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        tc::mbar_arrive(&p_full[h]);
      }
    }
  } else if (warp >= 12) {
    // ---------------- dQ_j c -> dq_acc: staged in smem, one TMA reduce-add per 32 x 32 box ----------------
    // (rows of queries past the tile end hold exact zeros: their dS columns are 0)
    const int q4 = warp & 3;
    const uint32_t lb = tmem + ((uint32_t)(q4 * 32) << 16);
    uint8_t* stg = sDQ + q4 * 4096;
    uint32_t li = 0, gq = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      const BItem it = take(sItem, it_full, it_empty, li);
      for (int j = 0; j < it.nq; ++j, ++gq) {
        tc::mbar_wait(dq_full, gq & 1);
        tc::tc_fence_after();
        uint32_t v[2][32];
        tc::tmem_ld32(lb + C_DQ, v[0]);
        tc::tmem_ld32(lb + C_DQ + 32, v[1]);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(dq_free);                      // TMEM dQ may take the next block's
        const int row0 = j * 128 + q4 * 32;          // first query of this warp's slice
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (lane == 0) tc::bulk_wait_read<0>();     // the previous reduce has read the staging box
          __syncwarp();
          uint8_t* row = stg + lane * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<float4*>(row + ((u ^ (lane & 7)) << 4)) =
                make_float4(__uint_as_float(v[half][4 * u]) * cs, __uint_as_float(v[half][4 * u + 1]) * cs,
                            __uint_as_float(v[half][4 * u + 2]) * cs, __uint_as_float(v[half][4 * u + 3]) * cs);
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && row0 < it.n && !ORBIT2_BWD_NODQ) {
            tc::tma_reduce_add_2d(&tdq, stg, it.h * DH + half * 32, (int32_t)(it.base + row0));
            tc::bulk_commit();
          }
        }
      }
      // item end (off the softmax warps' path): dV and dK c of key row r -> dqkv
      const int r = q4 * 32 + lane;
      const bool kval = it.k0 + r < it.n;
      tc::mbar_wait(dkv_full, li & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int part = 0; part < 2; ++part) {             // 0: dV, 1: dK
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 32) {
          uint32_t v[32];
          tc::tmem_ld32(lb + (part ? C_DK : C_DV) + c0, v);
          tc::tmem_ld_wait();
          if (kval) {
            const float f = part ? cs : 1.f;
            __nv_bfloat16* dst = dqkv + (it.base + it.k0 + r) * (int64_t)(3 * D) + (part ? D : 2 * D) +
                                 it.h * DH + c0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              reinterpret_cast<uint4*>(dst)[u] =
                  make_uint4(tc::pack_bf16(__uint_as_float(v[8 * u]) * f, __uint_as_float(v[8 * u + 1]) * f),
                             tc::pack_bf16(__uint_as_float(v[8 * u + 2]) * f, __uint_as_float(v[8 * u + 3]) * f),
                             tc::pack_bf16(__uint_as_float(v[8 * u + 4]) * f, __uint_as_float(v[8 * u + 5]) * f),
                             tc::pack_bf16(__uint_as_float(v[8 * u + 6]) * f, __uint_as_float(v[8 * u + 7]) * f));
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(dkv_free);
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool launch_attention_bwd_tc(const void* qkv, const void* dout, int64_t rows, const float* lse, const float* delta,
                             int64_t ld_stat, float* dq_acc, void* dqkv, const ChunkDev& ch, int B, int D, int heads,
                             int d, cudaStream_t st) {
  if (d != DH) return false;
  CUtensorMap tq, tdo, tdq;
  if (!make_tmap_bf16(&tq, qkv, rows, 3LL * D, 3LL * D, 128, DH, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&tdo, dout, rows, D, D, 128, DH, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_f32(&tdq, dq_acc, rows, D, D, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(attn_bwd_kernel), SMEM, &attr_done)) return false;
  const int64_t n_items = (int64_t)ch.nqb * heads * B;
  if (n_items == 0) return true;
  if (n_items >= (int64_t)INT32_MAX) return false;
  const unsigned grid = (unsigned)std::min<int64_t>(n_items, num_sms());
  attn_bwd_kernel<<<grid, THREADS, SMEM, st>>>(tq, tdo, tdq, lse, delta, ld_stat, dq_acc,
                                               reinterpret_cast<__nv_bfloat16*>(dqkv), ch, D, heads, (int)n_items);
  return true;
}

}  // namespace orbit2
