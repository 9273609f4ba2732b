// attn3_tc.cu -- per-tile attention at head dim 64 on tcgen05: THREE 128-query
// tiles per CTA sharing 64-key K/V blocks.
//
// P:527 "self-attention is restricted within each tile"; P:595 Flash Attention.
// Same computation as attn_tc.cu (O = softmax(Q K^T / sqrt(d)) V over the keys of
// the same tile, online softmax with a conditional reference-max rescale, R17/R18)
// with a different block structure, chosen for head dim 64 where the
// exponentials (one per score, 256 tensor FLOPs each) and not the tensor core
// bound the kernel:
//   * key blocks of 64: a Q tile needs S (64 fp32 columns) + O (64) + P (32
//     columns of bf16 pairs) = 160 TMEM columns, so THREE Q tiles fit the 512
//     columns (two with 128-key blocks);
//   * three softmax warps per SM sub-partition (one per Q tile) instead of two:
//     while one warp loads S / takes its row max / waits for the previous PV,
//     the other two keep the MUFU busy (the 2-warp kernel spends ~40 % of each
//     block with both warps outside their exponential phase);
//   * 64 scores per thread per block: half the registers per row (no spills at
//     the 128-register budget of 512 threads), half the serial row-max chain.
// Roles (512 threads): warp 0 TMA producer + TMEM allocator, warps 1-3 one
// tcgen05.mma issuer per Q tile, warps 4-15 softmax (4 per Q tile, thread = query
// row = TMEM lane) with a TMA-store epilogue.  A work item = up to 3 consecutive
// 128-query blocks of one (tile, head, sample) (plan: groups of 3).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int DH = 64;                  // head dim (every shipped configuration)
constexpr int NQ = 3;                   // Q tiles per CTA
constexpr int KB = 64;                  // keys per block
constexpr int RB = DH * 2;              // bytes per smem row (one 128-byte swizzle atom)
constexpr int QT = 128 * RB;            // bytes of a Q tile (128 rows)
constexpr int KVT = KB * RB;            // bytes of a K or V block
constexpr int QBUF = 2;                 // Q tile sets (the next item's Q is prefetched)
#ifndef ORBIT2_ATTN3_KVST
#define ORBIT2_ATTN3_KVST 3
#endif
constexpr int KST = ORBIT2_ATTN3_KVST, VST = ORBIT2_ATTN3_KVST;   // K / V ring slots
constexpr int TCOLS = KB + DH + KB / 2; // S | O | P per Q tile (160)
constexpr int CTRL_WARPS = 4;           // producer + 3 MMA issuers (one warpgroup)
constexpr int THREADS = 32 * CTRL_WARPS + 128 * NQ;   // 512
constexpr int OST_WARP = 32 * RB;       // epilogue staging per softmax warp (32 rows)
constexpr int IRING = 4;
constexpr int SMEM = QBUF * NQ * QT + (KST + VST) * KVT + 4 * NQ * OST_WARP + 1024 + 512;
constexpr float kRescaleLog2 = 8.0f;    // conditional rescale threshold (attn_tc.cu)
#ifndef ORBIT2_ATTN3_POLY
#define ORBIT2_ATTN3_POLY 2
#endif
constexpr int kPolyPer16 = ORBIT2_ATTN3_POLY;   // exponentials per 16 on the FMA pipe
#ifndef ORBIT2_ATTN3_DESYNC_CLK
#define ORBIT2_ATTN3_DESYNC_CLK 0
#endif
#ifndef ORBIT2_ATTN3_REGREALLOC
#define ORBIT2_ATTN3_REGREALLOC 1
#endif
static_assert(NQ * TCOLS <= 512, "TMEM");
static_assert(SMEM <= 227 * 1024, "shared memory");

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ffma2(float& a, float& b, float s, float t) {
  asm("{\n\t.reg .b64 x, sc, tt;\n\t"
      "mov.b64 x, {%0, %1};\n\t"
      "mov.b64 sc, {%2, %2};\n\t"
      "mov.b64 tt, {%3, %3};\n\t"
      "fma.rn.f32x2 x, x, sc, tt;\n\t"
      "mov.b64 {%0, %1}, x;\n\t}"
      : "+f"(a), "+f"(b)
      : "f"(s), "f"(t));
}
// 2^x on the FMA pipe for a pair (degree-3 fit of 2^f on [-1/2, 1/2], exponent
// field add; |rel err| <= 1.0e-4 < bf16's 2^-9; x clamped at -125) -- attn_tc.cu
__device__ __forceinline__ float2 ex2_poly2(float x0, float x1) {
  float2 x = make_float2(fmaxf(x0, -125.0f), fmaxf(x1, -125.0f));
  const float2 t = tc::add2(x, tc::splat2(12582912.0f));
  const float2 f = tc::fma2(tc::add2(t, tc::splat2(-12582912.0f)), tc::splat2(-1.0f), x);
  float2 p = tc::fma2(tc::splat2(0.05500886f), f, tc::splat2(0.24221101f));
  p = tc::fma2(p, f, tc::splat2(0.69328296f));
  p = tc::fma2(p, f, tc::splat2(1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

struct __align__(16) Item {
  int64_t base;     // first row of the tile's tokens in the packed workspace
  int n, q0, nq, nkb, h, pad_;
};

__device__ __forceinline__ Item item_info(const ChunkDev& ch, int heads, int id) {
  const int np = ch.core_pairs ? ch.nqgc : ch.nqg;
  const int per_b = np * heads;                       // item = (group fastest, head, sample)
  Item it;
  const int b = id / per_b;
  const int r = id - b * per_b;
  it.h = r / np;
  const int g = r - it.h * np;
  const int e = ch.core_pairs ? ch.qg3c[ch.qgc0 + g] : ch.qg3[ch.qg0 + g];
  const DevTile t = ch.tiles[e >> 16];
  it.q0 = ((e >> 2) & 0x3FFF) * 128;
  it.nq = (e & 3) + 1;
  it.n = t.n_tokens;
  it.base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  it.nkb = (it.n + KB - 1) / KB;
  return it;
}

__device__ __forceinline__ Item take_item(const Item* sItem, uint64_t* it_full, uint64_t* it_empty, uint32_t li) {
  const uint32_t is = li % IRING;
  tc::mbar_wait(&it_full[is], (li / IRING) & 1);
  const Item it = sItem[is];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) tc::mbar_arrive(&it_empty[is]);
  return it;
}

__global__ void __launch_bounds__(THREADS, 1)
    attn3_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmkv,
                    const __grid_constant__ CUtensorMap tmo, __nv_bfloat16* __restrict__ out, ChunkDev ch, int D,
                    int heads, int n_items, long long* __restrict__ tl) {
  // tl: debug timeline (-DORBIT2_ATTN3_TIMELINE): clock64 of CTA 0, [role][block][event]
#ifdef ORBIT2_ATTN3_TIMELINE
#define TL3(role, blk, ev)                                                                        \
  do {                                                                                            \
    if (tl != nullptr && blockIdx.x == 0 && (blk) < 64) tl[((role) * 64 + (blk)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define TL3(role, blk, ev) \
  do {                     \
  } while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                               // [QBUF][NQ][QT]
  uint8_t* sK = sQ + QBUF * NQ * QT;                // [KST][KVT]
  uint8_t* sV = sK + KST * KVT;                     // [VST][KVT]
  uint8_t* sOst = sV + VST * KVT;                   // [4 * NQ][OST_WARP]
  Item* sItem = reinterpret_cast<Item*>(sOst + 4 * NQ * OST_WARP);   // [IRING]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sItem + IRING);
  uint64_t* q_full = bar;                           // [QBUF]
  uint64_t* q_empty = q_full + QBUF;                // [QBUF]
  uint64_t* k_full = q_empty + QBUF;                // [KST]
  uint64_t* k_empty = k_full + KST;                 // [KST]
  uint64_t* v_full = k_empty + KST;                 // [VST]
  uint64_t* v_empty = v_full + VST;                 // [VST]
  uint64_t* s_full = v_empty + VST;                 // [NQ] S in TMEM
  uint64_t* s_free = s_full + NQ;                   // [NQ] softmax holds S in registers
  uint64_t* p_full = s_free + NQ;                   // [NQ] P written (+ O rescaled)
  uint64_t* p_free = p_full + NQ;                   // [NQ] PV done (P free, O complete)
  uint64_t* o_free = p_free + NQ;                   // [NQ] epilogue has read O
  uint64_t* it_full = o_free + NQ;                  // [IRING]
  uint64_t* it_empty = it_full + IRING;             // [IRING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(it_empty + IRING);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmq);
    tc::prefetch_tmap(&tmkv);
    for (int s = 0; s < QBUF; ++s) {
      tc::mbar_init(&q_full[s], 1);
      tc::mbar_init(&q_empty[s], NQ);
    }
    for (int s = 0; s < KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], NQ);
    }
    for (int s = 0; s < VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], NQ);
    }
    for (int s = 0; s < NQ; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&s_free[s], 128);
      tc::mbar_init(&p_full[s], 128);
      tc::mbar_init(&p_free[s], 1);
      tc::mbar_init(&o_free[s], 128);
    }
    for (int s = 0; s < IRING; ++s) {
      tc::mbar_init(&it_full[s], 1);
      tc::mbar_init(&it_empty[s], NQ + 4 * NQ);     // MMA-issuer warps + softmax warps
    }
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    __syncwarp();
    tc::tmem_alloc(tmem_slot, 512);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the control warpgroup needs few registers: give them to the softmax warpgroups
  if (ORBIT2_ATTN3_REGREALLOC) {
    if (warp < CTRL_WARPS) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 152;" ::: "memory");
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t li = 0, gk = 0, gv = 0;
      for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const Item it = item_info(ch, heads, id);
        {
          const uint32_t is = li % IRING;
          tc::mbar_wait(&it_empty[is], ((li / IRING) & 1) ^ 1);
          sItem[is] = it;
          tc::mbar_arrive(&it_full[is]);
        }
        const int32_t y0 = (int32_t)it.base;
        const uint32_t qb = li % QBUF;
        tc::mbar_wait(&q_empty[qb], ((li / QBUF) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qb], it.nq * QT);
        for (int qt = 0; qt < it.nq; ++qt)
          tc::tma_load_2d(&tmq, sQ + (qb * NQ + qt) * QT, &q_full[qb], it.h * DH, y0 + it.q0 + qt * 128);
        auto load_k = [&](int j) {
          const uint32_t st = gk % KST;
          tc::mbar_wait(&k_empty[st], ((gk / KST) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&k_full[st], KVT);
          tc::tma_load_2d(&tmkv, sK + st * KVT, &k_full[st], D + it.h * DH, y0 + j * KB);
          ++gk;
        };
        auto load_v = [&](int j) {
          const uint32_t st = gv % VST;
          tc::mbar_wait(&v_empty[st], ((gv / VST) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&v_full[st], KVT);
          tc::tma_load_2d(&tmkv, sV + st * KVT, &v_full[st], 2 * D + it.h * DH, y0 + j * KB);
          ++gv;
        };
        load_k(0);
        for (int j = 0; j < it.nkb; ++j) {
          if (j + 1 < it.nkb) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp <= NQ) {
    // ---------------- MMA issuers: warp 1 + qt -> Q tile qt ----------------
    const int qt = warp - 1;
    constexpr uint32_t id_s = tc::idesc_bf16(128, KB, 0, 0);   // Q K-major, K K-major
    constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);   // P (TMEM) K-major, V MN-major
    const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
    const uint32_t d_s = tmem + qt * TCOLS, d_o = d_s + KB, a_p = d_s + KB + DH;
    uint32_t li = 0, gk = 0, gv = 0, ns = 0, np = 0, ni = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      const Item it = take_item(sItem, it_full, it_empty, li);
      const bool active = qt < it.nq;
      const uint32_t qb = li % QBUF;
      tc::mbar_wait(&q_full[qb], (li / QBUF) & 1);
      auto issue_s = [&](bool last) {   // S = Q K_j^T
        const uint32_t st = gk % KST;
        tc::mbar_wait(&k_full[st], (gk / KST) & 1);
        if (active) {
          if (lane == 0) TL3(3 + qt, ns, 0);
          if (ns >= 1) tc::mbar_wait(&s_free[qt], (ns - 1) & 1);
          if (lane == 0) TL3(3 + qt, ns, 1);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint64_t qd0 = tc::sdesc(q_addr + (qb * NQ + qt) * QT, 16, 8 * RB, tc::SW_128B);
            const uint64_t kd0 = tc::sdesc(k_addr + st * KVT, 16, 8 * RB, tc::SW_128B);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)   // K = 16 dims per MMA: +32 bytes inside the atom
              tc::mma_bf16_ss(d_s, qd0 + (uint32_t)(kk * 2), kd0 + (uint32_t)(kk * 2), id_s, kk > 0);
            tc::mma_commit(&s_full[qt]);
            tc::mma_commit(&k_empty[st]);
            if (last) tc::mma_commit(&q_empty[qb]);
          }
          __syncwarp();
          ++ns;
        } else {
          if (lane == 0) {
            tc::mbar_arrive(&k_empty[st]);
            if (last) tc::mbar_arrive(&q_empty[qb]);
          }
          __syncwarp();
        }
        ++gk;
      };
      issue_s(it.nkb == 1);
      for (int j = 0; j < it.nkb; ++j) {
        if (j + 1 < it.nkb) issue_s(j + 2 == it.nkb);   // S_{j+1} overlaps the softmax of block j
        const uint32_t st = gv % VST;
        tc::mbar_wait(&v_full[st], (gv / VST) & 1);
        if (active) {
          if (j == 0 && ni >= 1) tc::mbar_wait(&o_free[qt], (ni - 1) & 1);
          const uint64_t vd0 = tc::sdesc(v_addr + st * KVT, KVT, 8 * RB, tc::SW_128B);
          if (lane == 0) TL3(3 + qt, np, 2);
          tc::mbar_wait(&p_full[qt], np & 1);
          if (lane == 0) TL3(3 + qt, np, 3);
          tc::tc_fence_after();
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk)   // K = 16 keys per MMA: 8 P columns, 16 V rows
              tc::mma_bf16_ts(d_o, a_p + kk * 8, vd0 + (uint32_t)((kk * 16 * RB) >> 4), id_o, (j > 0 || kk > 0) ? 1u : 0u);
            tc::mma_commit(&p_free[qt]);
            tc::mma_commit(&v_empty[st]);
          }
          __syncwarp();
          ++np;
        } else {
          if (lane == 0) tc::mbar_arrive(&v_empty[st]);
          __syncwarp();
        }
        ++gv;
      }
      if (active) ++ni;
    }
  } else {
    // ---------------- softmax / epilogue: thread = query row i of Q tile qt ----------------
    const int sidx = warp - CTRL_WARPS;
    const int qt = sidx / 4;
    const int q = warp & 3;                        // TMEM lane quarter of this warp
    const int i = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + qt * TCOLS;
    const uint32_t s_addr = lane_base, o_addr = lane_base + KB, p_tm = lane_base + KB + DH;
    const float sl = 1.4426950408889634f * rsqrtf((float)DH);   // log2(e)/sqrt(d)
    uint32_t cs = 0;                               // blocks processed by this Q tile (all items)
    uint32_t li = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      const Item it = take_item(sItem, it_full, it_empty, li);
      if (qt >= it.nq) continue;
      float m_ref = -INFINITY, l_run = 0.f;
      const bool row_valid = it.q0 + qt * 128 + i < it.n;
      const bool tlr = q == 0 && lane == 0;
      for (int j = 0; j < it.nkb; ++j, ++cs) {
        if (tlr) TL3(qt, cs, 0);
        tc::mbar_wait(&s_full[qt], cs & 1);
        if (tlr) TL3(qt, cs, 1);
        tc::tc_fence_after();
        float sv[KB];
        {
          uint32_t* r = reinterpret_cast<uint32_t*>(sv);
          tc::tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(r));
          tc::tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
          tc::tmem_ld_wait();
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&s_free[qt]);
        if (tlr) TL3(qt, cs, 2);
        const int kvalid = it.n - j * KB;
        if (kvalid < KB) {
#pragma unroll
          for (int c = 0; c < KB; ++c)
            if (c >= kvalid) sv[c] = -INFINITY;
        }
        float m0 = sv[0], m1 = sv[1], m2 = sv[2], m3 = sv[3];
#pragma unroll
        for (int c = 4; c < KB; c += 4) {
          m0 = fmaxf(m0, sv[c]); m1 = fmaxf(m1, sv[c + 1]);
          m2 = fmaxf(m2, sv[c + 2]); m3 = fmaxf(m3, sv[c + 3]);
        }
        const float m_blk = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl;
        // PV_{j-1} done: P columns free, O complete (first block of the item: nothing pending)
        bool pv_done = j == 0;
        auto wait_pv = [&]() {
          if (!pv_done) {
            tc::mbar_wait(&p_free[qt], (cs - 1) & 1);
            tc::tc_fence_after();
            pv_done = true;
          }
        };
        if (j == 0) {
          // the previous item's last PV must be done before P is overwritten
          if (cs > 0) {
            tc::mbar_wait(&p_free[qt], (cs - 1) & 1);
            tc::tc_fence_after();
          }
          m_ref = m_blk;
        } else if (__any_sync(0xffffffffu, row_valid && m_blk > m_ref + kRescaleLog2)) {
          // conditional rescale (R18): O and l by 2^(m_ref - m_new), warp-collective TMEM ld/st
          wait_pv();
          const float m_new = fmaxf(m_blk, m_ref);
          const float alpha = ex2(m_ref - m_new);
          l_run *= alpha;
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 16) {
            uint32_t r[16];
            tc::tmem_ld16(o_addr + c0, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tc::tmem_st16(o_addr + c0, r);
          }
          m_ref = m_new;
        }
        if (tlr) TL3(qt, cs, 3);
        if (ORBIT2_ATTN3_DESYNC_CLK > 0 && j == 0 && qt > 0) {
          // stagger the Q tiles' exponential phases at the start of an item
          const long long t0 = clock64();
          while (clock64() - t0 < (long long)qt * ORBIT2_ATTN3_DESYNC_CLK) {
          }
        }
        wait_pv();
        if (tlr) TL3(qt, cs, 4);
        // p = 2^(s log2(e)/sqrt(d) - m_ref) -> bf16 P in TMEM (A operand of PV), fp32 row sums
        uint32_t pk[KB / 2];
        float2 rs[ORBIT2_ATTN3_RS_SPLIT];   // independent partial sums (no 32-long add chain)
#pragma unroll
        for (int u = 0; u < ORBIT2_ATTN3_RS_SPLIT; ++u) rs[u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < KB; e += 2) {
          float x0 = sv[e], x1 = sv[e + 1];
          ffma2(x0, x1, sl, -m_ref);
          float2 pr;
          if ((e & 15) < kPolyPer16) pr = ex2_poly2(x0, x1);
          else pr = make_float2(ex2(x0), ex2(x1));
          rs[(e / 2) % ORBIT2_ATTN3_RS_SPLIT] = tc::add2(rs[(e / 2) % ORBIT2_ATTN3_RS_SPLIT], pr);
          pk[e / 2] = tc::pack_bf16(pr.x, pr.y);
        }
#pragma unroll
        for (int u = 1; u < ORBIT2_ATTN3_RS_SPLIT; ++u) rs[0] = tc::add2(rs[0], rs[u]);
        tc::tmem_st32(p_tm, pk);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&p_full[qt]);
        if (tlr) TL3(qt, cs, 5);
        l_run += rs[0].x + rs[0].y;
      }
      // epilogue: O / l  (wait for the item's last PV)
      tc::mbar_wait(&p_free[qt], (cs - 1) & 1);
      tc::tc_fence_after();
      const float inv = 1.f / l_run;
      uint8_t* swb = sOst + (qt * 4 + q) * OST_WARP;   // this warp's 32-row slice (SW128 like the store box)
      auto swz = [](uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); };
      if (lane == 0) tc::bulk_wait_read<0>();          // the previous item's store has read the slice
      __syncwarp();
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld32(o_addr + c0, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4*>(swb + swz(lane * RB + (c0 + 8 * u) * 2)) =
              make_uint4(tc::pack_bf16(__uint_as_float(r[8 * u]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                         tc::pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                         tc::pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                         tc::pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&o_free[qt]);                  // O read: the next item's PV may accumulate
      const int row0 = it.q0 + qt * 128 + q * 32;    // first query row of this warp
      if (row0 + 32 <= it.n) {
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_2d(&tmo, swb, it.h * DH, (int32_t)(it.base + row0));
          tc::bulk_commit();
        }
      } else {
        __syncwarp();
        if (row0 + lane < it.n) {
#pragma unroll
          for (int c = 0; c < DH / 8; ++c)
            *reinterpret_cast<uint4*>(out + (it.base + row0 + lane) * (int64_t)D + it.h * DH + c * 8) =
                *reinterpret_cast<const uint4*>(swb + swz(lane * RB + c * 16));
        }
      }
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

extern long long* g_attn_timeline;   // attn_tc.cu: set by orbit2_debug_attn_timeline

bool launch_attention3_tc(const void* qkv, int64_t rows, void* out, const ChunkDev& ch, int B, int D, int heads,
                          cudaStream_t st) {
  CUtensorMap tmq, tmkv, tmo;
  if (!make_tmap_bf16(&tmq, qkv, rows, 3LL * D, 3LL * D, 128, DH, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&tmkv, qkv, rows, 3LL * D, 3LL * D, KB, DH, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&tmo, out, rows, D, D, 32, DH, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(attn3_tc_kernel), SMEM, &attr_done)) return false;
  const int64_t n_items = (int64_t)(ch.core_pairs ? ch.nqgc : ch.nqg) * heads * B;
  if (n_items == 0) return true;
  if (n_items >= (int64_t)INT32_MAX) return false;
  const unsigned grid = (unsigned)std::min<int64_t>(n_items, num_sms());
  attn3_tc_kernel<<<grid, THREADS, SMEM, st>>>(tmq, tmkv, tmo, reinterpret_cast<__nv_bfloat16*>(out), ch, D, heads,
                                               (int)n_items, g_attn_timeline);
  return true;
}

}  // namespace orbit2
