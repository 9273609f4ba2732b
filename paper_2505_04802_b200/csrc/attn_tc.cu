// attn_tc.cu -- per-tile multi-head self-attention on tcgen05 tensor cores.
//
// "self-attention is restricted within each tile"; P:583 / P:595 the
// paper runs Flash Attention.  For every (query block of 128 tokens of a
// tile, head, sample):
//     O = softmax(Q K^T / sqrt(d)) V     over the keys of the SAME tile only
// with an online (flash) softmax over key blocks of 128 (R17, R18).
//
// Persistent (one CTA per SM).  A work item is NQ = 2 query blocks of the same
// (tile, head, sample); they share every K/V block (FA4-style ping-pong of two
// Q tiles):
//   warp 0 lane 0 : TMA producer (Q tiles once; K_j and V_j into separate 2-slot
//                   rings, issued in consumption order K_{j+1} before V_j)
//   warps 1, 3    : tcgen05.mma issuers, one per Q tile t:
//                     S_j = Q_t K_j^T -> TMEM buffer (t, j&1)   [128 x 128 fp32]
//                     O_j = P_j V_j   -> same TMEM buffer        [128 x d   fp32]
//   warp 2        : TMEM allocator (NQ * 256 columns)
//   warps 4..     : softmax, 4 warps per Q tile; thread i owns query row i
//                   (TMEM lane i): pass A row max of S_j, fold O_{j-1} into a
//                   register accumulator (online-softmax rescale), pass B
//                   p = exp2(s*c - m) -> bf16 P_j in smem (SW128 K-major A
//                   operand), fp32 row sums.
// The tensor core computes S_{j+1} of one tile while the softmax warps of
// both tiles work on block j; 2 softmax warps per SM sub-partition hide each
// other's latency.  V is consumed MN-major straight from its TMA tile.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

long long* g_attn_timeline = nullptr;   // debug: set by orbit2_debug_attn_timeline

// Design choices measured on B200 (scripts/ab_kernels.py, C2 B = 64, attention ms):
//   ping-pong of the two Q tiles' exp phases (FA4 style)        27.2
//   two softmax warps per row (64 keys each), with ping-pong   25.9
//   both tiles' softmax concurrently, one warp per row          24.5   <- kept
//   + 4 of 16 exponentials on the FMA pipe (ex2_poly)           23.2
//   + packed f32x2 polynomial and row sums (fewer issue slots)  21.7
//     with 2 of 16 on the FMA pipe                              21.4   <- kept
// (ping-pong leaves one warp per SM sub-partition in an exp phase, which
// reaches ~70% of the MUFU rate; two concurrent warps reach ~90%).
// Skipping the row max (exponentiate against the reference max, check the
// block's row sum afterwards) was measured slower (C2: 26.0 vs 23.8 ms) and removed.

namespace {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (FA4's trick to offload the MUFU): x = j + f with j the
// nearest integer (1.5*2^23 magic add), 2^f on [-1/2, 1/2] by a degree-3 fit
// (max relative error 1.0e-4, below bf16's half-ulp 2e-3 that P is rounded to),
// 2^j by adding j to the exponent field.  x is clamped at -125 (2^-125 ~ 0).
// (a, b) <- (a, b) * s + t with one packed FFMA2 (sm_100a fma.rn.f32x2)
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

// packed pair version: same arithmetic in f32x2 instructions (half the issue slots)
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



// debug timeline: tl[(role * 64 + block) * 8 + event] for CTA 0, first 64 blocks.
// Compiled in only with -DORBIT2_ATTN_TIMELINE (scripts/attn_timeline.py builds
// that variant): the stamps cost the softmax warps registers.
#ifdef ORBIT2_ATTN_TIMELINE
#define TL_STAMP(role, blk, ev)                                                          \
  do {                                                                                   \
    if (tl != nullptr && blockIdx.x == 0 && (blk) < 64) tl[((role) * 64 + (blk)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define TL_STAMP(role, blk, ev) \
  do {                          \
  } while (0)
#endif

#ifndef ORBIT2_ATTN_LATEPV
#define ORBIT2_ATTN_LATEPV 1
#endif
#ifndef ORBIT2_ATTN_REGREALLOC
#define ORBIT2_ATTN_REGREALLOC 0   // measured slower (C2: 20.45 vs 20.08 ms)
#endif
// control warpgroup gives registers to the softmax warpgroups (no spills in the exp loop)
constexpr bool kRegRealloc = ORBIT2_ATTN_REGREALLOC != 0;
#ifndef ORBIT2_ATTN_KVST
#define ORBIT2_ATTN_KVST 2
#endif
#ifndef ORBIT2_ATTN_PINGPONG
#define ORBIT2_ATTN_PINGPONG 0   // measured slower (C2: 22.0 vs 19.5 ms): one warp per SM sub-partition reaches ~69% of the MUFU rate
#endif
// the two Q tiles' exponential phases alternate (named barriers 1 / 2): one
// tile's row max, waits and epilogue overlap the other tile's exponentials
constexpr bool kPingPong = ORBIT2_ATTN_PINGPONG != 0;
#ifndef ORBIT2_ATTN_SPLITROW
#define ORBIT2_ATTN_SPLITROW 0   // measured slower (C2: 19.5 vs 19.1 ms)
#endif
// two softmax warps per query row (64 keys each) at head dim 64: four softmax
// warps per SM sub-partition to hide the exponential loop's latencies
constexpr bool kSplitRow = ORBIT2_ATTN_SPLITROW != 0;
#ifndef ORBIT2_ATTN_SPLITP
#define ORBIT2_ATTN_SPLITP 0   // measured slower (C2: 21.6 vs 19.9 ms): the 128-arrival part barriers wait for the slowest warp
#endif
// P_j written and consumed by the PV MMA in two 64-key parts
constexpr bool kSplitP = ORBIT2_ATTN_SPLITP != 0;
#ifndef ORBIT2_ATTN_STAGED_EPI
#define ORBIT2_ATTN_STAGED_EPI 1
#endif
// wait for the previous PV (P columns free, O complete) after the row max, not before
constexpr bool kLatePvWait = ORBIT2_ATTN_LATEPV != 0;
// epilogue rows staged in smem and stored 4 rows per instruction
constexpr bool kStagedEpilogue = ORBIT2_ATTN_STAGED_EPI != 0;
#ifndef ORBIT2_ATTN_TAILSKIP
#define ORBIT2_ATTN_TAILSKIP 0   // measured slower at C2 (19.7 vs 18.6 ms) and equal at C3 (14.7 vs 14.4 ms)
#endif
// Partial last key block of a tile: 64-key halves with no valid key are neither
// exponentiated nor written to P, the PV MMA stops at the last written chunk and
// S = Q K^T uses N = 64 when at most 64 keys are valid (MUFU work and tensor work
// follow the tile's true length instead of the 128-key block).
constexpr bool kTailSkip = ORBIT2_ATTN_TAILSKIP != 0;
#ifndef ORBIT2_ATTN_DESYNC
#define ORBIT2_ATTN_DESYNC 0   // measured no gain (C2: 20.6-20.9 vs 20.5 ms with the same tail skip)
#endif
// At the start of each work item the second Q tile's softmax warp (same SM
// sub-partition as the first tile's) starts its exponentials only when the first
// tile's warp has done half (1) / all (2) of its first block's: the two warps'
// exponential phases then interleave with each other's row-max / wait phases
// instead of colliding on the MUFU (0 = both start together).
constexpr int kDesync = ORBIT2_ATTN_DESYNC;
#ifndef ORBIT2_ATTN_SPIN_CLK
#define ORBIT2_ATTN_SPIN_CLK 0
#endif

template <int DH, int NQ>
struct AttnCfg {
  static constexpr int AC = DH < 64 ? DH : 64;        // columns per swizzle atom
  static constexpr int RB = AC * 2;                   // bytes per atom row
  static constexpr int NA = DH / AC;                  // atoms per 128-row block
  static constexpr int ATOM = 128 * RB;               // bytes per atom
  static constexpr int TILE = 128 * DH * 2;           // bytes of a Q/K/V block
  static constexpr uint32_t SW = DH == 32 ? tc::SW_64B : tc::SW_128B;
  static constexpr int QBUF = DH == 128 ? 1 : 2;      // Q tiles of the next work item prefetched
  static constexpr int NPH = kSplitP ? 2 : 1;         // P / PV parts with their own barriers
  static constexpr int KST = DH == 128 ? 1 : ORBIT2_ATTN_KVST;   // K ring (consumed by S_{j+1}, early)
  static constexpr int VST = DH == 128 ? 1 : ORBIT2_ATTN_KVST;   // V ring (consumed by PV_j, late)
  static constexpr int P_BYTES = 128 * 128 * 2;
  // producer (+TMEM alloc), one MMA issuer per Q tile; padded to a whole warpgroup
  // when registers are reallocated (setmaxnreg acts per warpgroup)
  static constexpr int CTRL_WARPS = kRegRealloc ? 4 : 1 + NQ;
  static constexpr int SPW_ = kSplitRow && DH == 64 ? 2 : 1;  // softmax warps per query row (see P_TMEM)
  // P lives in TMEM (64 columns of bf16 pairs) and feeds the PV MMA as the A
  // operand when TMEM allows: no shared-memory traffic for P (the SS form
  // re-reads the 128 x 16 A tile from smem on every K step, which made the
  // kernel shared-memory-bandwidth bound).
  static constexpr bool P_TMEM = NQ * (128 + DH + 64) <= 512;
  static constexpr int TCOLS = 128 + DH + (P_TMEM ? 64 : 0);   // S | O | (P)
  static constexpr int SPW = (SPW_ > 1 && P_TMEM && NPH == 1 && !kPingPong) ? SPW_ : 1;
  static constexpr int KC = 128 / SPW;                // keys per softmax thread and block
  static constexpr int THREADS = 32 * CTRL_WARPS + 128 * NQ * SPW;   // + SPW softmax threads per query row
  // row-max (2 block parities) and row-sum exchange between the warps of a row
  static constexpr int XCH_BYTES = SPW > 1 ? NQ * (2 * 2 + 2) * 128 * 4 : 0;
  static constexpr int TMEM_COLS = NQ * TCOLS <= 256 ? 256 : 512;
  static constexpr int P_SMEM = P_TMEM ? 0 : P_BYTES;
  static constexpr int SMEM_BASE = QBUF * NQ * TILE + (KST + VST) * TILE + NQ * P_SMEM + 1024 + 512;
  // epilogue staging (32 rows x DH bf16 per softmax warp) when shared memory allows
  static constexpr int OST_ROW = DH * 2;               // staged O row (swizzled like the TMA store's box)
  static constexpr uint32_t OSW_MASK = DH == 32 ? 3u : 7u;   // SWIZZLE_64B / SWIZZLE_128B
  static constexpr bool STAGED = kStagedEpilogue && SMEM_BASE + 4 * NQ * 32 * OST_ROW + 256 <= 227 * 1024;
  static constexpr int OST_WARP = STAGED ? 32 * OST_ROW : 0;
  static constexpr int IRING = 4;                      // work-item descriptors published by the producer
  static constexpr int SMEM = SMEM_BASE + 4 * NQ * OST_WARP + XCH_BYTES + 256;
};

// Conditional rescale threshold (log2 units): the reference max of a row is
// only moved when the running max exceeds it by more than 8, so probabilities
// stay <= 2^8 (exact in bf16's exponent range, fp32 accumulation) and the
// O rescale in TMEM is rare.  Mathematically identical softmax (R18).
constexpr float kRescaleLog2 = 8.0f;
#ifndef ORBIT2_ATTN_POLY
#define ORBIT2_ATTN_POLY 2
#endif
// exponentials per 16 computed on the FMA pipe (ex2_poly) instead of the MUFU
constexpr int kPolyPer16 = ORBIT2_ATTN_POLY;

struct __align__(16) Item {
  int64_t base;     // first row of the tile's tokens in the packed workspace
  int n, q0, nq, nkb, h, pad_;
};

template <int NQ>
__device__ __forceinline__ Item item_info(const ChunkDev& ch, int heads, int id) {
  // 32-bit division (n_items < 2^31 is checked at launch): a 64-bit one is a
  // subroutine call whose ABI spills registers in every role's loop
  const int np = ch.core_pairs ? ch.nqc : ch.nqp;
  const int per_b = np * heads;                       // item = (pair fastest, head, sample)
  Item it;
  const int b = id / per_b;
  const int r = id - b * per_b;
  it.h = r / np;
  const int pr = r - it.h * np;
  DevTile t;
  int nq_max = NQ;
  if (ch.core_pairs) {                                // last block: query blocks holding core tokens
    const int e = ch.qpair_core[ch.qc0 + pr];
    t = ch.tiles[e >> 16];
    it.q0 = ((e & 0xFFFF) >> 1) * 128;
    nq_max = min(NQ, (e & 1) + 1);
  } else {
    const int g = ch.qp0 + pr;
    t = ch.tiles[ch.qpair_tile[g]];
    it.q0 = (g - t.qp_off) * 128 * NQ;
  }
  it.n = t.n_tokens;
  it.base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  it.nq = min(nq_max, (it.n - it.q0 + 127) / 128);
  it.nkb = (it.n + 127) / 128;
  return it;
}

// Item li of this CTA as published by the producer (whole warp; one release per warp).
__device__ __forceinline__ Item take_item(const Item* sItem, uint64_t* it_full, uint64_t* it_empty, uint32_t li,
                                          int ring) {
  const uint32_t is = li % ring;
  tc::mbar_wait(&it_full[is], (li / ring) & 1);
  const Item it = sItem[is];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) tc::mbar_arrive(&it_empty[is]);
  return it;
}

// Persistent: CTA c handles work items c, c + gridDim.x, ... where an item is
// (query-block pair of a tile, head, sample).  Every barrier phase is tracked
// with counters that run across items, so the producer prefetches the next
// item's Q / K / V and the tensor core starts its S_0 while the softmax warps
// finish the previous item.
template <int DH, int NQ>
__global__ void __launch_bounds__(AttnCfg<DH, NQ>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo,
                   __nv_bfloat16* __restrict__ out, ChunkDev ch, int D,
                   int heads, int n_items, long long* __restrict__ tl, float* __restrict__ lse,
                   int64_t ld_stat) {
  // tl: optional debug timeline (clock64 stamps of CTA 0), null in production
  using C = AttnCfg<DH, NQ>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the __shared__ array (keeps the shared address space: STS, not generic ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                               // [QBUF][NQ][TILE]
  uint8_t* sK = sQ + C::QBUF * NQ * C::TILE;        // [KST][TILE]
  uint8_t* sV = sK + C::KST * C::TILE;              // [VST][TILE]
  uint8_t* sP = sV + C::VST * C::TILE;              // [NQ][P_SMEM]
  uint8_t* sOst = sP + NQ * C::P_SMEM;              // [4 * NQ][OST_WARP]
  float* sXch = reinterpret_cast<float*>(sOst + 4 * NQ * C::OST_WARP);   // [XCH_BYTES / 4]
  Item* sItem = reinterpret_cast<Item*>(reinterpret_cast<uint8_t*>(sXch) + C::XCH_BYTES);   // [IRING]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sItem + C::IRING);
  uint64_t* q_full = bar;                           // [QBUF]
  uint64_t* q_empty = q_full + C::QBUF;             // [QBUF]
  uint64_t* k_full = q_empty + C::QBUF;             // [KST]
  uint64_t* k_empty = k_full + C::KST;              // [KST]
  uint64_t* v_full = k_empty + C::KST;              // [VST]
  uint64_t* v_empty = v_full + C::VST;              // [VST]
  uint64_t* s_full = v_empty + C::VST;              // [NQ]  S in TMEM
  uint64_t* s_free = s_full + NQ;                   // [NQ]  softmax holds S in registers
  uint64_t* p_full = s_free + NQ;                   // [NQ][NPH]  part h of P written (+ O rescaled)
  uint64_t* p_free = p_full + NQ * C::NPH;          // [NQ][NPH]  part h of PV done (P part free)
  uint64_t* o_free = p_free + NQ * C::NPH;          // [NQ]  epilogue has read O
  uint64_t* it_full = o_free + NQ;                 // [IRING]  item descriptor published
  uint64_t* it_empty = it_full + C::IRING;          // [IRING]  read by every consumer warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(it_empty + C::IRING);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm);
    for (int s = 0; s < C::QBUF; ++s) {
      tc::mbar_init(&q_full[s], 1);
      tc::mbar_init(&q_empty[s], NQ);   // one arrival per MMA-issuer warp
    }
    for (int s = 0; s < C::KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], NQ);
    }
    for (int s = 0; s < C::VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], NQ);
    }
    for (int s = 0; s < NQ; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&s_free[s], 128 * C::SPW);
      for (int h = 0; h < C::NPH; ++h) {
        tc::mbar_init(&p_full[s * C::NPH + h], 128 * C::SPW);
        tc::mbar_init(&p_free[s * C::NPH + h], 1);
      }
      tc::mbar_init(&o_free[s], 128 * C::SPW);
    }
    for (int s = 0; s < C::IRING; ++s) {
      tc::mbar_init(&it_full[s], 1);
      tc::mbar_init(&it_empty[s], NQ + 4 * NQ * C::SPW);   // MMA-issuer warps + softmax warps
    }
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    __syncwarp();
    tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (kRegRealloc) {
    if (warp < C::CTRL_WARPS) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t li = 0, gk = 0, gv = 0;
      for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const Item it = item_info<NQ>(ch, heads, id);
        {   // publish the item to the other roles (they never touch the tile tables)
          const uint32_t is = li % C::IRING;
          tc::mbar_wait(&it_empty[is], ((li / C::IRING) & 1) ^ 1);
          sItem[is] = it;
          tc::mbar_arrive(&it_full[is]);
        }
        const int32_t y0 = (int32_t)it.base;
        const uint32_t qb = li % C::QBUF;
        tc::mbar_wait(&q_empty[qb], ((li / C::QBUF) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&q_full[qb], it.nq * C::TILE);
        for (int qt = 0; qt < it.nq; ++qt)
          for (int a = 0; a < C::NA; ++a)
            tc::tma_load_2d(&tm, sQ + (qb * NQ + qt) * C::TILE + a * C::ATOM, &q_full[qb], it.h * DH + a * C::AC,
                            y0 + it.q0 + qt * 128);
        auto load_k = [&](int j) {
          const uint32_t st = gk % C::KST;
          tc::mbar_wait(&k_empty[st], ((gk / C::KST) & 1) ^ 1);
          TL_STAMP(4, gk, 0);
          tc::mbar_arrive_expect_tx(&k_full[st], C::TILE);
          for (int a = 0; a < C::NA; ++a)
            tc::tma_load_2d(&tm, sK + st * C::TILE + a * C::ATOM, &k_full[st], D + it.h * DH + a * C::AC,
                            y0 + j * 128);
          ++gk;
        };
        auto load_v = [&](int j) {
          const uint32_t st = gv % C::VST;
          tc::mbar_wait(&v_empty[st], ((gv / C::VST) & 1) ^ 1);
          TL_STAMP(4, gv, 1);
          tc::mbar_arrive_expect_tx(&v_full[st], C::TILE);
          for (int a = 0; a < C::NA; ++a)
            tc::tma_load_2d(&tm, sV + st * C::TILE + a * C::ATOM, &v_full[st], 2 * D + it.h * DH + a * C::AC,
                            y0 + j * 128);
          ++gv;
        };
        // issue order = consumption order: K_0, then per j: K_{j+1}, V_j
        load_k(0);
        for (int j = 0; j < it.nkb; ++j) {
          if (j + 1 < it.nkb) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp <= NQ) {
    {   // whole warp runs the loop (uniform descriptors); one elected lane issues
      // ---------------- MMA issuers: warp 1 -> Q tile 0, warp 2 -> Q tile 1 ----------------
      // Each Q tile has its own issuing thread so the two softmax warpgroups
      // are not forced into lockstep (their exp phases then alternate on the
      // MUFU instead of colliding).  Shared Q/K/V slots are released by one
      // arrival per issuer; an issuer whose tile is idle for a work item still
      // walks the ring phases (wait full, arrive empty) to stay aligned.
      const int qt = warp - 1;
      constexpr uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t id_s64 = tc::idesc_bf16(128, 64, 0, 0);  // short last key block
      constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);    // P K-major, V MN-major
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const uint32_t p_addr = tc::smem_u32(sP);
      uint32_t li = 0, gk = 0, gv = 0, ns = 0, np = 0, ni = 0;
      for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const Item it = take_item(sItem, it_full, it_empty, li, C::IRING);
        const bool active = qt < it.nq;
        const uint32_t qb = li % C::QBUF;
        tc::mbar_wait(&q_full[qb], (li / C::QBUF) & 1);
        int js = 0;                       // key block of the next S
        auto issue_s = [&](bool last) {   // S = Q K_j^T for this Q tile
          const uint32_t st = gk % C::KST;
          const bool n64 = kTailSkip && it.n - js * 128 <= 64;   // at most 64 valid keys: N = 64
          ++js;
          tc::mbar_wait(&k_full[st], (gk / C::KST) & 1);
          if (lane == 0) TL_STAMP(2 + qt, ns, 0);
          if (active) {
            if (ns >= 1) tc::mbar_wait(&s_free[qt], (ns - 1) & 1);
            if (lane == 0) TL_STAMP(2 + qt, ns, 1);
            tc::tc_fence_after();
            if (tc::elect_one()) {
              // descriptors built once; k-steps advance the start-address field (addr >> 4)
              const uint64_t qd0 = tc::sdesc(q_addr + (qb * NQ + qt) * C::TILE, 16, 8 * C::RB, C::SW);
              const uint64_t kd0 = tc::sdesc(k_addr + st * C::TILE, 16, 8 * C::RB, C::SW);
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk) {
                const uint32_t adv = (uint32_t)(((kk * 16) / C::AC) * C::ATOM + ((kk * 16) % C::AC) * 2) >> 4;
                tc::mma_bf16_ss(tmem + qt * C::TCOLS, qd0 + adv, kd0 + adv, n64 ? id_s64 : id_s, kk > 0);
              }
              tc::mma_commit(&s_full[qt]);
              tc::mma_commit(&k_empty[st]);
              if (last) tc::mma_commit(&q_empty[qb]);   // Q buffer free once the item's S MMAs finish
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
          if (j + 1 < it.nkb) issue_s(j + 2 == it.nkb);   // S_{j+1} overlaps softmax of block j
          const uint32_t st = gv % C::VST;
          tc::mbar_wait(&v_full[st], (gv / C::VST) & 1);
          if (lane == 0) TL_STAMP(2 + qt, np, 2);
          if (active) {
            if (j == 0 && ni >= 1) tc::mbar_wait(&o_free[qt], (ni - 1) & 1);
            // PV in NPH parts, each released by its own p_full / p_free pair: the
            // softmax warps may write part h of P_{j+1} as soon as part h of PV_j
            // has consumed P_j (no wait for the whole PV on their critical path).
            const uint32_t ptm = tmem + qt * C::TCOLS + 128 + DH;   // P columns (P_TMEM)
            const uint64_t pd0 = tc::sdesc(p_addr + qt * C::P_SMEM, 16, 1024, tc::SW_128B);
            const uint64_t vd0 = tc::sdesc(v_addr + st * C::TILE, C::ATOM, 8 * C::RB, C::SW);
#pragma unroll
            for (int h = 0; h < C::NPH; ++h) {
              tc::mbar_wait(&p_full[qt * C::NPH + h], np & 1);
              if (lane == 0 && h == 0) TL_STAMP(2 + qt, np, 3);
              tc::tc_fence_after();
              if (tc::elect_one()) {
                // K steps holding keys the softmax wrote (64-key halves; kTailSkip)
                const int kv = it.n - j * 128;
                const int kk_end = kTailSkip && kv <= 64 ? 4 : 8;
#pragma unroll
                for (int kk = h * (8 / C::NPH); kk < (h + 1) * (8 / C::NPH); ++kk) {   // K = 16 keys per MMA
                  if (kk >= kk_end) break;
                  const uint32_t padv = (uint32_t)((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                  const uint32_t vadv = (uint32_t)(kk * 16 * C::RB) >> 4;
                  const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
                  if (C::P_TMEM)
                    tc::mma_bf16_ts(tmem + qt * C::TCOLS + 128, ptm + kk * 8, vd0 + vadv, id_o, acc);
                  else
                    tc::mma_bf16_ss(tmem + qt * C::TCOLS + 128, pd0 + padv, vd0 + vadv, id_o, acc);
                }
                tc::mma_commit(&p_free[qt * C::NPH + h]);
                if (h == C::NPH - 1) {
                  tc::mma_commit(&v_empty[st]);
                  if (lane == 0) TL_STAMP(2 + qt, np, 4);
                }
              }
              __syncwarp();
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
    }
  } else if (warp < C::CTRL_WARPS) {
    // spare warp of the control warpgroup (register reallocation): idle
  } else {
    // ---------------- softmax / correction / epilogue ----------------
    // Thread = query row i of Q tile qt (TMEM lane i: warp w reads lane quarter
    // w % 4; any 4 consecutive warps cover the quarters).  Both tiles' softmax
    // warps run concurrently (two warps per SM sub-partition feed the MUFU).
    constexpr int SPW = C::SPW, KC = C::KC;
    const int sidx = warp - C::CTRL_WARPS;
    const int qt = sidx / (4 * SPW);
    const int hh = (sidx / 4) % SPW;               // which KC keys of the block this warp owns
    const int q = warp & 3;
    const int i = q * 32 + lane;                   // query row within the Q tile
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + qt * C::TCOLS;
    const uint32_t s_addr = lane_base + hh * KC;
    const uint32_t o_addr = lane_base + 128;
    const uint32_t p_tm = lane_base + 128 + DH + hh * (KC / 2);
    constexpr int OC = DH / SPW;                   // O columns this warp rescales / stores
    const uint32_t tile_bar = 1 + qt;              // both halves of a tile's rows (SPW > 1)
    const uint32_t pair_bar = 3 + qt * 4 + q;      // the SPW warps of one 32-row slice
    const float sl = 1.4426950408889634f * rsqrtf((float)DH);   // log2(e)/sqrt(d)
    uint32_t cs = 0;                               // blocks processed by this Q tile (all items)
    uint32_t ni_sm = 0;                            // items processed (debug timeline only)
    // ping-pong turns: barrier 1 + t = "tile t may exponentiate"; 256 = both tiles' warps
    auto pp_sync = [](int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); };
    auto pp_arrive = [](int id) { asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory"); };
    if (kPingPong && qt == 1) pp_arrive(1);        // tile 0 goes first
    uint32_t li = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
      if (q == 0 && lane == 0) TL_STAMP(5 + qt, ni_sm, 6);
      const Item it = take_item(sItem, it_full, it_empty, li, C::IRING);
      if (q == 0 && lane == 0) TL_STAMP(5 + qt, ni_sm, 7);
      if (qt >= it.nq) {
        if constexpr (kPingPong) {   // keep the turn-taking aligned with the active tile
          for (int j = 0; j < it.nkb; ++j) {
            pp_sync(1 + qt);
            pp_arrive(1 + (qt ^ 1));
          }
        }
        continue;
      }
      float m_ref = -INFINITY, l_run = 0.f;
      const bool tlr = q == 0 && lane == 0 && hh == 0;
      // Only rows inside the tile take part in the (warp-uniform) range votes, so
      // results do not depend on packing, chunking or the rank assignment.
      const bool row_valid = it.q0 + qt * 128 + i < it.n;
      for (int j = 0; j < it.nkb; ++j, ++cs) {
        if (tlr) TL_STAMP(qt, cs, 0);
        tc::mbar_wait(&s_full[qt], cs & 1);
        if (tlr) TL_STAMP(qt, cs, 1);
        tc::tc_fence_after();
        float sv[KC];
        {
          uint32_t* r = reinterpret_cast<uint32_t*>(sv);
#pragma unroll
          for (int c0 = 0; c0 < KC; c0 += 32)
            tc::tmem_ld32(s_addr + c0, *reinterpret_cast<uint32_t(*)[32]>(r + c0));
          tc::tmem_ld_wait();
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&s_free[qt]);               // TMEM S columns may take the next S
        if (tlr) TL_STAMP(qt, cs, 2);
        const int kvalid = it.n - j * 128 - hh * KC;
        if (kvalid < KC) {
#pragma unroll
          for (int c = 0; c < KC; ++c)
            if (c >= kvalid) sv[c] = -INFINITY;
        }
        auto row_max = [&]() {
          float m0 = sv[0], m1 = sv[1], m2 = sv[2], m3 = sv[3];
#pragma unroll
          for (int c = 4; c < KC; c += 4) {
            m0 = fmaxf(m0, sv[c]); m1 = fmaxf(m1, sv[c + 1]);
            m2 = fmaxf(m2, sv[c + 2]); m3 = fmaxf(m3, sv[c + 3]);
          }
          float m = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
          if constexpr (SPW > 1) {   // the other warp of the row: exchange through smem
            float* xm = sXch + (qt * 2 + (cs & 1)) * 2 * 128;
            xm[hh * 128 + i] = m;
            asm volatile("bar.sync %0, %1;" ::"r"(tile_bar), "r"(128 * SPW) : "memory");
            m = fmaxf(m, xm[(hh ^ 1) * 128 + i]);
          }
          return m * sl;
        };
        // O rescale by 2^(m_ref - m_new) (tcgen05.ld/st are warp-collective: callers
        // take the decision warp-uniformly); needs the previous PV complete.
        auto rescale = [&](float m_new) {
          const float alpha = ex2(m_ref - m_new);
          l_run *= alpha;
#pragma unroll
          for (int c0 = hh * OC; c0 < (hh + 1) * OC; c0 += 16) {
            uint32_t r[16];
            tc::tmem_ld16(o_addr + c0, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tc::tmem_st16(o_addr + c0, r);
          }
          m_ref = m_new;
        };
        // Part h of PV_{j-1} done: P columns of part h free (all parts: O complete).
        uint32_t pv_done = cs == 0 ? (1u << C::NPH) - 1 : 0u;
        auto wait_pv = [&](int h) {
          if (!(pv_done >> h & 1u)) {
            tc::mbar_wait(&p_free[qt * C::NPH + h], (cs - 1) & 1);
            tc::tc_fence_after();
            pv_done |= 1u << h;
            if (tlr && h == 0) TL_STAMP(qt, cs, 4);
          }
        };
        if (!kLatePvWait)
          for (int h = 0; h < C::NPH; ++h) wait_pv(h);
        // Conditional rescale (R18): the reference max moves only when the block max
        // exceeds it by more than kRescaleLog2 (p <= 2^8, the O rescale is rare).
        {
          const float m_blk = row_max();
          if (j == 0)
            m_ref = m_blk;
          else if (__any_sync(0xffffffffu, row_valid && m_blk > m_ref + kRescaleLog2)) {
            for (int h = 0; h < C::NPH; ++h) wait_pv(h);
            rescale(fmaxf(m_blk, m_ref));
          }
        }
        if (tlr) TL_STAMP(qt, cs, 3);
        // p = 2^(s * log2(e)/sqrt(d) - m_ref) -> bf16 P (TMEM: A operand of the PV MMA;
        // smem when TMEM is short), part by part, with fp32 row sums
        constexpr int KP = KC / C::NPH;                // keys per part
        float rs0 = 0.f, rs1 = 0.f;
        if constexpr (kPingPong) pp_sync(1 + qt);   // this tile's turn on the MUFU
        // first block of an item with both Q tiles active: offset the two tiles'
        // exponential phases (named barrier of this sub-partition's two warps)
        const bool desync = kDesync > 0 && SPW == 1 && !kPingPong && j == 0 && it.nq == NQ && NQ == 2;
        const uint32_t dbar = 11 + q;
        if (desync && qt == 1) asm volatile("bar.sync %0, 64;" ::"r"(dbar) : "memory");
        if (ORBIT2_ATTN_SPIN_CLK > 0 && j == 0 && qt == 1 && it.nq == NQ) {
          // stagger the second Q tile's first exponential phase by a fixed delay
          const long long t0 = clock64();
          while (clock64() - t0 < (long long)ORBIT2_ATTN_SPIN_CLK) {
          }
        }
        const int kv_blk = it.n - j * 128;         // valid keys of this block (SPW == 1)
        const int c_arr = (kDesync == 1 ? KC / 2 : KC) - 64;   // half after which tile 0 releases tile 1
#pragma unroll
        for (int h = 0; h < C::NPH; ++h) {
          wait_pv(h);
          if constexpr (C::P_TMEM) {
#pragma unroll
            for (int c0 = h * KP; c0 < (h + 1) * KP; c0 += 64) {
              if (kTailSkip && SPW == 1 && c0 >= kv_blk) break;   // half past the tile end
              uint32_t pk[32];
              // ORBIT2_ATTN_RS_SPLIT independent packed partial sums: the row sum is not one
              // 32-long chain of dependent adds behind the exponentials
              float2 rs[ORBIT2_ATTN_RS_SPLIT];
#pragma unroll
              for (int u = 0; u < ORBIT2_ATTN_RS_SPLIT; ++u) rs[u] = make_float2(0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 64; e += 2) {
                float x0 = sv[c0 + e], x1 = sv[c0 + e + 1];
                ffma2(x0, x1, sl, -m_ref);                 // FFMA2: both (s*c - m) in one instruction
                float2 pr;
                if ((e & 15) < kPolyPer16) pr = ex2_poly2(x0, x1);
                else pr = make_float2(ex2(x0), ex2(x1));
                rs[(e / 2) % ORBIT2_ATTN_RS_SPLIT] = tc::add2(rs[(e / 2) % ORBIT2_ATTN_RS_SPLIT], pr);
                pk[e / 2] = tc::pack_bf16(pr.x, pr.y);     // column = keys (2c, 2c+1), lower key in low half
              }
#pragma unroll
              for (int u = 1; u < ORBIT2_ATTN_RS_SPLIT; ++u) rs[0] = tc::add2(rs[0], rs[u]);
              rs0 += rs[0].x;
              rs1 += rs[0].y;
              tc::tmem_st32(p_tm + c0 / 2, pk);
              if (desync && qt == 0 && c0 == c_arr) asm volatile("bar.arrive %0, 64;" ::"r"(dbar) : "memory");
            }
            if (desync && qt == 0 && kTailSkip && kv_blk <= c_arr)   // loop left before c_arr: still release
              asm volatile("bar.arrive %0, 64;" ::"r"(dbar) : "memory");
            tc::tmem_st_wait();
          } else {   // P to smem (SW128 K-major, 64-key atoms of 16 KB)
            uint8_t* prow = sP + qt * C::P_SMEM + i * 128;
            const int sw = i & 7;
#pragma unroll
            for (int c0 = h * KP; c0 < (h + 1) * KP; c0 += 16) {
              uint32_t pk[8];
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                float x0 = sv[c0 + e], x1 = sv[c0 + e + 1];
                ffma2(x0, x1, sl, -m_ref);
                const float p0 = ex2(x0), p1 = ex2(x1);
                rs0 += p0;
                rs1 += p1;
                pk[e / 2] = tc::pack_bf16(p0, p1);
              }
              uint8_t* atom = prow + (c0 >> 6) * 16384;
              const int cb = (c0 & 63) >> 3;
              *reinterpret_cast<uint4*>(atom + ((cb ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              *reinterpret_cast<uint4*>(atom + (((cb + 1) ^ sw) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
            tc::fence_proxy_async_smem();
          }
          tc::tc_fence_before();
          tc::mbar_arrive(&p_full[qt * C::NPH + h]);
        }
        if constexpr (kPingPong) pp_arrive(1 + (qt ^ 1));   // the other tile's turn
        l_run += rs0 + rs1;
        if (tlr) TL_STAMP(qt, cs, 5);
      }
      // epilogue: O / l
      if (tlr) TL_STAMP(5 + qt, ni_sm, 0);
      for (int h = 0; h < C::NPH; ++h) tc::mbar_wait(&p_free[qt * C::NPH + h], (cs - 1) & 1);
      tc::tc_fence_after();
      if (tlr) TL_STAMP(5 + qt, ni_sm, 1);
      if constexpr (SPW > 1) {   // row sum over both warps of the row
        float* xl = sXch + NQ * 2 * 2 * 128 + qt * 2 * 128;
        xl[hh * 128 + i] = l_run;
        asm volatile("bar.sync %0, %1;" ::"r"(tile_bar), "r"(128 * SPW) : "memory");
        l_run += xl[(hh ^ 1) * 128 + i];
      }
      const float inv = 1.f / l_run;
      if (lse != nullptr && hh == 0) {   // training: per-row log-sum-exp (log2 units) for the backward
        const int qr = it.q0 + qt * 128 + i;
        if (qr < it.n) lse[(int64_t)it.h * ld_stat + it.base + qr] = m_ref + log2f(l_run);
      }
      if constexpr (C::STAGED) {
        // O / l -> bf16, staged in this warp's 32-row slice in the TMA store's
        // swizzled layout (16-B chunk c of row r at chunk c ^ (r & mask):
        // conflict-free), then one TMA tensor store of the 32 x DH box issued by
        // one lane.  A warp whose rows run past the tile end (the partial last
        // query block) stores its valid rows directly instead.
        uint8_t* sw = sOst + (qt * 4 + q) * C::OST_WARP;   // the 32-row slice of this warp (pair)
        auto swz = [](uint32_t off) { return off ^ (((off >> 7) & C::OSW_MASK) << 4); };
        const bool st_lane = lane == 0 && hh == 0;     // issues the slice's TMA store
        if (st_lane) tc::bulk_wait_read<0>();          // the previous item's store has read the slice
        if constexpr (SPW > 1) asm volatile("bar.sync %0, %1;" ::"r"(pair_bar), "r"(32 * SPW) : "memory");
        else __syncwarp();
#pragma unroll
        for (int c0 = hh * OC; c0 < (hh + 1) * OC; c0 += 32) {   // 32 columns per TMEM load
          uint32_t r[32];
          tc::tmem_ld32(o_addr + c0, r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(sw + swz(lane * C::OST_ROW + (c0 + 8 * u) * 2)) =
                make_uint4(tc::pack_bf16(__uint_as_float(r[8 * u]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                           tc::pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                           tc::pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                           tc::pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
        }
        if (tlr) TL_STAMP(5 + qt, ni_sm, 2);
        tc::tc_fence_before();
        tc::mbar_arrive(&o_free[qt]);                  // O read: the next item's PV may accumulate
        if (tlr) TL_STAMP(5 + qt, ni_sm, 4);
        const int row0 = it.q0 + qt * 128 + q * 32;    // first query row of this warp
        if (row0 + 32 <= it.n) {
          tc::fence_proxy_async_smem();
          if constexpr (SPW > 1) asm volatile("bar.sync %0, %1;" ::"r"(pair_bar), "r"(32 * SPW) : "memory");
          else __syncwarp();
          if (tlr) TL_STAMP(5 + qt, ni_sm, 5);
          if (st_lane) {
            tc::tma_store_2d(&tmo, sw, it.h * DH, (int32_t)(it.base + row0));
            tc::bulk_commit();
          }
        } else {
          __syncwarp();
          if (row0 + lane < it.n) {
#pragma unroll
            for (int c = hh * OC / 8; c < (hh + 1) * OC / 8; ++c)
              *reinterpret_cast<uint4*>(out + (it.base + row0 + lane) * (int64_t)D + it.h * DH + c * 8) =
                  *reinterpret_cast<const uint4*>(sw + swz(lane * C::OST_ROW + c * 16));
          }
        }
        if (tlr) TL_STAMP(5 + qt, ni_sm, 3);
        ++ni_sm;
        continue;
      }
      const int qrow = it.q0 + qt * 128 + i;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(o_addr + c0, r);
        tc::tmem_ld_wait();
        if (qrow < it.n) {
          uint4* dst = reinterpret_cast<uint4*>(out + (it.base + qrow) * (int64_t)D + it.h * DH + c0);
#pragma unroll
          for (int u = 0; u < 2; ++u)
            dst[u] = make_uint4(tc::pack_bf16(__uint_as_float(r[8 * u]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                                tc::pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                                tc::pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                                tc::pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&o_free[qt]);
    }
  }
  if (C::STAGED && warp >= C::CTRL_WARPS && lane == 0) tc::bulk_wait_all();   // epilogue stores done with smem
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int DH>
bool launch_dh(const void* qkv, int64_t rows, void* out, const ChunkDev& ch, int B, int D, int heads,
               cudaStream_t st, float* lse, int64_t ld_stat) {
  constexpr int NQ = 2;
  using C = AttnCfg<DH, NQ>;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, rows, 3LL * D, 3LL * D, 128, C::AC,
                      DH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  CUtensorMap tmo;   // attention output [rows][D], box 32 rows x DH columns (epilogue stores)
  if (C::STAGED && !make_tmap_bf16(&tmo, out, rows, D, D, 32, DH,
                                   DH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(attn_tc_kernel<DH, NQ>), C::SMEM, &attr_done)) return false;
  const int sms = num_sms();
  const int64_t n_items = (int64_t)(ch.core_pairs ? ch.nqc : ch.nqp) * heads * B;
  if (n_items == 0) return true;
  if (n_items >= (int64_t)INT32_MAX) return false;
  const unsigned grid = (unsigned)std::min<int64_t>(n_items, sms);   // persistent: one CTA per SM
  attn_tc_kernel<DH, NQ><<<grid, C::THREADS, C::SMEM, st>>>(tm, tmo, reinterpret_cast<__nv_bfloat16*>(out), ch, D,
                                                             heads, (int)n_items, g_attn_timeline, lse, ld_stat);
  return true;
}

}  // namespace

bool launch_attention_tc(const void* qkv_bf16, int64_t qkv_rows, void* out_bf16, const ChunkDev& ch, int B, int D,
                         int heads, int d, cudaStream_t st, float* lse, int64_t ld_stat) {
  if (d == 32) return launch_dh<32>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st, lse, ld_stat);
  if (d == 64) {
    // Short tiles (mean under 768 tokens, e.g. C3's 312-432): three Q tiles on 64-key
    // blocks (attn3_tc.cu; less padding of the last key block, three softmax warps per
    // sub-partition): measured 12.4 vs 14.8 ms at C3.  Long tiles (C2 / C4 / C5):
    // this kernel (19.0 vs 19.3-19.7 ms at C2).  ORBIT2_ATTN=2 / 3 forces one.
    const char* e = std::getenv("ORBIT2_ATTN");
    const int64_t mean_n = ch.tc > 0 ? ch.chunk_tokens / ch.tc : 0;
    // (training forward, lse != null: this kernel, which also writes the row log-sum-exp)
    const bool use3 = lse == nullptr && (e && e[0] == '3' ? true : (e && e[0] == '2' ? false : mean_n < 768));
    if (use3) return launch_attention3_tc(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st);
    return launch_dh<64>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st, lse, ld_stat);
  }
  if (d == 128) return launch_dh<128>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st, lse, ld_stat);
  return false;
}

}  // namespace orbit2
