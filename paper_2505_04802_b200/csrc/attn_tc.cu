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
//   warp 1 lane 0 : tcgen05.mma issuer, per Q tile t:
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

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DH, int NQ>
struct AttnCfg {
  static constexpr int AC = DH < 64 ? DH : 64;        // columns per swizzle atom
  static constexpr int RB = AC * 2;                   // bytes per atom row
  static constexpr int NA = DH / AC;                  // atoms per 128-row block
  static constexpr int ATOM = 128 * RB;               // bytes per atom
  static constexpr int TILE = 128 * DH * 2;           // bytes of a Q/K/V block
  static constexpr uint32_t SW = DH == 32 ? tc::SW_64B : tc::SW_128B;
  static constexpr int QBUF = DH == 128 ? 1 : 2;      // Q tiles of the next work item prefetched
  static constexpr int PBUF = 1;                      // P buffers per Q tile (2 deadlocked with QBUF=1; no gain seen)
  static constexpr int KST = DH == 128 ? 1 : 2;       // K ring (consumed by S_{j+1}, early)
  static constexpr int VST = DH == 128 ? 1 : 2;       // V ring (consumed by PV_j, late)
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int THREADS = 128 + 128 * NQ;
  static constexpr int TCOLS = 128 + DH;              // TMEM columns per Q tile: S | O
  static constexpr int TMEM_COLS = NQ * TCOLS <= 256 ? 256 : 512;
  static constexpr int SMEM = QBUF * NQ * TILE + (KST + VST) * TILE + NQ * PBUF * P_BYTES + 1024 + 512;
};

// Conditional rescale threshold (log2 units): the reference max of a row is
// only moved when the running max exceeds it by more than 8, so probabilities
// stay <= 2^8 (exact in bf16's exponent range, fp32 accumulation) and the
// O rescale in TMEM is rare.  Mathematically identical softmax (R18).
constexpr float kRescaleLog2 = 8.0f;

struct Item {
  int64_t base;     // first row of the tile's tokens in the packed workspace
  int n, q0, nq, nkb, h;
};

template <int NQ>
__device__ __forceinline__ Item item_info(const ChunkDev& ch, int heads, int64_t id) {
  const int64_t per_b = (int64_t)ch.nqp * heads;      // item = (pair fastest, head, sample)
  Item it;
  const int b = (int)(id / per_b);
  const int64_t r = id - (int64_t)b * per_b;
  it.h = (int)(r / ch.nqp);
  const int g = ch.qp0 + (int)(r - (int64_t)it.h * ch.nqp);
  const DevTile t = ch.tiles[ch.qpair_tile[g]];
  it.n = t.n_tokens;
  it.base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  it.q0 = (g - t.qp_off) * 128 * NQ;
  it.nq = min(NQ, (it.n - it.q0 + 127) / 128);
  it.nkb = (it.n + 127) / 128;
  return it;
}

// Persistent: CTA c handles work items c, c + gridDim.x, ... where an item is
// (query-block pair of a tile, head, sample).  Every barrier phase is tracked
// with counters that run across items, so the producer prefetches the next
// item's Q / K / V and the tensor core starts its S_0 while the softmax warps
// finish the previous item.
template <int DH, int NQ>
__global__ void __launch_bounds__(AttnCfg<DH, NQ>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out, ChunkDev ch, int D,
                   int heads, int64_t n_items) {
  using C = AttnCfg<DH, NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                               // [QBUF][NQ][TILE]
  uint8_t* sK = sQ + C::QBUF * NQ * C::TILE;        // [KST][TILE]
  uint8_t* sV = sK + C::KST * C::TILE;              // [VST][TILE]
  uint8_t* sP = sV + C::VST * C::TILE;              // [NQ][PBUF][P_BYTES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + NQ * C::PBUF * C::P_BYTES);
  uint64_t* q_full = bar;                           // [QBUF]
  uint64_t* q_empty = q_full + C::QBUF;             // [QBUF]
  uint64_t* k_full = q_empty + C::QBUF;             // [KST]
  uint64_t* k_empty = k_full + C::KST;              // [KST]
  uint64_t* v_full = k_empty + C::KST;              // [VST]
  uint64_t* v_empty = v_full + C::VST;              // [VST]
  uint64_t* s_full = v_empty + C::VST;              // [NQ]  S in TMEM
  uint64_t* s_free = s_full + NQ;                   // [NQ]  softmax holds S in registers
  uint64_t* p_full = s_free + NQ;                   // [NQ]  P in smem (+ O rescaled)
  uint64_t* p_free = p_full + NQ;                   // [NQ][PBUF]  PV done (P buffer free, O updated)
  uint64_t* o_free = p_free + NQ * C::PBUF;         // [NQ]  epilogue has read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + NQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm);
    for (int s = 0; s < C::QBUF; ++s) {
      tc::mbar_init(&q_full[s], 1);
      tc::mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < C::KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < NQ; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&s_free[s], 128);
      tc::mbar_init(&p_full[s], 128);
      for (int u = 0; u < C::PBUF; ++u) tc::mbar_init(&p_free[s * C::PBUF + u], 1);
      tc::mbar_init(&o_free[s], 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t li = 0, gk = 0, gv = 0;
      for (int64_t id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const Item it = item_info<NQ>(ch, heads, id);
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
          tc::mbar_arrive_expect_tx(&k_full[st], C::TILE);
          for (int a = 0; a < C::NA; ++a)
            tc::tma_load_2d(&tm, sK + st * C::TILE + a * C::ATOM, &k_full[st], D + it.h * DH + a * C::AC,
                            y0 + j * 128);
          ++gk;
        };
        auto load_v = [&](int j) {
          const uint32_t st = gv % C::VST;
          tc::mbar_wait(&v_empty[st], ((gv / C::VST) & 1) ^ 1);
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
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);    // P K-major, V MN-major
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const uint32_t p_addr = tc::smem_u32(sP);
      uint32_t li = 0, gk = 0, gv = 0;
      uint32_t ns[NQ], np[NQ], ni[NQ];   // per Q tile: S issued, PV issued, items finished
#pragma unroll
      for (int qt = 0; qt < NQ; ++qt) ns[qt] = np[qt] = ni[qt] = 0;
      for (int64_t id = blockIdx.x; id < n_items; id += gridDim.x, ++li) {
        const Item it = item_info<NQ>(ch, heads, id);
        const uint32_t qb = li % C::QBUF;
        tc::mbar_wait(&q_full[qb], (li / C::QBUF) & 1);
        auto issue_s_all = [&](bool last) {   // S = Q K_j^T for every active Q tile
          const uint32_t st = gk % C::KST;
          tc::mbar_wait(&k_full[st], (gk / C::KST) & 1);
          for (int qt = 0; qt < it.nq; ++qt) {
            if (ns[qt] >= 1) tc::mbar_wait(&s_free[qt], (ns[qt] - 1) & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const int a = (kk * 16) / C::AC, off = ((kk * 16) % C::AC) * 2;
              const uint64_t qd =
                  tc::sdesc(q_addr + (qb * NQ + qt) * C::TILE + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
              const uint64_t kd = tc::sdesc(k_addr + st * C::TILE + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
              tc::mma_bf16_ss(tmem + qt * C::TCOLS, qd, kd, id_s, kk > 0);
            }
            tc::mma_commit(&s_full[qt]);
            ++ns[qt];
          }
          tc::mma_commit(&k_empty[st]);
          if (last) tc::mma_commit(&q_empty[qb]);   // Q buffer free once the item's S MMAs finish
          ++gk;
        };
        issue_s_all(it.nkb == 1);
        for (int j = 0; j < it.nkb; ++j) {
          if (j + 1 < it.nkb) issue_s_all(j + 2 == it.nkb);   // S_{j+1} overlaps softmax of block j
          const uint32_t st = gv % C::VST;
          tc::mbar_wait(&v_full[st], (gv / C::VST) & 1);
          for (int qt = 0; qt < it.nq; ++qt) {
            if (j == 0 && ni[qt] >= 1) tc::mbar_wait(&o_free[qt], (ni[qt] - 1) & 1);
            tc::mbar_wait(&p_full[qt], np[qt] & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {   // 128 keys, K = 16 per MMA
              const uint64_t pd = tc::sdesc(p_addr + (qt * C::PBUF + np[qt] % C::PBUF) * C::P_BYTES +
                                                (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
              const uint64_t vd = tc::sdesc(v_addr + st * C::TILE + kk * 16 * C::RB, C::ATOM, 8 * C::RB, C::SW);
              tc::mma_bf16_ss(tmem + qt * C::TCOLS + 128, pd, vd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
            }
            tc::mma_commit(&p_free[qt * C::PBUF + np[qt] % C::PBUF]);
            ++np[qt];
          }
          tc::mma_commit(&v_empty[st]);
          ++gv;
        }
        for (int qt = 0; qt < it.nq; ++qt) ++ni[qt];
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax / correction / epilogue ----------------
    const int qt = (warp - 4) / 4;
    const int q = warp & 3;
    const int i = q * 32 + lane;                   // query row within the Q tile
    const uint32_t s_addr = tmem + ((uint32_t)(q * 32) << 16) + qt * C::TCOLS;
    const uint32_t o_addr = s_addr + 128;
    const float sl = 1.4426950408889634f * rsqrtf((float)DH);   // log2(e)/sqrt(d)
    uint64_t* my_p_free = p_free + qt * C::PBUF;
    const int sw = i & 7;
    uint32_t cs = 0;                               // blocks processed by this Q tile (all items)
    for (int64_t id = blockIdx.x; id < n_items; id += gridDim.x) {
      const Item it = item_info<NQ>(ch, heads, id);
      if (qt >= it.nq) continue;
      float m_ref = -INFINITY, l_run = 0.f;
      for (int j = 0; j < it.nkb; ++j, ++cs) {
        tc::mbar_wait(&s_full[qt], cs & 1);
        tc::tc_fence_after();
        float sv[128];
        {
          uint32_t* r = reinterpret_cast<uint32_t*>(sv);
#pragma unroll
          for (int c0 = 0; c0 < 128; c0 += 32)
            tc::tmem_ld32(s_addr + c0, *reinterpret_cast<uint32_t(*)[32]>(r + c0));
          tc::tmem_ld_wait();
        }
        tc::tc_fence_before();
        tc::mbar_arrive(&s_free[qt]);               // TMEM S columns may take the next S
        const int kvalid = it.n - j * 128;
        if (kvalid < 128) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= kvalid) sv[c] = -INFINITY;
        }
        float m0 = sv[0], m1 = sv[1], m2 = sv[2], m3 = sv[3];
#pragma unroll
        for (int c = 4; c < 128; c += 4) {
          m0 = fmaxf(m0, sv[c]); m1 = fmaxf(m1, sv[c + 1]);
          m2 = fmaxf(m2, sv[c + 2]); m3 = fmaxf(m3, sv[c + 3]);
        }
        const float m_blk = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl;
        // PV of block cs-PBUF released this P buffer
        if (cs >= (uint32_t)C::PBUF) tc::mbar_wait(&my_p_free[cs % C::PBUF], ((cs / C::PBUF) - 1) & 1);
        // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
        // (rows whose max did not move get alpha = 1).
        const bool rescaled = j > 0 && __any_sync(0xffffffffu, m_blk > m_ref + kRescaleLog2);
        if (j == 0 || rescaled) {
          const float m_new = fmaxf(m_blk, m_ref);
          if (rescaled) {   // O must hold PV_{j-1} (block cs-1) before it is rescaled
            tc::mbar_wait(&my_p_free[(cs - 1) % C::PBUF], ((cs - 1) / C::PBUF) & 1);
            tc::tc_fence_after();
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
          }
          m_ref = m_new;
        }
        // probabilities -> bf16 P (SW128 K-major), row sum in fp32
        uint8_t* prow = sP + (qt * C::PBUF + cs % C::PBUF) * C::P_BYTES + i * 128;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float p0 = ex2(fmaf(sv[c0 + e], sl, -m_ref));
            const float p1 = ex2(fmaf(sv[c0 + e + 1], sl, -m_ref));
            rs0 += p0;
            rs1 += p1;
            pk[e / 2] = tc::pack_bf16(p0, p1);
          }
          uint8_t* atom = prow + (c0 >> 6) * 16384;
          const int cb = (c0 & 63) >> 3;
          *reinterpret_cast<uint4*>(atom + ((cb ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(atom + (((cb + 1) ^ sw) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        l_run += rs0 + rs1;
        if (rescaled) tc::tmem_st_wait();
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        tc::mbar_arrive(&p_full[qt]);
      }
      // epilogue: O / l for this row of the head's output, then hand O back
      tc::mbar_wait(&my_p_free[(cs - 1) % C::PBUF], ((cs - 1) / C::PBUF) & 1);
      tc::tc_fence_after();
      const int qrow = it.q0 + qt * 128 + i;
      const float inv = 1.f / l_run;
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
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int DH>
bool launch_dh(const void* qkv, int64_t rows, void* out, const ChunkDev& ch, int B, int D, int heads,
               cudaStream_t st) {
  constexpr int NQ = 2;
  using C = AttnCfg<DH, NQ>;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, rows, 3LL * D, 3LL * D, 128, C::AC,
                      DH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static bool attr = false;
  static int sms = 0;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_tc_kernel<DH, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return false;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    attr = true;
  }
  const int64_t n_items = (int64_t)ch.nqp * heads * B;
  if (n_items == 0) return true;
  const unsigned grid = (unsigned)std::min<int64_t>(n_items, sms);   // persistent: one CTA per SM
  attn_tc_kernel<DH, NQ><<<grid, C::THREADS, C::SMEM, st>>>(tm, reinterpret_cast<__nv_bfloat16*>(out), ch, D,
                                                             heads, n_items);
  return true;
}

}  // namespace

bool launch_attention_tc(const void* qkv_bf16, int64_t qkv_rows, void* out_bf16, const ChunkDev& ch, int B, int D,
                         int heads, int d, cudaStream_t st) {
  if (d == 32) return launch_dh<32>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st);
  if (d == 64) return launch_dh<64>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st);
  if (d == 128) return launch_dh<128>(qkv_bf16, qkv_rows, out_bf16, ch, B, D, heads, st);
  return false;
}

}  // namespace orbit2
