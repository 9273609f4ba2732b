// attn_tc.cu -- per-tile multi-head self-attention on tcgen05 tensor cores.
//
// "self-attention is restricted within each tile"; P:583 / P:595 the
// paper runs Flash Attention.  For every (query block of 128 tokens of a
// tile, head, sample):
//     O = softmax(Q K^T / sqrt(d)) V     over the keys of the SAME tile only
// with an online (flash) softmax over key blocks of 128 (R17, R18).
//
// One CTA handles NQ = 2 query blocks of the same (tile, head, sample) and
// shares every K/V block between them (FA4-style ping-pong of two Q tiles):
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
  static constexpr int KST = DH == 128 ? 1 : 2;       // K ring (consumed by S_{j+1}, early)
  static constexpr int VST = DH == 128 ? 1 : 2;       // V ring (consumed by PV_j, late)
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int THREADS = 128 + 128 * NQ;
  static constexpr int TCOLS = 128 + DH;              // TMEM columns per Q tile: S | O
  static constexpr int TMEM_COLS = NQ * TCOLS <= 256 ? 256 : 512;
  static constexpr int PBUF = DH == 128 ? 1 : 2;      // P buffers per Q tile (DH=64: 224 KB smem)
  static constexpr int SMEM = NQ * TILE + (KST + VST) * TILE + NQ * PBUF * P_BYTES + 1024 + 512;
};

// Conditional rescale threshold (log2 units): the reference max of a row is
// only moved when the running max exceeds it by more than 8, so probabilities
// stay <= 2^8 (exact in bf16's exponent range, fp32 accumulation) and the
// O rescale in TMEM is rare.  Mathematically identical softmax (R18).
constexpr float kRescaleLog2 = 8.0f;

template <int DH, int NQ>
__global__ void __launch_bounds__(AttnCfg<DH, NQ>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out, ChunkDev ch, int D) {
  using C = AttnCfg<DH, NQ>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                               // [NQ][TILE]
  uint8_t* sK = sQ + NQ * C::TILE;                  // [KST][TILE]
  uint8_t* sV = sK + C::KST * C::TILE;              // [VST][TILE]
  uint8_t* sP = sV + C::VST * C::TILE;              // [NQ][PBUF][P_BYTES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + NQ * C::PBUF * C::P_BYTES);
  uint64_t* q_full = bar;                           // 1
  uint64_t* k_full = q_full + 1;                    // [KST]
  uint64_t* k_empty = k_full + C::KST;              // [KST]
  uint64_t* v_full = k_empty + C::KST;              // [VST]
  uint64_t* v_empty = v_full + C::VST;              // [VST]
  uint64_t* s_full = v_empty + C::VST;              // [NQ]  S_j in TMEM
  uint64_t* s_free = s_full + NQ;                   // [NQ]  softmax has S_j in registers
  uint64_t* p_full = s_free + NQ;                   // [NQ]  P_j in smem (+ O rescaled)
  uint64_t* p_free = p_full + NQ;                   // [NQ][PBUF]  PV done reading P buffer (and O updated)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + NQ * C::PBUF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = ch.qp0 + blockIdx.x;
  const int li = ch.qpair_tile[g];
  const DevTile t = ch.tiles[li];
  const int h = blockIdx.y, b = blockIdx.z;
  const int n = t.n_tokens;
  const int64_t base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  const int q0 = (g - t.qp_off) * 128 * NQ;          // first query of Q tile 0
  const int nq = min(NQ, (n - q0 + 127) / 128);     // active Q tiles in this CTA
  const int nkb = (n + 127) / 128;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm);
    tc::mbar_init(q_full, 1);
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
      const int32_t y0 = (int32_t)base;
      tc::mbar_arrive_expect_tx(q_full, nq * C::TILE);
      for (int qt = 0; qt < nq; ++qt)
        for (int a = 0; a < C::NA; ++a)
          tc::tma_load_2d(&tm, sQ + qt * C::TILE + a * C::ATOM, q_full, h * DH + a * C::AC, y0 + q0 + qt * 128);
      // issue order = consumption order: K_0, then per j: K_{j+1}, V_j
      auto load_k = [&](int j) {
        const int st = j % C::KST;
        tc::mbar_wait(&k_empty[st], ((j / C::KST) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&k_full[st], C::TILE);
        for (int a = 0; a < C::NA; ++a)
          tc::tma_load_2d(&tm, sK + st * C::TILE + a * C::ATOM, &k_full[st], D + h * DH + a * C::AC, y0 + j * 128);
      };
      auto load_v = [&](int j) {
        const int st = j % C::VST;
        tc::mbar_wait(&v_empty[st], ((j / C::VST) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&v_full[st], C::TILE);
        for (int a = 0; a < C::NA; ++a)
          tc::tma_load_2d(&tm, sV + st * C::TILE + a * C::ATOM, &v_full[st], 2 * D + h * DH + a * C::AC,
                          y0 + j * 128);
      };
      load_k(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t id_o = tc::idesc_bf16(128, DH, 0, 1);    // P K-major, V MN-major
      const uint32_t q_addr = tc::smem_u32(sQ), k_addr = tc::smem_u32(sK), v_addr = tc::smem_u32(sV);
      const uint32_t p_addr = tc::smem_u32(sP);
      auto issue_s = [&](int j, int qt) {
        const int st = j % C::KST;
        if (j >= 1) tc::mbar_wait(&s_free[qt], (j - 1) & 1);   // softmax holds S_{j-1} in registers
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const int a = (kk * 16) / C::AC, off = ((kk * 16) % C::AC) * 2;
          const uint64_t qd = tc::sdesc(q_addr + qt * C::TILE + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
          const uint64_t kd = tc::sdesc(k_addr + st * C::TILE + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
          tc::mma_bf16_ss(tmem + qt * C::TCOLS, qd, kd, id_s, kk > 0);
        }
        tc::mma_commit(&s_full[qt]);
      };
      auto issue_pv = [&](int j, int qt) {
        const int st = j % C::VST;
        tc::mbar_wait(&p_full[qt], j & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // 128 keys, K = 16 per MMA
          const uint64_t pd = tc::sdesc(p_addr + (qt * C::PBUF + j % C::PBUF) * C::P_BYTES + (kk >> 2) * 16384 +
                                            (kk & 3) * 32, 16, 1024, tc::SW_128B);
          const uint64_t vd = tc::sdesc(v_addr + st * C::TILE + kk * 16 * C::RB, C::ATOM, 8 * C::RB, C::SW);
          tc::mma_bf16_ss(tmem + qt * C::TCOLS + 128, pd, vd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&p_free[qt * C::PBUF + j % C::PBUF]);
      };
      tc::mbar_wait(q_full, 0);
      tc::mbar_wait(&k_full[0], 0);
      for (int qt = 0; qt < nq; ++qt) issue_s(0, qt);
      tc::mma_commit(&k_empty[0]);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) {   // S_{j+1} overlaps the softmax of block j
          tc::mbar_wait(&k_full[(j + 1) % C::KST], ((j + 1) / C::KST) & 1);
          for (int qt = 0; qt < nq; ++qt) issue_s(j + 1, qt);
          tc::mma_commit(&k_empty[(j + 1) % C::KST]);
        }
        tc::mbar_wait(&v_full[j % C::VST], (j / C::VST) & 1);
        for (int qt = 0; qt < nq; ++qt) issue_pv(j, qt);
        tc::mma_commit(&v_empty[j % C::VST]);
      }
    }
  } else if (warp >= 4 && (warp - 4) / 4 < nq) {
    // ---------------- softmax / correction / epilogue ----------------
    const int qt = (warp - 4) / 4;
    const int q = warp & 3;
    const int i = q * 32 + lane;                   // query row within the Q tile
    const uint32_t s_addr = tmem + ((uint32_t)(q * 32) << 16) + qt * C::TCOLS;
    const uint32_t o_addr = s_addr + 128;
    const float sl = 1.4426950408889634f * rsqrtf((float)DH);   // log2(e)/sqrt(d)
    float m_ref = -INFINITY, l_run = 0.f;
    uint64_t* my_p_free = p_free + qt * C::PBUF;
    const int sw = i & 7;

    for (int j = 0; j < nkb; ++j) {
      tc::mbar_wait(&s_full[qt], j & 1);
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
      tc::mbar_arrive(&s_free[qt]);               // TMEM S buffer may take S_{j+1}
      const int kvalid = n - j * 128;
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
      // PV_{j-PBUF} has released this P buffer (PV_{j-1} too when PBUF == 1)
      if (j >= C::PBUF) tc::mbar_wait(&my_p_free[j % C::PBUF], ((j / C::PBUF) - 1) & 1);
      // tcgen05.ld/st are warp-collective: the rescale decision is warp-uniform
      // (rows whose max did not move get alpha = 1).
      const bool rescaled = j > 0 && __any_sync(0xffffffffu, m_blk > m_ref + kRescaleLog2);
      if (j == 0 || rescaled) {
        const float m_new = fmaxf(m_blk, m_ref);
        if (rescaled) {
          // O must hold PV_{j-1} before it is rescaled
          tc::mbar_wait(&my_p_free[(j - 1) % C::PBUF], ((j - 1) / C::PBUF) & 1);
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
      // probabilities -> bf16 P_j (SW128 K-major), row sum in fp32
      uint8_t* prow = sP + (qt * C::PBUF + j % C::PBUF) * C::P_BYTES + i * 128;
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
    // epilogue: O / l for this row of the head's output
    tc::mbar_wait(&my_p_free[(nkb - 1) % C::PBUF], ((nkb - 1) / C::PBUF) & 1);
    tc::tc_fence_after();
    const int qrow = q0 + qt * 128 + i;
    const float inv = 1.f / l_run;
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 16) {
      uint32_t r[16];
      tc::tmem_ld16(o_addr + c0, r);
      tc::tmem_ld_wait();
      if (qrow < n) {
        uint4* dst = reinterpret_cast<uint4*>(out + (base + qrow) * (int64_t)D + h * DH + c0);
#pragma unroll
        for (int u = 0; u < 2; ++u)
          dst[u] = make_uint4(tc::pack_bf16(__uint_as_float(r[8 * u]) * inv, __uint_as_float(r[8 * u + 1]) * inv),
                              tc::pack_bf16(__uint_as_float(r[8 * u + 2]) * inv, __uint_as_float(r[8 * u + 3]) * inv),
                              tc::pack_bf16(__uint_as_float(r[8 * u + 4]) * inv, __uint_as_float(r[8 * u + 5]) * inv),
                              tc::pack_bf16(__uint_as_float(r[8 * u + 6]) * inv, __uint_as_float(r[8 * u + 7]) * inv));
      }
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
  if (!attr) {
    if (cudaFuncSetAttribute(attn_tc_kernel<DH, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return false;
    attr = true;
  }
  dim3 grid(ch.nqp, heads, B);
  attn_tc_kernel<DH, NQ><<<grid, C::THREADS, C::SMEM, st>>>(tm, reinterpret_cast<__nv_bfloat16*>(out), ch, D);
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
