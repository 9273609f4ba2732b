// attn_tc.cu -- per-tile multi-head self-attention on tcgen05 tensor cores.
//
// "self-attention is restricted within each tile"; P:595 / P:583 the
// paper runs Flash Attention.  For every (query block of 128 tokens of a
// tile, head, sample):
//     O = softmax(Q K^T / sqrt(d)) V     over the keys of the SAME tile only
// with an online (flash) softmax over key blocks of 128 (R17, R18).
//
// Roles (256 threads, one query block per CTA):
//   warp 0 lane 0 : TMA producer (Q once; K_j,V_j into a 2-stage ring)
//   warp 1 lane 0 : tcgen05.mma issuer:  S_j = Q K_j^T  -> TMEM buffer j&1
//                                        O_j = P_j V_j  -> same TMEM buffer
//   warp 2        : TMEM allocator (256 columns = 2 buffers x 128)
//   warps 4-7     : softmax; thread i owns query row i (TMEM lane i):
//                   pass A row max of S_j, fold O_{j-1} into a register
//                   accumulator, pass B p = exp2(s*c - m) -> bf16 P_j in smem
//                   (SW128 K-major A operand), row sums in fp32.
// S_{j+1} is computed by the tensor core while the softmax warps run pass B
// of block j.  V is consumed MN-major straight from the TMA tile.
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

template <int DH>
struct AttnCfg {
  static constexpr int AC = DH < 64 ? DH : 64;        // columns per swizzle atom
  static constexpr int RB = AC * 2;                   // bytes per atom row
  static constexpr int NA = DH / AC;                  // atoms per 128-row block
  static constexpr int ATOM = 128 * RB;               // bytes per atom
  static constexpr int TILE = 128 * DH * 2;           // bytes of a Q/K/V block
  static constexpr uint32_t SW = DH == 32 ? tc::SW_64B : tc::SW_128B;
  static constexpr int KVST = 2;
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int SMEM = TILE + 2 * KVST * TILE + P_BYTES + 1024 + 256;
};

template <int DH>
__global__ void __launch_bounds__(256, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out, ChunkDev ch, int D) {
  using C = AttnCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::TILE;
  uint8_t* sV = sK + C::KVST * C::TILE;
  uint8_t* sP = sV + C::KVST * C::TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;             // [KVST]
  uint64_t* kv_empty = kv_full + C::KVST;  // [KVST]
  uint64_t* s_full = kv_empty + C::KVST;   // [2]
  uint64_t* o_full = s_full + 2;           // [2]
  uint64_t* t_free = o_full + 2;           // [2]
  uint64_t* p_full = t_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = ch.qb0 + blockIdx.x;
  const int li = ch.qblk_tile[g];
  const DevTile t = ch.tiles[li];
  const int h = blockIdx.y, b = blockIdx.z;
  const int n = t.n_tokens;
  const int64_t base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  const int q0 = (g - t.qb_off) * 128;
  const int nkb = (n + 127) / 128;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tm);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < C::KVST; ++s) {
      tc::mbar_init(&kv_full[s], 1);
      tc::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&o_full[s], 1);
      tc::mbar_init(&t_free[s], 128);
    }
    tc::mbar_init(p_full, 128);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const int32_t y0 = (int32_t)base;
      tc::mbar_arrive_expect_tx(q_full, C::TILE);
      for (int a = 0; a < C::NA; ++a) tc::tma_load_2d(&tm, sQ + a * C::ATOM, q_full, h * DH + a * C::AC, y0 + q0);
      for (int j = 0; j < nkb; ++j) {
        const int st = j % C::KVST;
        tc::mbar_wait(&kv_empty[st], ((j / C::KVST) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&kv_full[st], 2 * C::TILE);
        for (int a = 0; a < C::NA; ++a) {
          tc::tma_load_2d(&tm, sK + st * C::TILE + a * C::ATOM, &kv_full[st], D + h * DH + a * C::AC, y0 + j * 128);
          tc::tma_load_2d(&tm, sV + st * C::TILE + a * C::ATOM, &kv_full[st], 2 * D + h * DH + a * C::AC,
                          y0 + j * 128);
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
      tc::mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int bf = j & 1, st = j % C::KVST;
        tc::mbar_wait(&kv_full[st], (j / C::KVST) & 1);
        if (j >= 2) tc::mbar_wait(&t_free[bf], ((j - 2) >> 1) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const int a = (kk * 16) / C::AC, off = ((kk * 16) % C::AC) * 2;
          const uint64_t qd = tc::sdesc(q_addr + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
          const uint64_t kd = tc::sdesc(k_addr + st * C::TILE + a * C::ATOM + off, 16, 8 * C::RB, C::SW);
          tc::mma_bf16_ss(tmem + bf * 128, qd, kd, id_s, kk > 0);
        }
        tc::mma_commit(&s_full[bf]);
      };
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) issue_s(j + 1);
        const int bf = j & 1, st = j % C::KVST;
        tc::mbar_wait(p_full, j & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {   // 128 keys, K = 16 per MMA
          const uint64_t pd = tc::sdesc(p_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
          const uint64_t vd = tc::sdesc(v_addr + st * C::TILE + kk * 16 * C::RB, C::ATOM, 8 * C::RB, C::SW);
          tc::mma_bf16_ss(tmem + bf * 128, pd, vd, id_o, kk > 0);
        }
        tc::mma_commit(&o_full[bf]);
        tc::mma_commit(&kv_empty[st]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax / correction / epilogue ----------------
    const int q = warp - 4;
    const int i = q * 32 + lane;                   // query row within the block
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    const float sl = 1.4426950408889634f * rsqrtf((float)DH);   // log2(e)/sqrt(d)
    float m_run = -INFINITY, l_run = 0.f, alpha_prev = 0.f;
    float acc[DH];
#pragma unroll
    for (int c = 0; c < DH; ++c) acc[c] = 0.f;
    uint8_t* prow = sP + i * 128;
    const int sw = i & 7;

    auto fold_o = [&](int jo) {
      const int bf = jo & 1;
      tc::mbar_wait(&o_full[bf], (jo >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld32(lane_addr + bf * 128 + c0, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[c0 + e] = fmaf(acc[c0 + e], alpha_prev, __uint_as_float(r[e]));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&t_free[bf]);
    };

    for (int j = 0; j < nkb; ++j) {
      const int bf = j & 1;
      const int kvalid = n - j * 128;
      tc::mbar_wait(&s_full[bf], (j >> 1) & 1);
      tc::tc_fence_after();
      // pass A: row max
      float mx = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld32(lane_addr + bf * 128 + c0, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (c0 + e < kvalid) mx = fmaxf(mx, __uint_as_float(r[e]));
      }
      const float m_new = fmaxf(m_run, mx * sl);
      const float alpha = ex2(m_run - m_new);
      if (j > 0) fold_o(j - 1);           // frees TMEM buffer of block j-1 and the P buffer
      // pass B: probabilities -> bf16 P_j (SW128 K-major), row sum
      float rs = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld32(lane_addr + bf * 128 + c0, r);
        tc::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float p0 = (c0 + e < kvalid) ? ex2(fmaf(__uint_as_float(r[e]), sl, -m_new)) : 0.f;
          const float p1 = (c0 + e + 1 < kvalid) ? ex2(fmaf(__uint_as_float(r[e + 1]), sl, -m_new)) : 0.f;
          rs += p0 + p1;
          pk[e / 2] = tc::pack_bf16(p0, p1);
        }
        uint8_t* atom = prow + (c0 >> 6) * 16384;
        const int cbase = (c0 & 63) >> 3;   // 16-byte chunk index within the 128-byte row
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4*>(atom + (((cbase + u) ^ sw) << 4)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      l_run = l_run * alpha + rs;
      m_run = m_new;
      alpha_prev = alpha;
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      tc::mbar_arrive(p_full);
    }
    fold_o(nkb - 1);
    // epilogue: normalise and store this row of the head's output
    if (q0 + i < n) {
      const float inv = 1.f / l_run;
      uint4* dst = reinterpret_cast<uint4*>(out + (base + q0 + i) * (int64_t)D + h * DH);
#pragma unroll
      for (int c = 0; c < DH; c += 8)
        dst[c / 8] = make_uint4(tc::pack_bf16(acc[c] * inv, acc[c + 1] * inv), tc::pack_bf16(acc[c + 2] * inv, acc[c + 3] * inv),
                                tc::pack_bf16(acc[c + 4] * inv, acc[c + 5] * inv), tc::pack_bf16(acc[c + 6] * inv, acc[c + 7] * inv));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
}

template <int DH>
bool launch_dh(const void* qkv, int64_t rows, void* out, const ChunkDev& ch, int B, int D, int heads,
               cudaStream_t st) {
  using C = AttnCfg<DH>;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, rows, 3LL * D, 3LL * D, 128, C::AC,
                      DH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_tc_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return false;
    attr = true;
  }
  dim3 grid(ch.nqb, heads, B);
  attn_tc_kernel<DH><<<grid, 256, C::SMEM, st>>>(tm, reinterpret_cast<__nv_bfloat16*>(out), ch, D);
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
