// wgrad_tc.cu -- weight gradients of the training step on tcgen05 (
// oracle/train.py: gw["W"] = dY^T X, gw["b"] = sum_m dY).
//
//     dW[n][k] += sum_m dY[m][n] X[m][k]        (contraction over the M tokens)
//     db[n]    += sum_m dY[m][n]                 (optional)
// dY [M][lda] and X [M][ldb] are the token-major activations the forward and the
// backward keep (bf16): the contraction dimension is the ROW index of both, so both
// operands are MN-major -- TMA boxes of [64 tokens][64 columns] (SW128) feed the
// MMA with transposed-operand descriptors (no transpose pass over HBM).
// Split-K over token chunks (the output tiles are few: D x 4D at most), fp32
// accumulation in TMEM, red.global.add.v4.f32 into the caller's gradient (which the
// caller zeroes once per step).  The bias gradient is summed from the same dY
// tiles in shared memory by the epilogue warps while the MMAs run.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int TK = 64;                       // tokens per stage
constexpr int ATOM = TK * 128;               // [64 tokens][64 bf16] = 8 KB

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int BN, int STAGES>
struct WCfg {
  static constexpr int A_BYTES = 2 * ATOM;              // 128 n-columns
  static constexpr int B_BYTES = (BN / 64) * ATOM;
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 + 256;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                 float* __restrict__ out, int64_t ldo, int N, int Kc, int64_t M, int n_tiles_k, int64_t chunks,
                 int splits, float* __restrict__ dbias) {
  using C = WCfg<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int n0 = (tile / n_tiles_k) * 128, k0 = (tile % n_tiles_k) * BN;
  const int64_t c_begin = chunks * split / splits, c_end = chunks * (split + 1) / splits;
  const int nck = (int)(c_end - c_begin);
  const bool bias = dbias != nullptr && (tile % n_tiles_k) == 0;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tma);
    tc::prefetch_tmap(&tmb);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1 + (bias ? 128 : 0));
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer ----------------
      for (int c = 0; c < nck; ++c) {
        const uint32_t s = c % STAGES, ph = (c / STAGES) & 1;
        tc::mbar_wait(&empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES);
        const int32_t m = (int32_t)((c_begin + c) * TK);
        for (int a = 0; a < 2; ++a) tc::tma_load_2d(&tma, sA + s * C::A_BYTES + a * ATOM, &full[s], n0 + a * 64, m);
        for (int b = 0; b < BN / 64; ++b)
          tc::tma_load_2d(&tmb, sB + s * C::B_BYTES + b * ATOM, &full[s], k0 + b * 64, m);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = tc::idesc_bf16(128, BN, 1, 1);   // both operands MN-major
      for (int c = 0; c < nck; ++c) {
        const uint32_t s = c % STAGES, ph = (c / STAGES) & 1;
        tc::mbar_wait(&full[s], ph);
        tc::tc_fence_after();
        const uint64_t ad = tc::sdesc(tc::smem_u32(sA + s * C::A_BYTES), ATOM, 1024, tc::SW_128B);
        const uint64_t bd = tc::sdesc(tc::smem_u32(sB + s * C::B_BYTES), ATOM, 1024, tc::SW_128B);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk) {   // 16 tokens = 2 groups of 8 rows per MMA
          const uint32_t adv = (uint32_t)(kk * 2048) >> 4;
          tc::mma_bf16_ss(tmem, ad + adv, bd + adv, idesc, (c | kk) != 0);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(done);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (thread = output row n0 + r) ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    // bias: thread (a, ch, g) = (r >> 6, (r >> 3) & 7, r & 7) sums the 8 columns
    // 64 a + 8 ch + [0, 8) of dY over the tokens t = 8 i + g of every stage (16-byte loads;
    // the 8 g-lanes of a chunk hit 8 different bank groups), then a 3-step shuffle over g
    float bsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int ga = r >> 6, gch = (r >> 3) & 7, gg = r & 7;
    if (bias) {   // tokens past M are TMA zero-fill
      const uint8_t* abase = sA + ga * ATOM + gg * 128 + ((gch ^ gg) << 4);   // token g, swizzled chunk
      for (int c = 0; c < nck; ++c) {
        const uint32_t s = c % STAGES, ph = (c / STAGES) & 1;
        tc::mbar_wait(&full[s], ph);
        const uint8_t* base = abase + s * C::A_BYTES;
#pragma unroll
        for (int i = 0; i < TK / 8; ++i) {   // token 8 i + g: same swizzle phase (t & 7 == g)
          const uint4 w = *reinterpret_cast<const uint4*>(base + i * 8 * 128);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            bsum[2 * e] += f.x;
            bsum[2 * e + 1] += f.y;
          }
        }
        tc::mbar_arrive(&empty[s]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bsum[j] += __shfl_xor_sync(0xffffffffu, bsum[j], 1);
        bsum[j] += __shfl_xor_sync(0xffffffffu, bsum[j], 2);
        bsum[j] += __shfl_xor_sync(0xffffffffu, bsum[j], 4);
      }
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    if (bias && gg == 0 && nck > 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int nb = n0 + ga * 64 + gch * 8 + j;
        if (nb < N) atomicAdd(dbias + nb, bsum[j]);
      }
    }
    const int n = n0 + r;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      tc::tmem_ld32(taddr + c0, v);
      tc::tmem_ld_wait();
      if (n < N && nck > 0) {
        float* dst = out + (int64_t)n * ldo + k0 + c0;
        const int kv = Kc - (k0 + c0);              // valid columns of this chunk
        if (kv >= 32 && (ldo & 3) == 0) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            red_add_v4(dst + 4 * u, __uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]),
                       __uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3]));
        } else {
          for (int j = 0; j < 32 && j < kv; ++j) atomicAdd(dst + j, __uint_as_float(v[j]));
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, BN);
  }
}

template <int BN, int STAGES>
bool launch_bn(const GemmOperand& A, const GemmOperand& X, int64_t M, int N, int Kc, float* out, int64_t ldo,
               float* dbias, cudaStream_t st) {
  using C = WCfg<BN, STAGES>;
  CUtensorMap ta, tb;
  if (!make_tmap_bf16(&ta, A.ptr, M, N, A.ld, TK, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&tb, X.ptr, M, Kc, X.ld, TK, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(wgrad_kernel<BN, STAGES>), C::SMEM, &attr_done)) return false;
  const int n_tiles_n = (N + 127) / 128, n_tiles_k = (Kc + BN - 1) / BN;
  const int tiles = n_tiles_n * n_tiles_k;
  const int64_t chunks = (M + TK - 1) / TK;
  // split the token range (each split >= 16 chunks = 1024 tokens) so the grid fills whole
  // waves of SMs as well as possible: tiles x splits / (SMs x waves), the fewest splits among
  // the best (fewer fp32 atomics); at most max(32 splits, 16 waves): many short CTAs also
  // spread the slower bias-summing tiles (C3 QKV weight gradient 28.8 -> 20.9 ms, r02bf)
  const int sms = num_sms();
#ifndef ORBIT2_WGRAD_SPLITS_BASE   // many short CTAs balance the bias-summing tiles (r02bf)
#define ORBIT2_WGRAD_SPLITS_BASE 32
#endif
#ifndef ORBIT2_WGRAD_WAVES
#define ORBIT2_WGRAD_WAVES 16
#endif
#ifndef ORBIT2_WGRAD_SPLITS_MAX   // A/B experiments: cap on the token splits
#define ORBIT2_WGRAD_SPLITS_MAX 1 << 30
#endif
  const int64_t smax = std::max<int64_t>(
      1, std::min<int64_t>({std::max<int64_t>(ORBIT2_WGRAD_SPLITS_BASE, (int64_t)ORBIT2_WGRAD_WAVES * sms / tiles),
                            chunks / 16, (int64_t)(ORBIT2_WGRAD_SPLITS_MAX)}));
#ifndef ORBIT2_WGRAD_CHUNK_TARGET   // > 0: at most this many 64-token chunks per CTA (A/B experiments)
#define ORBIT2_WGRAD_CHUNK_TARGET 0
#endif
  int64_t splits = 1, sp_lo = 1, sp_hi = smax;
  if (ORBIT2_WGRAD_CHUNK_TARGET > 0) {   // short token ranges: the CTAs sharing a range stay within L2 reach
    sp_lo = std::max<int64_t>(1, (chunks + ORBIT2_WGRAD_CHUNK_TARGET - 1) / ORBIT2_WGRAD_CHUNK_TARGET);
    sp_hi = 2 * sp_lo;
    splits = sp_lo;
  }
  double best = 0.0;
  for (int64_t sp = sp_lo; sp <= sp_hi; ++sp) {
    const int64_t ctas = tiles * sp, waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff > best + 0.02) {
      best = eff;
      splits = sp;
    }
  }
  if (splits > 65535) splits = 65535;
  dim3 grid((unsigned)tiles, (unsigned)splits);
  wgrad_kernel<BN, STAGES><<<grid, 256, C::SMEM, st>>>(ta, tb, out, ldo, N, Kc, M, n_tiles_k, chunks, (int)splits,
                                                        dbias);
  return true;
}

}  // namespace

bool launch_wgrad_tc(const GemmOperand& dY, const GemmOperand& X, int64_t M, int N, int Kc, float* dW, int64_t ldo,
                     float* db, cudaStream_t st) {
  if (M <= 0 || N <= 0 || Kc <= 0) return true;
  if ((dY.ld * 2) % 16 || (X.ld * 2) % 16) return false;   // TMA row pitch
  if (Kc > 128) return launch_bn<256, 4>(dY, X, M, N, Kc, dW, ldo, db, st);
  return launch_bn<128, 6>(dY, X, M, N, Kc, dW, ldo, db, st);
}

}  // namespace orbit2
