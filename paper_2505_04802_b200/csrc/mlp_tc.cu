// mlp_tc.cu -- fused transformer MLP on tcgen05 for D = 256 (the 9.5M-class
// Reslim):   z += W_2 . GELU(W_1 . x + b_1) + b_2      (R9, exact-erf GELU)
// with x = LN2(z) in bf16.  The 128 x 1024 hidden tile of a row block never
// leaves the SM: S_h = X W_1[h]^T lands in TMEM, 8 epilogue warps apply
// bias + GELU and write bf16 H_h into shared memory (SW128 K-major), and the
// tensor core accumulates O += H_h W_2[:,h]^T in TMEM.  Saves the 2 x 4D x 2 B
// per token hidden-activation round trip through HBM of the unfused pair.
//
// Persistent, one CTA per SM, warp-specialised (384 threads):
//   warp 0 lane 0 : TMA producer: X tile (64 KB) per row block, then W_1 / W_2
//                   slices (32 KB slots) through a 3-slot ring, in the order the
//                   MMA consumes them: W1(0) W1(1) W2(0) W1(2) W2(1) ... W2(7)
//   warp 1 lane 0 : MMA issuer: GEMM1(h) into S buffer h&1 (2 x 128 TMEM cols),
//                   GEMM2(h-1) transposed: O^T = W_2 H^T into 2 x 128 TMEM cols
//                   (features on TMEM lanes, tokens on columns: coalesced z update)
//   warp 2        : TMEM allocator (512 columns)
//   warps 4-11    : epilogue, two warpgroups (64 hidden columns each)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int BM = 128;
constexpr int DM = 256;         // model width D
constexpr int FH = 1024;        // hidden width 4D
constexpr int HC = 128;         // hidden chunk
constexpr int NCH = FH / HC;    // 8 chunks
constexpr int RS = 3;           // ring slots
constexpr int SLOT = 32768;
constexpr int X_BYTES = BM * DM * 2;     // 64 KB
constexpr int H_BYTES = BM * HC * 2;     // 32 KB
constexpr int SMEM = X_BYTES + 2 * H_BYTES + RS * SLOT + 1024 + 512;

__global__ void __launch_bounds__(384, 1)
    mlp_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmW2, const float* __restrict__ b1,
                  const float* __restrict__ b2, float* __restrict__ z, int64_t M) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the __shared__ array (keeps the shared address space: STS, not generic ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sH = sX + X_BYTES;          // [2][H_BYTES]
  uint8_t* sW = sH + 2 * H_BYTES;      // [RS][SLOT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sW + RS * SLOT);
  uint64_t* x_full = bar;
  uint64_t* x_free = x_full + 1;
  uint64_t* w_full = x_free + 1;       // [RS]
  uint64_t* w_empty = w_full + RS;     // [RS]
  uint64_t* s_full = w_empty + RS;     // [2]
  uint64_t* s_free = s_full + 2;       // [2]
  uint64_t* h_full = s_free + 2;       // [2]
  uint64_t* h_free = h_full + 2;       // [2]
  uint64_t* o_full = h_free + 2;
  uint64_t* o_free = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = (M + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmW1);
    tc::prefetch_tmap(&tmW2);
    tc::mbar_init(x_full, 1);
    tc::mbar_init(x_free, 1);
    for (int s = 0; s < RS; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&s_free[s], 256);
      tc::mbar_init(&h_full[s], 256);
      tc::mbar_init(&h_free[s], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_free, 256);
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
      uint32_t it = 0, tl = 0;
      auto slot_begin = [&]() -> uint8_t* {
        const uint32_t s = it % RS, ph = (it / RS) & 1;
        tc::mbar_wait(&w_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&w_full[s], SLOT);
        return sW + s * SLOT;
      };
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl) {
        const int32_t m0 = (int32_t)(tile * BM);
        tc::mbar_wait(x_free, (tl & 1) ^ 1);
        tc::mbar_arrive_expect_tx(x_full, X_BYTES);
        for (int a = 0; a < DM / 64; ++a) tc::tma_load_2d(&tmX, sX + a * 16384, x_full, a * 64, m0);
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
      constexpr uint32_t id1 = tc::idesc_bf16(BM, HC, 0, 0);
      constexpr uint32_t id2 = tc::idesc_bf16(128, BM, 0, 0);   // O^T half: 128 features x 128 tokens
      const uint32_t x_addr = tc::smem_u32(sX), h_addr = tc::smem_u32(sH), w_addr = tc::smem_u32(sW);
      uint32_t it = 0, tl = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl) {
        tc::mbar_wait(x_full, tl & 1);
        tc::tc_fence_after();
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            const uint32_t gc = tl * NCH + s, buf = gc & 1, use = gc >> 1;
            if (use >= 1) tc::mbar_wait(&s_free[buf], (use - 1) & 1);
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
            const uint32_t gc = tl * NCH + h, hb = gc & 1;
            tc::mbar_wait(&h_full[hb], (gc >> 1) & 1);
            if (h == 0) tc::mbar_wait(o_free, (tl & 1) ^ 1);
            tc::tc_fence_after();
            for (int k2 = 0; k2 < 2; ++k2, ++it) {
              const uint32_t sl = it % RS;
              tc::mbar_wait(&w_full[sl], (it / RS) & 1);
              tc::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {     // O^T[f,t] += W2[f, hidden] H[t, hidden]
                const int half = kk >> 2;
                const uint64_t ad =
                    tc::sdesc(w_addr + sl * SLOT + half * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                const uint64_t bd =
                    tc::sdesc(h_addr + hb * H_BYTES + k2 * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ss(tmem + 256 + half * 128, ad, bd, id2, (h | k2 | (kk & 3)) != 0);
              }
              tc::mma_commit(&w_empty[sl]);
            }
            tc::mma_commit(&h_free[hb]);
            if (h == NCH - 1) tc::mma_commit(o_full);
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
    uint32_t tl = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl) {
      for (int h = 0; h < NCH; ++h) {
        const uint32_t gc = tl * NCH + h, buf = gc & 1, use = gc >> 1;
        tc::mbar_wait(&s_full[buf], use & 1);
        tc::tc_fence_after();
        float v[64];
        tc::tmem_ld32(lane_addr + buf * HC + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
        tc::tmem_ld32(lane_addr + buf * HC + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s_free[buf]);
        if (use >= 1) tc::mbar_wait(&h_free[buf], (use - 1) & 1);
        const float4* bb = reinterpret_cast<const float4*>(b1 + h * HC + wg * 64);
        uint8_t* hrow = sH + buf * H_BYTES + wg * 16384 + r * 128;
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const float4 ba = __ldg(bb + 2 * c16), bc = __ldg(bb + 2 * c16 + 1);
          const float* x8 = v + 8 * c16;
          uint4 w;
          w.x = tc::pack_bf16(tc::gelu_erf_fast(x8[0] + ba.x), tc::gelu_erf_fast(x8[1] + ba.y));
          w.y = tc::pack_bf16(tc::gelu_erf_fast(x8[2] + ba.z), tc::gelu_erf_fast(x8[3] + ba.w));
          w.z = tc::pack_bf16(tc::gelu_erf_fast(x8[4] + bc.x), tc::gelu_erf_fast(x8[5] + bc.y));
          w.w = tc::pack_bf16(tc::gelu_erf_fast(x8[6] + bc.z), tc::gelu_erf_fast(x8[7] + bc.w));
          *reinterpret_cast<uint4*>(hrow + ((c16 ^ (r & 7)) << 4)) = w;
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&h_full[buf]);
      }
      // O^T -> residual stream: thread = feature f (TMEM lane), columns = tokens,
      // so each warp access to z[token][f..f+31] is one coalesced 128-byte line.
      tc::mbar_wait(o_full, tl & 1);
      tc::tc_fence_after();
      const int f = wg * 128 + r;
      const float bf = __ldg(b2 + f);
#pragma unroll 1
      for (int c0 = 0; c0 < BM; c0 += 32) {
        uint32_t o[32];
        tc::tmem_ld32(lane_addr + 256 + wg * 128 + c0, o);
        tc::tmem_ld_wait();
        if (c0 == BM - 32) {
          tc::tc_fence_before();
          tc::mbar_arrive(o_free);
        }
        const int64_t t0 = tile * BM + c0;
        float* zc = z + t0 * DM + f;
        if (t0 + 32 <= M) {
          float zv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) zv[j] = zc[(int64_t)j * DM];
#pragma unroll
          for (int j = 0; j < 32; ++j) zc[(int64_t)j * DM] = zv[j] + (__uint_as_float(o[j]) + bf);
        } else {
          for (int j = 0; j < 32; ++j)
            if (t0 + j < M) zc[(int64_t)j * DM] += __uint_as_float(o[j]) + bf;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool launch_mlp_fused(const void* xn, int64_t rows_alloc, const void* w1, const float* b1, const void* w2,
                      const float* b2, float* z, int64_t M, int D, cudaStream_t st) {
  if (D != DM || M <= 0) return false;
  CUtensorMap tx, t1, t2;
  if (!make_tmap_bf16(&tx, xn, rows_alloc, DM, DM, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t1, w1, FH, DM, DM, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t2, w2, DM, FH, FH, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return false;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (M + BM - 1) / BM;
  const int grid = (int)std::min<int64_t>(tiles, sms);
  mlp_tc_kernel<<<grid, 384, SMEM, st>>>(tx, t1, t2, b1, b2, z, M);
  return true;
}

}  // namespace orbit2
